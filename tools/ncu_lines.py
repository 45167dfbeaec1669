"""Hot source lines of one ncu --set full --import-source on report: warp-stall samples and executed
instructions per CUDA source line (needs -lineinfo).  Usage: python tools/ncu_lines.py <rep> <out.txt> [N]"""
import csv
import io
import subprocess
import sys


def main(rep, out, n=45):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hi = next(i for i, r in enumerate(rows) if "Source" in r)
    h = rows[hi]
    def col(*names):
        for nm in names:
            for i, x in enumerate(h):
                if x.strip() == nm:
                    return i
        return None
    iS, iL = col("Source"), col("#", "Line")
    iW = col("Warp Stall Sampling (All Samples)", "Warp Stall Sampling (All Cycles)")
    iE = col("Instructions Executed")
    recs, file_ = [], ""
    tot_w = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= max(x for x in (iS, iW, iE) if x is not None):
            if r and r[0].startswith("File"):
                file_ = r[0]
            continue
        try:
            w = float(r[iW] or 0)
            e = float(r[iE] or 0) if iE is not None else 0.0
        except ValueError:
            continue
        tot_w += w
        recs.append((w, e, r[iL] if iL is not None else "", r[iS].strip()[:110]))
    recs.sort(reverse=True)
    with open(out, "w") as fh:
        fh.write(f"hot CUDA source lines of {rep} (warp-stall samples, % of all; executed warp instructions)\n")
        fh.write(f"columns: {h[:8]}\n")
        for w, e, ln, src in recs[:n]:
            fh.write(f"{100 * w / max(tot_w, 1):6.2f}%  {e:12.0f}  L{ln:>5}  {src}\n")
    print(open(out).read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 45)
