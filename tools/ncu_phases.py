"""Attribute an ncu source-page export (--print-source cuda,sass, csv) of one kernel to phases given as
kernels.cuh line ranges: every SASS instruction takes the phase of its own kernels.cuh line, or, for
code inlined from helpers (dev_common / proto_both / sched), the phase of the nearest preceding
address that has one.  Usage: python tools/ncu_phases.py <export.csv[.gz]> name:lo-hi ..."""
import csv
import gzip
import io
import sys


def main(path, specs):
    phases = []
    for s in specs:
        nm, rg = s.split(":")
        lo, hi = (int(v) for v in rg.split("-"))
        phases.append((nm, lo, hi))
    raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
    rows = list(csv.reader(io.StringIO(raw)))
    insts = []            # (addr, file, line, samples, executed, mnemonic)
    file_, line_ = "", 0
    h = None
    for r in rows:
        if r and r[0] == "File Path":
            file_ = r[1]
            continue
        if r and r[0] == "Line No":
            h = r
            continue
        if h is None or len(r) < 8:
            continue
        if r[0]:
            line_ = int(r[0])
            continue
        try:
            addr = int(r[2], 16)
        except ValueError:
            continue
        insts.append((addr, file_.split("/")[-1], line_, float(r[4] or 0), float(r[7] or 0), r[3].split()[0] if r[3].split() else ""))
    insts.sort()
    def phase_of(f, ln):
        if f != "kernels.cuh":
            return None
        for nm, lo, hi in phases:
            if lo <= ln <= hi:
                return nm
        return "other"
    cur = "prologue"
    tot = {}
    for addr, f, ln, w, e, mn in insts:
        p = phase_of(f, ln)
        if p is not None:
            cur = p
        t = tot.setdefault(cur, [0.0, 0.0, 0.0])
        t[0] += w; t[1] += e
        if mn.startswith("IMAD.WIDE"):
            t[2] += e
    W = sum(v[0] for v in tot.values())
    E = sum(v[1] for v in tot.values())
    print(f"{'phase':12s} {'stall samples %':>16s} {'warp instr %':>13s} {'IMAD.WIDE (M)':>14s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:12s} {100 * v[0] / W:16.1f} {100 * v[1] / E:13.1f} {v[2] / 1e6:14.2f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
