"""Summarise an `ncu --metrics gpu__time_duration.sum` launch list (cold-cache, serialised):
per-kernel launch count, mean duration and share of the listed GPU time."""
import collections
import csv
import io
import sys


def main(path, out):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    agg = collections.defaultdict(list)
    for r in rows:
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        agg[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]) * scale)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"launch list {path}: {len(rows)} launches, {tot / 1e3:.3f} ms listed GPU time (ncu, serialised)",
             f"{'kernel':70s} {'n':>4s} {'mean_us':>10s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:70]:70s} {len(v):4d} {sum(v) / len(v):10.1f} {100 * sum(v) / tot:6.1f}%")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
