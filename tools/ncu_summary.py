"""Summarise an ncu --set full report (one kernel launch) into profiles/: duration, DRAM
traffic, pipe utilisation, occupancy, stall reasons and the executed SASS mix.
Usage: python tools/ncu_summary.py <report.ncu-rep> <out.txt> [traffic.json key]"""
import collections
import csv
import io
import json
import os
import subprocess
import sys


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0}


def raw_metrics(rep):
    """metric -> value; byte and time metrics converted to bytes / seconds"""
    txt = ncu([rep, "--page", "raw", "--csv"])
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2]
    out = {}
    for name, unit, val in zip(h, u, v):
        if unit in SCALE:
            try:
                val = repr(float(val) * SCALE[unit])
            except ValueError:
                pass
        out[name] = val
    return out


def sass_mix(rep):
    txt = ncu([rep, "--page", "source", "--csv"])
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    iS, iE = h.index("Source"), h.index("Instructions Executed")
    c, tot = collections.Counter(), 0
    for r in rows[2:]:
        if len(r) <= iE or not r[iS].strip():
            continue
        op = r[iS].strip().split()
        mn = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        n = int(r[iE] or 0)
        c[mn] += n
        tot += n
    return c, tot


def main():
    rep, out = sys.argv[1], sys.argv[2]
    m = raw_metrics(rep)
    keys = [
        ("kernel", "Kernel Name"), ("duration_s", "gpu__time_duration.sum"),
        ("dram_read_bytes", "dram__bytes_read.sum"), ("dram_write_bytes", "dram__bytes_write.sum"),
        ("dram_throughput_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("issue_active_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        ("fmaheavy_pct", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("fma_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        ("alu_pct", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        ("tensor_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("achieved_occupancy_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("registers_per_thread", "launch__registers_per_thread"), ("grid", "launch__grid_size"),
        ("block", "launch__block_size"), ("sm_clock_hz", "smsp__cycles_elapsed.avg.per_second"),
    ]
    lines, summ = [], {}
    for k, name in keys:
        val = m.get(name, "n/a")
        summ[k] = val
        lines.append(f"{k:28s} {val:>20s}   ({name})")
    stalls = sorted(((float(v or 0), k) for k, v in m.items()
                     if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                    reverse=True)[:8]
    lines.append("\ntop stall reasons (warps per issue):")
    for v, k in stalls:
        lines.append(f"  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {v:.3f}")
    c, tot = sass_mix(rep)
    lines.append(f"\nexecuted SASS (warp instructions) total {tot}:")
    for k, v in c.most_common(16):
        lines.append(f"  {k:22s} {v:12d} {100 * v / max(tot, 1):5.1f}%")
    with open(out, "w") as fh:
        fh.write(f"ncu --set full summary of {os.path.basename(rep)}\n\n" + "\n".join(lines) + "\n")
    if len(sys.argv) > 3:
        tj = os.path.join(os.path.dirname(out), "traffic.json")
        d = json.load(open(tj)) if os.path.exists(tj) else {}
        d[sys.argv[3]] = {"dram_bytes": int(float(summ["dram_read_bytes"] or 0) + float(summ["dram_write_bytes"] or 0)),
                          "duration_s": float(summ["duration_s"] or 0), "report": os.path.basename(rep),
                          "kernel": summ["kernel"]}
        json.dump(d, open(tj, "w"), indent=1)
    print("\n".join(lines[:14]))


if __name__ == "__main__":
    main()
