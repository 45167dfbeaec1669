"""Measure the device Philox4x32-10 rate (the ALU roofline's generator) on cuda:0:
mpc_prg_fill with `reps` chained blocks per thread, so memory traffic is negligible."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_19711_b200 as m  # noqa: E402


def main():
    ctx = m.Ctx(1, 2, 3)
    res = {}
    for n, reps in ((148 * 2048, 200), (148 * 2048 * 4, 100)):
        ctx.prg_fill(7, 0, 1, 2, n, reps)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            ctx.prg_fill(7, 0, 1, 2, n, reps)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        res[f"n={n},reps={reps}"] = {"ms": ms, "gblocks_per_s": n * reps / (ms / 1e3) / 1e9}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
