"""A/B of the row kernels' half-tile tail (kernels.cuh tile_plan): MPC_TAIL_HALF=0 / 1, one process
each (the knob is read once per process), cfg2 softmax (+ clamp, + bcast), cfg5 1024-wide softmax
rows and the standalone max on the cfg2 shape; L2 flushed between steps as bench.py does."""
import os
import subprocess
import sys

code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2511_19711_b200 as m, workloads
c = m.Ctx.for_cfg(workloads.keys(2))
rows, cols = workloads.SHAPES["cfg2_softmax"]
x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
z = c._empty(rows * cols)
zm = c._empty(rows)
r5 = 12288
x5 = c.share(torch.from_numpy(workloads.softmax_inputs(r5, 1024)).cuda())
z5 = c._empty(r5 * 1024)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); fn(); b.record(s)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps
r = [f"softmax {t(lambda: c.softmax(x, rows, cols, out=z)):.4f}",
     f"softmax_clamp {t(lambda: c.softmax(x, rows, cols, exp_clamp=1, out=z)):.4f}",
     f"softmax_bcast {t(lambda: c.softmax(x, rows, cols, bcast=1, out=z)):.4f}",
     f"softmax1024 {t(lambda: c.softmax(x5, r5, 1024, out=z5), 5):.4f}",
     f"max {t(lambda: c.max(x, rows, cols, out=zm)):.4f}"]
print("MPC_TAIL_HALF=" + os.environ.get("MPC_TAIL_HALF", "1"), " | ".join(r), flush=True)
'''
for rep in range(2):
    for half in ("0", "1"):
        env = dict(os.environ, MPC_TAIL_HALF=half)
        subprocess.run([sys.executable, "-c", code], env=env, check=True)
