"""Phase probe for a split softmax: times the fused cfg2 softmax next to the standalone ops a split
pipeline would run (row max tree, element-wise exp, per-row reciprocal, element product), each on
cfg2's shapes, for the default library and A/B builds (MPC200_LIB, one process per library).
python tools/split_probe.py [abtmp/lib_x.so ...]"""
import os
import subprocess
import sys

code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2511_19711_b200 as m, workloads
c = m.Ctx.for_cfg(workloads.keys(2))
rows, cols = workloads.SHAPES["cfg2_softmax"]
n = rows * cols
x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
z = c._empty(n)
mx = c._empty(rows)
rs = c.share(torch.from_numpy(workloads.act_inputs(rows, lo=1, hi=128)).cuda())
rz = c._empty(rows)
d = c.share(torch.from_numpy(workloads.act_inputs(n, lo=-8, hi=0)).cuda())
s = torch.cuda.current_stream()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps): fn()
    b.record(s); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
r = [f"softmax {t(lambda: c.softmax(x, rows, cols, out=z)):.4f}",
     f"max {t(lambda: c.max(x, rows, cols, out=mx)):.4f}",
     f"exp {t(lambda: c.exp(d, t=8, out=z)):.4f}",
     f"recip(rows) {t(lambda: c.recip(rs, out=rz)):.4f}",
     f"mul {t(lambda: c.mul(d, d, trunc_bits=16, out=z)):.4f}"]
print(os.path.basename(os.environ.get("MPC200_LIB", "default")), " | ".join(r), flush=True)
'''
for rep in range(2):
    for lib in [None] + sys.argv[1:]:
        env = dict(os.environ)
        if lib:
            env["MPC200_LIB"] = lib
        subprocess.run([sys.executable, "-c", code], env=env, check=True)
