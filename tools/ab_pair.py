"""A/B of PAIR-loopback device times (both parties' kernels on one GPU) between the default
library and builds given on the command line (MPC200_LIB, one process per library)."""
import os
import subprocess
import sys

code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2511_19711_b200 as m, workloads
c = m.Ctx.for_cfg(workloads.keys(2), mode=m.binding.MODE_PAIR_LOOPBACK)
rows, cols = workloads.SHAPES["cfg2_softmax"]
x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols).ravel()).cuda())
g = c.share(torch.from_numpy(workloads.normal_inputs(1 << 20, 3)).cuda())
r = c.share(torch.from_numpy(workloads.relu_inputs(1 << 22)).cuda())
s = torch.cuda.current_stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps): fn()
    b.record(s); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
res = [f"softmax {t(lambda: c.softmax(x, rows, cols)):.4f}",
       f"gelu1M {t(lambda: c.gelu(g, form='poly_abs', degree=4)):.4f}",
       f"relu4M {t(lambda: c.relu(r)):.4f}",
       f"mul4M {t(lambda: c.mul(r, r, trunc_bits=16)):.4f}"]
c.set_ltz_circuit(1)
res.append(f"relu4M_cone {t(lambda: c.relu(r)):.4f}")
c.sync()
print(os.environ.get("MPC200_LIB", "default"), " | ".join(res))
'''
for rep in range(2):
    for lib in [None] + sys.argv[1:]:
        env = dict(os.environ)
        if lib:
            env["MPC200_LIB"] = lib
        subprocess.run([sys.executable, "-c", code], env=env, check=True)
