"""A/B of per-op device times (cfg2 softmax, cfg3 GELU, Beaver mul, exp) between the default
library and A/B builds given on the command line (MPC200_LIB, one process per library)."""
import os, subprocess, sys

code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2511_19711_b200 as m, workloads
c = m.Ctx.for_cfg(workloads.keys(2))
rows, cols = workloads.SHAPES["cfg2_softmax"]
x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
z = c._empty(rows * cols)
n3 = workloads.SHAPES["cfg3_gelu"]
g = c.share(torch.from_numpy(workloads.normal_inputs(n3, 3)).cuda())
z3 = c._empty(n3)
s = torch.cuda.current_stream()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps): fn()
    b.record(s); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
r5, c5 = workloads.SHAPES["cfg5_ln"]
l5 = c.share(torch.from_numpy(workloads.layernorm_inputs(r5, c5)).cuda())
z5 = c._empty(r5 * c5)
r = [f"softmax {t(lambda: c.softmax(x, rows, cols, out=z)):.4f}",
     f"layernorm {t(lambda: c.layernorm(l5, r5, c5, out=z5)):.4f}",
     f"relu {t(lambda: c.relu(g, out=z3)):.4f}",
     f"gelu {t(lambda: c.gelu(g, form='poly_abs', degree=4, out=z3)):.4f}",
     f"exp {t(lambda: c.exp(g, t=8, out=z3)):.4f}",
     f"mul {t(lambda: c.mul(g, g, trunc_bits=16, out=z3)):.4f}"]
print(os.environ.get("MPC200_LIB", "default"), " | ".join(r))
'''
for rep in range(2):
    for lib in [None] + sys.argv[1:]:
        env = dict(os.environ)
        if lib:
            env["MPC200_LIB"] = lib
        subprocess.run([sys.executable, "-c", code], env=env, check=True)
