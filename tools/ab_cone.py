"""A/B of the carry-cone paths (BOTH): cmp w=33/64, ReLU cfg4 shard w=33/21, MaxPool cfg4 shard,
cfg2 softmax and cfg3 GELU with the cone, for the default library and builds on the command line."""
import os
import subprocess
import sys

code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2511_19711_b200 as m, workloads
c = m.Ctx.for_cfg(workloads.keys(4))
c.set_ltz_circuit(1)
s = torch.cuda.current_stream()
def t(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps): fn()
    b.record(s); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
n = 1 << 22
x = c.share(torch.from_numpy(workloads.act_inputs(n)).cuda())
N, C, H, W = workloads.SHAPES["cfg4_relu_first"]
n4 = N * C * H * W // 4
r = c.share(torch.from_numpy(workloads.relu_inputs(n4)).cuda())
mp = c.share(torch.from_numpy(workloads.maxpool_inputs((8, 64, 112, 112))).cuda())
rows, cols = workloads.SHAPES["cfg2_softmax"]
sm = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
n3 = workloads.SHAPES["cfg3_gelu"]
g = c.share(torch.from_numpy(workloads.normal_inputs(n3, 3)).cuda())
res = [f"cmp33 {t(lambda: c.cmp(x, window=33)):.4f}", f"cmp64 {t(lambda: c.cmp(x, window=64)):.4f}",
       f"relu33 {t(lambda: c.relu(r, window=33)):.4f}", f"relu21 {t(lambda: c.relu(r, window=21)):.4f}",
       f"maxpool {t(lambda: c.maxpool2d(mp, 8, 64, 112, 112)):.4f}",
       f"softmax {t(lambda: c.softmax(sm, rows, cols)):.4f}",
       f"gelu {t(lambda: c.gelu(g, form='poly_abs', degree=4)):.4f}"]
print(os.path.basename(os.environ.get("MPC200_LIB", "default")), " | ".join(res), flush=True)
'''
for rep in range(2):
    for lib in [None] + sys.argv[1:]:
        env = dict(os.environ)
        if lib:
            env["MPC200_LIB"] = lib
        subprocess.run([sys.executable, "-c", code], env=env, check=True)
