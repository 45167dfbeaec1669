"""A/B timing of the group-layout element-wise kernels (ReLU, cmp, GELU, exp clamp)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19711_b200 as m
import workloads
flush = torch.empty(128 << 20, dtype=torch.int32, device="cuda")


def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    tot = 0.0
    for i in range(reps):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps


c = m.Ctx.for_cfg(workloads.keys(4))
sh = lambda x: c.share(torch.from_numpy(x.ravel()).cuda())
r = sh(workloads.relu_inputs(32 * 64 * 112 * 112 // 4))
g = sh(workloads.normal_inputs(workloads.SHAPES["cfg3_gelu"], 3))
e = sh(workloads.exp_inputs(1 << 22))
res = {"relu": t(lambda: c.relu(r)), "cmp": t(lambda: c.cmp(r)), "gelu_abs4": t(lambda: c.gelu(g, form="poly_abs", degree=4)),
       "gelu_x4": t(lambda: c.gelu(g, form="poly_x", degree=4)), "exp_clamp": t(lambda: c.exp(e, clamp=1)),
       "cmp_w64": t(lambda: c.cmp(r, window=64))}
print(os.environ.get("MPC200_LIB", "new")[-18:], " ".join(f"{k} {v:.4f}" for k, v in res.items()))
