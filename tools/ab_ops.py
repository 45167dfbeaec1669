"""A/B timing of element-wise and row ops in BOTH mode (library from MPC200_LIB)."""
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


c = m.Ctx.for_cfg(workloads.keys(2))
sh = lambda x: c.share(torch.from_numpy(x.ravel()).cuda())
x = sh(workloads.softmax_inputs(12288, 128))
g = sh(workloads.normal_inputs(workloads.SHAPES["cfg3_gelu"], 3))
e = sh(workloads.exp_inputs(1 << 22))
ln = sh(workloads.layernorm_inputs(8192, 768))
r = {"softmax": t(lambda: c.softmax(x, 12288, 128)), "softmax_sq": t(lambda: c.softmax(x, 12288, 128, exp_square=1, recip_square=1)),
     "gelu": t(lambda: c.gelu(g, form="poly_abs", degree=4)), "exp4M": t(lambda: c.exp(e)),
     "recip4M": t(lambda: c.recip(e)), "mul4M": t(lambda: c.mul(e, e, trunc_bits=16)), "ln": t(lambda: c.layernorm(ln, 8192, 768))}
print(os.environ.get("MPC200_LIB", "new")[-20:], " ".join(f"{k} {v:.4f}" for k, v in r.items()))
