"""Quick timing of the PAIR protocol in loopback vs BOTH on one GPU (A/B with MPC200_LIB)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19711_b200 as m
import workloads


def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


keys = workloads.keys(2)
rows, cols = workloads.SHAPES["cfg2_softmax"]
for mode in (m.binding.MODE_BOTH, m.binding.MODE_PAIR_LOOPBACK):
    c = m.Ctx.for_cfg(keys, mode=mode)
    x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols).ravel()).cuda())
    g = c.share(torch.from_numpy(workloads.normal_inputs(1 << 20, 3)).cuda())
    r = c.share(torch.from_numpy(workloads.relu_inputs(1 << 22)).cuda())
    ln = c.share(torch.from_numpy(workloads.layernorm_inputs(2048, 768).ravel()).cuda())
    res = {"softmax": t(lambda: c.softmax(x, rows, cols)),
           "softmax_clamp": t(lambda: c.softmax(x, rows, cols, exp_clamp=1)),
           "gelu1M": t(lambda: c.gelu(g, form="poly_abs", degree=4)),
           "gelu1M_x4": t(lambda: c.gelu(g, form="poly_x", degree=4)),
           "exp1M_clamp": t(lambda: c.exp(g, clamp=1)),
           "relu4M": t(lambda: c.relu(r)),
           "mul4M": t(lambda: c.mul(r, r)),
           "ln2048": t(lambda: c.layernorm(ln, 2048, 768))}
    c.set_ltz_circuit(1)
    res["softmax_cone"] = t(lambda: c.softmax(x, rows, cols))
    res["gelu1M_cone"] = t(lambda: c.gelu(g, form="poly_abs", degree=4))
    res["relu4M_cone"] = t(lambda: c.relu(r))
    c.set_ltz_circuit(0)
    print("BOTH    " if mode == m.binding.MODE_BOTH else "LOOPBACK", " ".join(f"{k} {v:.3f}" for k, v in res.items()))
    if mode != m.binding.MODE_BOTH:
        c.sync()
