"""Quick timing of the PAIR protocol in loopback vs BOTH on one GPU."""
import os, sys, time
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
    print(mode, "softmax ms", round(t(lambda: c.softmax(x, rows, cols)), 3),
          "gelu(1M) ms", round(t(lambda: c.gelu(g, form="poly_abs", degree=4)), 3),
          "relu(4M) ms", round(t(lambda: c.relu(r)), 3),
          "mul(4M) ms", round(t(lambda: c.mul(r, r)), 3))
    if mode != m.binding.MODE_BOTH:
        c.sync()
