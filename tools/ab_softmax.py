"""A/B timing of the row kernels (softmax cfg2 / 1024-wide, max) for the library in MPC200_LIB."""
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
res = []
for rows, cols in ((12288, 128), (12288, 1024)):
    x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
    z = c._empty(rows * cols)
    mx = c._empty(rows)
    res.append(f"softmax {rows}x{cols} {t(lambda: c.softmax(x, rows, cols, out=z)):.4f}")
    res.append(f"clamp {t(lambda: c.softmax(x, rows, cols, exp_clamp=1, out=z)):.4f}")
    res.append(f"max {t(lambda: c.max(x, rows, cols, out=mx)):.4f}")
print(os.environ.get("MPC200_LIB", "default"), " | ".join(res))
