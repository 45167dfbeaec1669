"""Wave-quantization probe for the fused softmax: time per 32-row tile at tile counts that are
multiples / non-multiples of the resident CTA slots (148 SMs x 2 CTAs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19711_b200 as m
import workloads

flush = torch.empty(128 << 20, dtype=torch.int32, device="cuda")


def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    tot = 0.0
    for i in range(reps):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps


c = m.Ctx.for_cfg(workloads.keys(2))
cols = 128
for tiles in (148, 222, 296, 384, 444, 592, 888):
    rows = 32 * tiles
    x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols).ravel()).cuda())
    z = c._empty(rows * cols)
    ms = t(lambda: c.softmax(x, rows, cols, out=z))
    mx = c._empty(rows)
    ms_max = t(lambda: c.max(x, rows, cols, out=mx))
    e = t(lambda: c.exp(x, out=z))
    print(f"tiles {tiles:4d}  softmax {ms:.4f} ms ({ms / tiles * 1e3:.2f} us/tile)   max {ms_max:.4f} ms "
          f"({ms_max / tiles * 1e3:.2f} us/tile)   exp-only {e:.4f} ms")
