"""Time the row max alone on the softmax cfg2 input (BOTH): the max-tree phase of softmax."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19711_b200 as m
import workloads

flush = torch.empty(128 << 20, dtype=torch.int32, device="cuda")
c = m.Ctx.for_cfg(workloads.keys(2))
rows, cols = workloads.SHAPES["cfg2_softmax"]
x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols).ravel()).cuda())
reps = int(os.environ.get("REPS", "20"))
c.max(x, rows, cols); torch.cuda.synchronize()
c.reset_stats()
ts = []
for i in range(reps):
    flush.fill_(i)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); c.max(x, rows, cols); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
ph = c.stats()["philox_calls"] / reps
print(f"max cfg2: median {ts[len(ts)//2]:.4f} ms  {ph / ts[len(ts)//2] / 1e6:.1f} Gphilox/s")
