"""Time softmax cfg2 only (BOTH) for A/B builds: MPC200_LIB=<so> python tools/perf_softmax.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19711_b200 as m
import workloads

flush = torch.empty(128 << 20, dtype=torch.int32, device="cuda")
c = m.Ctx.for_cfg(workloads.keys(2))
rows, cols = workloads.SHAPES["cfg2_softmax"]
x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols).ravel()).cuda())
c.softmax(x, rows, cols); torch.cuda.synchronize()
ts = []
for i in range(20):
    flush.fill_(i)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); c.softmax(x, rows, cols); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
print(f"{os.path.basename(os.environ.get('MPC200_LIB', 'default'))}: median {ts[10]:.4f} ms  min {ts[0]:.4f}")
