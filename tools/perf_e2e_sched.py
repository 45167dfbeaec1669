"""A/B of mpc_softmax_hostio chunk schedules on cfg2 (MPC_HIO_SCHED, one process per schedule
because the library reads the variable once)."""
import os, subprocess, sys

SCHEDS = ["3072", "1024,3584,3584,3072,1024", "1536,3584,3584,3584", "1024,2816,2816,2816,2048,768",
          "768,2304,2304,2304,2304,2304", "2048,3584,3584,3072", "1536,3072,3072,3072,1536",
          "1024,3072,3072,3072,2048"]
code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2511_19711_b200 as m, workloads
rows, cols = workloads.SHAPES["cfg2_softmax"]
c = m.Ctx.for_cfg(workloads.keys(2))
x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
hx = tuple(t.cpu().pin_memory() for t in x)
hz = tuple(torch.empty_like(t).pin_memory() for t in hx)
s = torch.cuda.current_stream()
best = []
for trial in range(5):
    for _ in range(3): c.softmax_hostio(hx, hz, rows, cols, chunk_rows=0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(10): c.softmax_hostio(hx, hz, rows, cols, chunk_rows=0)
    b.record(s); torch.cuda.synchronize()
    best.append(a.elapsed_time(b) / 10)
best.sort()
print(f"{os.environ['MPC_HIO_SCHED']:36s} median {best[2]:.4f} ms  min {best[0]:.4f} ms")
'''
for sc in SCHEDS:
    env = dict(os.environ, MPC_HIO_SCHED=sc)
    subprocess.run([sys.executable, "-c", code], env=env, check=True)
