"""Host-buffer softmax (cfg2) e2e per step under explicit chunk schedules (MPC_HIO_SCHED, chunk_rows=0)
and pipeline slot counts (MPC_HIO_SLOTS), one process per setting, L2 flushed between steps."""
import os
import subprocess
import sys

code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2511_19711_b200 as m, workloads
c = m.Ctx.for_cfg(workloads.keys(2))
rows = 12288
g = c.share(torch.from_numpy(workloads.softmax_inputs(rows, 128)).cuda())
hs = torch.empty((2, rows * 128), dtype=torch.uint64).pin_memory()
hs[0].copy_(g[0].cpu()); hs[1].copy_(g[1].cpu())
hz = torch.empty((2, rows * 128), dtype=torch.uint64).pin_memory()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
def hio():
    c.softmax_hostio((hs[0], hs[1]), (hz[0], hz[1]), rows, 128, chunk_rows=0)
for _ in range(3): hio()
torch.cuda.synchronize()
tot = []
for _ in range(30):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); hio(); b.record(s)
    torch.cuda.synchronize()
    tot.append(a.elapsed_time(b))
tot.sort()
print(f"{os.environ.get('MPC_HIO_SCHED')} slots={os.environ.get('MPC_HIO_SLOTS', '4')}: mean {sum(tot)/len(tot):.4f} median {tot[len(tot)//2]:.4f}", flush=True)
'''
S = ["1536", "1024", "2048", "768,1536,1536,1536,1536,1536,1536,1536,768", "512,1024,1536,1536,1536,1536,1536,1536,1024,512",
     "384,768,1536,1536,1536,1536,1536,1536,1152,768,384"]
for rep in range(2):
    for sch in S:
        for slots in ("4", "8"):
            subprocess.run([sys.executable, "-c", code], env=dict(os.environ, MPC_HIO_SCHED=sch, MPC_HIO_SLOTS=slots), check=True)
