"""Host-buffer softmax (cfg2) e2e per step: chunk sizes x MPC_SOFTMAX_BAL modes for the chunks' kernels
(1: 32-row tiles, 2: balanced on all CTAs, 3: balanced on one CTA per SM), one process per mode."""
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
out = []
for ch in (1536, 2048, 3072, 4096):
    def hio():
        c.softmax_hostio((hs[0], hs[1]), (hz[0], hz[1]), rows, 128, chunk_rows=ch)
    for _ in range(3): hio()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(20):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); hio(); b.record(s)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    out.append(f"chunk{ch} {tot / 20:.4f}")
print("MPC_SOFTMAX_BAL=" + os.environ.get("MPC_SOFTMAX_BAL", "default"), " | ".join(out), flush=True)
'''
for rep in range(2):
    for v in ("1", "2", "3"):
        subprocess.run([sys.executable, "-c", code], env=dict(os.environ, MPC_SOFTMAX_BAL=v), check=True)
