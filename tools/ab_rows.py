"""Softmax (cols 128) at several row counts and the host-buffer e2e, MPC_SOFTMAX_BAL=1 vs 2 (one
process each), L2 flushed between steps."""
import os
import subprocess
import sys

code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2511_19711_b200 as m, workloads
c = m.Ctx.for_cfg(workloads.keys(2))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); fn(); b.record(s)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps
out = []
for rows in (512, 1024, 3072, 4096, 8192, 12288):
    x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, 128)).cuda())
    z = c._empty(rows * 128)
    out.append(f"{rows}: {t(lambda: c.softmax(x, rows, 128, out=z)):.4f}")
rows = 12288
hx = torch.from_numpy(workloads.softmax_inputs(rows, 128))
g = c.share(hx.cuda())
hs = torch.empty((2, rows * 128), dtype=torch.uint64).pin_memory()
hs[0].copy_(g[0].cpu()); hs[1].copy_(g[1].cpu())
hz = torch.empty((2, rows * 128), dtype=torch.uint64).pin_memory()
def hio():
    c.softmax_hostio((hs[0], hs[1]), (hz[0], hz[1]), rows, 128, chunk_rows=3072)
out.append(f"hostio {t(hio):.4f}")
print("MPC_SOFTMAX_BAL=" + os.environ.get("MPC_SOFTMAX_BAL", "1"), " | ".join(out), flush=True)
'''
for rep in range(2):
    for v in ("2",):
        subprocess.run([sys.executable, "-c", code], env=dict(os.environ, MPC_SOFTMAX_BAL=v), check=True)
