"""A/B of the BOTH LayerNorm kernels on cfg5 (8192 x 768, rsqrt 3 iters): MPC_LN_ROW=1 (k_ln_row, one
warp per row) vs 0 (k_ln_fused, row blocks), one process each, L2 flushed between steps; also the
GPT-2 shard (24576 rows) and BERT-base LayerNorm (1024 x 768)."""
import os
import subprocess
import sys

code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2511_19711_b200 as m, workloads
c = m.Ctx.for_cfg(workloads.keys(5))
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
for rows, cols in [(8192, 768), (24576, 768), (1024, 768)]:
    x = c.share(torch.from_numpy(workloads.layernorm_inputs(rows, cols)).cuda())
    z = c._empty(rows * cols)
    out.append(f"ln{rows}x{cols} {t(lambda: c.layernorm(x, rows, cols, out=z)):.4f}")
print("MPC_LN_ROW=" + os.environ.get("MPC_LN_ROW", "1"), " | ".join(out), flush=True)
'''
for rep in range(2):
    for v in ("0", "1"):
        env = dict(os.environ, MPC_LN_ROW=v)
        subprocess.run([sys.executable, "-c", code], env=env, check=True)
