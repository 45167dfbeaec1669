"""Timeline of one mpc_softmax_hostio call (MPC_HIO_TRACE=1): per chunk, when its H2D copy, its
compute and its D2H copy start and end -- what bounds the host-buffer e2e number."""
import os, sys
os.environ["MPC_HIO_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19711_b200 as m
import workloads

rows, cols = workloads.SHAPES["cfg2_softmax"]
c = m.Ctx.for_cfg(workloads.keys(2))
x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
# both parties in one pinned [2][n] tensor each way, as bench.py (one 2D DMA per chunk and direction)
hin = torch.empty((2, rows * cols), dtype=torch.uint64).pin_memory()
hout = torch.empty((2, rows * cols), dtype=torch.uint64).pin_memory()
hin[0].copy_(x[0].cpu()); hin[1].copy_(x[1].cpu())
hx, hz = (hin[0], hin[1]), (hout[0], hout[1])
for ch in [int(a) for a in (sys.argv[1:] or ["3072", "1536"])]:
    for rep in range(3):
        print(f"--- chunk {ch} rep {rep}", file=sys.stderr, flush=True)
        c.softmax_hostio(hx, hz, rows, cols, chunk_rows=ch)
        torch.cuda.synchronize()
