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
hx = tuple(t.cpu().pin_memory() for t in x)
hz = tuple(torch.empty_like(t).pin_memory() for t in hx)
for ch in [int(a) for a in (sys.argv[1:] or ["3072", "1536"])]:
    for rep in range(3):
        print(f"--- chunk {ch} rep {rep}", file=sys.stderr, flush=True)
        c.softmax_hostio(hx, hz, rows, cols, chunk_rows=ch)
        torch.cuda.synchronize()
