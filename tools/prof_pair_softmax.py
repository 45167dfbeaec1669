"""One PAIR-loopback softmax (cfg2) launch for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19711_b200 as m
import workloads
c = m.Ctx.for_cfg(workloads.keys(2), mode=m.binding.MODE_PAIR_LOOPBACK)
rows, cols = workloads.SHAPES["cfg2_softmax"]
x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
for _ in range(2):
    c.softmax(x, rows, cols)
c.sync()
