"""One PAIR-loopback GELU launch over 2^20 elements (|x|-form deg 4, cfg3 distribution) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19711_b200 as m
import workloads
c = m.Ctx.for_cfg(workloads.keys(3), mode=m.binding.MODE_PAIR_LOOPBACK)
g = c.share(torch.from_numpy(workloads.normal_inputs(1 << 20, 3)).cuda())
for _ in range(2):
    c.gelu(g, form="poly_abs", degree=4)
c.sync()
