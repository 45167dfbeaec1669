"""Profiling driver: the cfg2 row max tree alone (k_max), a few calls -- for ncu -k regex:k_max."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_19711_b200 as m  # noqa: E402
import workloads  # noqa: E402

c = m.Ctx.for_cfg(workloads.keys(2))
rows, cols = workloads.SHAPES["cfg2_softmax"]
x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
mx = c._empty(rows)
for _ in range(4):
    c.max(x, rows, cols, out=mx)
torch.cuda.synchronize()
print("done")
