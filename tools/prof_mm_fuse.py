"""One BERT-base QK^T Beaver matmul (96 x 128x64x128, tensor-core engine, BOTH mode) for ncu
captures of the fused masking / limb-tiling kernels and the GEMM."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19711_b200 as m
import workloads

B, M, K, N = (int(v) for v in (sys.argv[1:] or ["96", "128", "64", "128"]))
c = m.Ctx.for_cfg(workloads.keys(2))
x = c.share(torch.from_numpy(workloads.act_inputs(B * M * K, lo=-2, hi=2)).cuda())
y = c.share(torch.from_numpy(workloads.act_inputs(B * K * N, seed_cfg=5, lo=-2, hi=2)).cuda())
z = c._empty(B * M * N)
for _ in range(2):
    c.matmul(x, y, B, M, K, N, trunc_bits=16, out=z)
torch.cuda.synchronize()
print("done")
