"""Run each hot op once on its BASELINE workload (after one warm-up call) so that
`ncu -k regex:<kernel>` can capture it.  Usage: python tools/prof_ops.py [softmax gelu relu ln sm1024]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_19711_b200 as m  # noqa: E402
import workloads  # noqa: E402


def main(which):
    ctx = m.Ctx.for_cfg(workloads.keys(2))
    dev = torch.device("cuda", 0)
    if "softmax" in which:
        rows, cols = workloads.SHAPES["cfg2_softmax"]
        x = ctx.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).to(dev))
        for _ in range(2):
            ctx.softmax(x, rows, cols)
    if "sm1024" in which:
        rows, cols = 8 * 12 * 128, 1024      # 1/8 of the GPT-2 layer (cfg5)
        x = ctx.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).to(dev))
        for _ in range(2):
            ctx.softmax(x, rows, cols)
    if "gelu" in which:
        n = workloads.SHAPES["cfg3_gelu"]
        x = ctx.share(torch.from_numpy(workloads.normal_inputs(n, 3)).to(dev))
        for _ in range(2):
            ctx.gelu(x, form="poly_abs", degree=4)
    if "relu" in which:
        n = 32 * 64 * 112 * 112 // 4
        x = ctx.share(torch.from_numpy(workloads.relu_inputs(n)).to(dev))
        for _ in range(2):
            ctx.relu(x)
    if "maxpool" in which:
        N, C, H, W = 8, 64, 112, 112          # one pair's shard of the cfg4 MaxPool input
        x = ctx.share(torch.from_numpy(workloads.maxpool_inputs((N, C, H, W))).to(dev))
        for _ in range(2):
            ctx.maxpool2d(x, N, C, H, W, 3, 2, 1)
    if "matmul" in which:
        B, M, K, N = 1, 1024, 768, 3072        # BERT-base FFN Linear, tensor-core engine
        x = ctx.share(torch.from_numpy(workloads.act_inputs(B * M * K, lo=-2, hi=2)).to(dev))
        y = ctx.share(torch.from_numpy(workloads.act_inputs(B * K * N, seed_cfg=5, lo=-2, hi=2)).to(dev))
        ctx.set_matmul_engine(2)
        for _ in range(2):
            ctx.matmul(x, y, B, M, K, N, trunc_bits=16)
    if "ln" in which:
        rows, cols = workloads.SHAPES["cfg5_ln"]
        x = ctx.share(torch.from_numpy(workloads.layernorm_inputs(rows, cols)).to(dev))
        for _ in range(2):
            ctx.layernorm(x, rows, cols)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1:] or ["softmax", "gelu", "relu", "ln"])
