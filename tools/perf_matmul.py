"""Beaver matmul timing: SIMT vs tensor-core engine on BERT-base shapes (cfg2 attention
QK^T and AV over 96 heads, the FFN Linear 1024 x 768 x 3072)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19711_b200 as m
import workloads

flush = torch.empty(128 << 20, dtype=torch.int32, device="cuda")


def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    tot = 0.0
    for i in range(reps):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps


c = m.Ctx.for_cfg(workloads.keys(2))
c.enable_kernel_timing(True)
for name, (B, M, K, N) in {"qk^T 96x128x64x128": (96, 128, 64, 128), "av 96x128x128x64": (96, 128, 128, 64),
                           "ffn 1024x768x3072": (1, 1024, 768, 3072), "ffn2 1024x3072x768": (1, 1024, 3072, 768)}.items():
    x = c.share(torch.from_numpy(workloads.act_inputs(B * M * K, lo=-2, hi=2)).cuda())
    y = c.share(torch.from_numpy(workloads.act_inputs(B * K * N, seed_cfg=5, lo=-2, hi=2)).cuda())
    z = c._empty(B * M * N)
    row = [name]
    for eng in (1, 2):
        c.set_matmul_engine(eng)
        c.kernel_times()
        ms = t(lambda: c.matmul(x, y, B, M, K, N, trunc_bits=16, out=z))
        kt = c.kernel_times()
        agg = {}
        for nm, kms, _ph, _u in kt:
            agg[nm] = agg.get(nm, 0.0) + kms
        reps = 11
        macs = B * M * K * N
        gemm = agg.get("matmul_tc", agg.get("matmul", 0.0)) / reps
        i8 = 36 * 5 * macs                                  # int8 MACs of both parties' limb GEMMs
        row.append(f"eng{eng}: {ms:.4f} ms ({macs / ms / 1e9:.2f} T ring-MAC/s; gemm kernel {gemm:.4f} ms"
                   + (f", {2 * i8 / gemm / 1e9:.0f} int8 TOPS" if eng == 2 else
                      f", {5 * macs / gemm / 1e9:.2f} T u64-MAC/s") + "; "
                   + ", ".join(f"{k} {v / reps:.4f}" for k, v in agg.items()) + ")")
    print(" | ".join(row))
