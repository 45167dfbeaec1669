"""Per-kernel device times (mpc_ctx_enable_kernel_timing) of one op on its BASELINE workload:
python tools/ktimes.py [ln|softmax|gelu|...] -- prints each launch's name, ms and Gphilox/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_19711_b200 as m  # noqa: E402
import workloads  # noqa: E402


def main(which):
    c = m.Ctx.for_cfg(workloads.keys(5))
    if which == "ln":
        rows, cols = workloads.SHAPES["cfg5_ln"]
        x = c.share(torch.from_numpy(workloads.layernorm_inputs(rows, cols)).cuda())
        fn = lambda **kw: c.layernorm(x, rows, cols, **kw)   # noqa: E731
    else:
        rows, cols = workloads.SHAPES["cfg2_softmax"]
        x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
        fn = lambda **kw: c.softmax(x, rows, cols, **kw)     # noqa: E731
    for kw in ({}, {"bcast": 1}):
        for _ in range(3):
            fn(**kw)
        torch.cuda.synchronize()
        c.enable_kernel_timing(True)
        c.kernel_times()
        for _ in range(5):
            fn(**kw)
        kt = c.kernel_times()
        c.enable_kernel_timing(False)
        agg = {}
        for name, ms, ph, _u in kt:
            a = agg.setdefault(name, [0.0, 0, 0])
            a[0] += ms; a[1] += ph; a[2] += 1
        print(which, kw, " | ".join(f"{k}: {v[0] / v[2]:.4f} ms {v[1] / v[2] / (v[0] / v[2] / 1e3) / 1e9:.0f} G/s"
                                    for k, v in agg.items()))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "ln")
