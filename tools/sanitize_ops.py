"""Every ABI op once on small ragged shapes, in MPC_MODE_BOTH and MPC_MODE_PAIR_LOOPBACK, with
both LTZ circuits -- the workload for compute-sanitizer memcheck / racecheck / synccheck:
  compute-sanitizer --tool memcheck python tools/sanitize_ops.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_19711_b200 as m  # noqa: E402
import workloads  # noqa: E402


def run(mode, circuit):
    c = m.Ctx.for_cfg(workloads.keys(1), mode=mode)
    c.set_ltz_circuit(circuit)
    sh = lambda x: c.share(torch.from_numpy(x.ravel()).cuda())  # noqa: E731
    x = sh(workloads.act_inputs(1000))
    c.open(x)
    c.mul(x, x, off=3, trunc_bits=16)
    c.square(x, trunc_bits=16)
    c.trunc(x, 16)
    c.cmp(x, window=33)
    c.cmp(x, window=64)
    c.relu(x)
    c.exp(x, t=8)
    c.exp(x, t=4, clamp=1, square=1)
    r = sh(workloads.recip_inputs(300))
    c.recip(r)
    c.recip(r, clamp=1)
    c.rsqrt(r, iters=3)
    for form, deg in (("poly_x", 4), ("poly_abs", 4), ("relu", 0), ("erf", 8)):
        kw = dict(form=form, erf_terms=deg) if form == "erf" else dict(form=form, degree=deg)
        c.gelu(x, **kw)
    c.sigmoid(x, form="poly_x", degree=4)
    s = sh(workloads.softmax_inputs(45, 77))
    c.max(s, 45, 77)
    c.softmax(s, 45, 77)
    c.softmax(s, 45, 77, exp_clamp=1, exp_square=1)
    s2 = sh(workloads.softmax_inputs(33, 300))
    c.softmax(s2, 33, 300)
    p = sh(workloads.maxpool_inputs((1, 4, 9, 10)))
    c.maxpool2d(p, 1, 4, 9, 10)
    ln = sh(workloads.layernorm_inputs(40, 96))
    c.layernorm(ln, 40, 96)
    if mode != m.binding.MODE_BOTH:
        c.sync()
    torch.cuda.synchronize()


if __name__ == "__main__":
    for mode in (m.binding.MODE_BOTH, m.binding.MODE_PAIR_LOOPBACK):
        for circuit in (0, 1):
            run(mode, circuit)
    print("sanitize_ops: done")
