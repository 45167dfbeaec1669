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
    # round-1b additions: short-row max / MaxPool windows, NEXT #2 (broadcast triple, power basis),
    # NEXT #3 (Beaver matmul, both engines), NEXT #4 (plaintext evaluator), host-buffer softmax
    c.max(s, 45, 9)
    c.maxpool2d(p, 1, 4, 9, 10, k=2, stride=2, pad=0)
    y = sh(workloads.recip_inputs(45))
    c.mul_bcast(s, y, 45, 77, off=1, row_off=3, trunc_bits=16)
    c.softmax(s, 45, 77, bcast=1)
    c.softmax(s, 45, 77, causal=1)                       # causal instantiation
    c.softmax(s, 45, 77, causal=1, bcast=1, exp_clamp=1)
    c.layernorm(ln, 40, 96, bcast=1)
    c.gelu(x, form="poly_abs", degree=4, basis=1)
    c.sigmoid(x, form="poly_x", degree=3, B=4.0, coeffs=[0.5, 0.2, 0.0, -0.01], basis=1)
    a = sh(workloads.act_inputs(2 * 70 * 33))
    b = sh(workloads.act_inputs(2 * 33 * 129, seed_cfg=5))
    # MPC_SAN_TC=0 skips the tensor-core engine (its TMA / tcgen05 async-proxy ordering through
    # mbarriers is not modelled by racecheck / synccheck, which report false hazards there)
    for eng in ((1, 2) if os.environ.get("MPC_SAN_TC", "1") == "1" else (1,)):
        c.set_matmul_engine(eng)
        c.matmul(a, b, 2, 70, 33, 129, batch_off=1, trunc_bits=16)
    if mode == m.binding.MODE_BOTH:
        xd = c.open(s)[1]
        c.plain_eval("softmax", xd, rows=45, cols=77)
        c.plain_eval("softmax", xd, rows=45, cols=77, causal=1)
        c.plain_eval("gelu", c.open(x)[1], form="poly_abs", degree=4)
        c.plain_eval("layernorm", c.open(ln)[1], rows=40, cols=96)
    hx = tuple(t.cpu().pin_memory() for t in s)
    hz = tuple(torch.empty_like(t).pin_memory() for t in hx)
    c.softmax_hostio(hx, hz, 45, 77, chunk_rows=32)
    if mode != m.binding.MODE_BOTH:
        # round 2: the trusted dealer's stream -- the dealer's pass (stream role,
        # writes) and party 1 reading it (stream role, loads) over the same op sequence
        d = m.Ctx.dealer(workloads.keys(1), target=mode)
        d.set_ltz_circuit(circuit)
        def seq(cc, xx, ss, lnn, aa, bb):
            cc.mul(xx, xx, trunc_bits=16)
            cc.relu(xx)
            cc.gelu(xx, form="poly_abs", degree=4)
            cc.softmax(ss, 45, 77)
            cc.layernorm(lnn, 40, 96)
            cc.matmul(aa, bb, 2, 70, 33, 129, trunc_bits=16)
        d.set_step(c.step)
        like = m.Ctx.like
        seq(d, like(1000), like(45 * 77), like(40 * 96), like(2 * 70 * 33), like(2 * 33 * 129))
        c.set_corrections(d.dealer_stream())
        seq(c, x, s, ln, a, b)
        c.sync()
        c.set_corrections(None)
        c.sync()
    torch.cuda.synchronize()


if __name__ == "__main__":
    for mode in (m.binding.MODE_BOTH, m.binding.MODE_PAIR_LOOPBACK):
        for circuit in (0, 1):
            run(mode, circuit)
    print("sanitize_ops: done")
