"""Seeded randomized parity sweep: every op of include/mpc200.h with random shapes, global
offsets, step ids and knobs (DESIGN.md 2 contract), GPU shares vs the oracle bit-exact.

Each case draws its parameters from a counter-seeded numpy Generator, so a failure names
the case id that reproduces it.  The fixed-parameter tests (test_gpu_parity.py, ...) pin the
known edge cases; this sweep covers the combinations between them: ragged sizes, odd row
lengths, large step ids, LTZ circuit (Kogge-Stone / cone), protocol variants (square pairs,
broadcast triple, power basis), matmul engines, and a share of the cases in PAIR_LOOPBACK (half of
those with party 1 reading the trusted dealer's correction stream).
"""
import os

import numpy as np
import pytest

import workloads
from oracle import Oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

# MPC_FUZZ_CASES / MPC_FUZZ_SEED widen the sweep for long runs (default: 512 cases, seed 0x5eed)
N_CASES = int(os.environ.get("MPC_FUZZ_CASES", "512"))
SEED = int(os.environ.get("MPC_FUZZ_SEED", str(0x5eed)), 0)


@pytest.fixture(scope="module")
def m():
    import paper_2511_19711_b200 as mod
    return mod


def _same(g, o, what):
    a0, a1 = g[0].cpu().numpy(), g[1].cpu().numpy()
    bad = np.nonzero((a0 != o[0]) | (a1 != o[1]))[0]
    assert bad.size == 0, f"{what}: {bad.size} mismatching shares, first at {bad[:5]}"


def _exp_knobs(r):
    return dict(t=int(r.integers(0, 9)), clamp=int(r.integers(0, 2)), window=int(r.choice([17, 25, 33, 40, 64])),
                square=int(r.integers(0, 2)))


def _case(r, m):
    """-> (name, kwargs for the GPU call, callable(ctx) -> shares, callable(oracle) -> shares, x)."""
    op = r.choice(["mul", "square", "mul_bcast", "trunc", "cmp", "relu", "exp", "recip", "rsqrt", "act",
                   "max", "maxpool", "softmax", "layernorm", "matmul"])
    a32 = 32 * int(r.integers(0, 1 << 20))            # comparison ops: 32-aligned global offsets
    anyoff = int(r.integers(0, 1 << 30))
    if op in ("mul", "square", "trunc"):
        n = int(r.integers(1, 6000))
        x = workloads.act_inputs(n, seed_cfg=int(r.integers(1, 9)), lo=-50, hi=50)
        y = workloads.recip_inputs(n, seed_cfg=int(r.integers(1, 9)))
        tb = int(r.choice([0, 16]))
        if op == "mul":
            return op, [x, y], lambda c, s: c.mul(s[0], s[1], off=anyoff, trunc_bits=tb), \
                lambda o, s: o.mul(s[0], s[1], off=anyoff, trunc_bits=tb)
        if op == "square":
            return op, [x], lambda c, s: c.square(s[0], off=anyoff, trunc_bits=tb), \
                lambda o, s: o.square(s[0], off=anyoff, trunc_bits=tb)
        bits = int(r.integers(1, 33))
        return op, [x], lambda c, s: c.trunc(s[0], bits), lambda o, s: Oracle.trunc(s[0], bits)
    if op == "mul_bcast":
        rows, cols = int(r.integers(1, 60)), int(r.integers(1, 300))
        x = workloads.act_inputs(rows * cols, seed_cfg=3)
        y = workloads.recip_inputs(rows, seed_cfg=4)
        off, roff, tb = 2 * int(r.integers(0, 1 << 20)), int(r.integers(0, 1 << 20)), int(r.choice([0, 16]))
        return op, [x, y], lambda c, s: c.mul_bcast(s[0], s[1], rows, cols, off=off, row_off=roff, trunc_bits=tb), \
            lambda o, s: o.mul_bcast(s[0], s[1], rows, cols, off=off, row_off=roff, trunc_bits=tb)
    if op in ("cmp", "relu"):
        n = int(r.integers(1, 6000))
        w = int(r.integers(1, 65))
        x = workloads.act_inputs(n, seed_cfg=int(r.integers(1, 9)), lo=-8, hi=8)
        if w < 21:   # keep rec(x) inside the window so the result is also the true sign
            x = x / 64.0
        return op, [x], lambda c, s: getattr(c, op)(s[0], off=a32, window=w), \
            lambda o, s: (o.ltz if op == "cmp" else o.relu)(s[0], off=a32, window=w)
    if op == "exp":
        n = int(r.integers(1, 6000))
        k = _exp_knobs(r)
        x = workloads.exp_inputs(n, seed_cfg=int(r.integers(1, 9)), tail_frac=0.2)
        return op, [x], lambda c, s: c.exp(s[0], off=a32, **k), lambda o, s: o.exp(s[0], off=a32, **k)
    if op in ("recip", "rsqrt"):
        n = int(r.integers(1, 6000))
        k = _exp_knobs(r)
        iters = int(r.integers(1, 13))
        x = (workloads.recip_inputs if op == "recip" else workloads.rsqrt_inputs)(n, seed_cfg=int(r.integers(1, 9)))
        return op, [x], lambda c, s: getattr(c, op)(s[0], off=a32, iters=iters, **k), \
            lambda o, s: getattr(o, op)(s[0], off=a32, iters=iters, **k)
    if op == "act":
        act = str(r.choice(["gelu", "silu", "sigmoid"]))
        forms = {"gelu": ["poly_x", "poly_abs", "relu", "erf"], "silu": ["poly_x", "poly_abs", "relu"],
                 "sigmoid": ["poly_x", "relu"]}[act]
        form = str(r.choice(forms))
        w = int(r.choice([20, 25, 33, 48, 64]))
        n = int(r.integers(1, 6000))
        x = workloads.act_inputs(n, seed_cfg=int(r.integers(1, 9)))
        if form == "erf":
            K = int(r.integers(2, 13))
            kn = m.default_act(act, "erf", erf_terms=K, window=w)
            return f"{act}/erf{K}", [x], lambda c, s: getattr(c, act)(s[0], off=a32, **kn), \
                lambda o, s: o.act(s[0], act, "erf", 1, kn["B"], None, K, off=a32, window=w)
        if form == "relu":
            kn = m.default_act(act, "relu", window=w)
            return f"{act}/relu", [x], lambda c, s: getattr(c, act)(s[0], off=a32, **kn), \
                lambda o, s: o.act(s[0], act, "relu", 0, kn["B"], None, off=a32, window=w)
        deg = int(r.integers(1, 5))
        B = float(r.choice([2.0, 3.0, 5.0]))
        coeffs = [float(v) for v in r.normal(0.0, 0.5, deg + 1)]
        basis = int(r.integers(0, 2))
        kn = dict(form=form, degree=deg, B=B, coeffs=coeffs, erf_terms=0, window=w, basis=basis)
        return f"{act}/{form}{deg}/b{basis}", [x], lambda c, s: getattr(c, act)(s[0], off=a32, **kn), \
            lambda o, s: o.act(s[0], act, form, deg, B, coeffs, off=a32, window=w, basis=basis)
    if op == "max":
        rows, cols = int(r.integers(1, 80)), int(r.integers(1, 300))
        w = int(r.choice([20, 33, 40, 64]))
        x = workloads.softmax_inputs(rows, cols, seed_cfg=int(r.integers(1, 9)))
        return op, [x], lambda c, s: c.max(s[0], rows, cols, row_off=a32, window=w), \
            lambda o, s: o.max(s[0], rows, cols, row_off=a32, window=w)
    if op == "maxpool":
        N, C = int(r.integers(1, 3)), int(r.integers(1, 5))
        k = int(r.integers(1, 5))
        stride, pad = int(r.integers(1, 4)), int(r.integers(0, k // 2 + 1))
        H, W = int(r.integers(k, 21)), int(r.integers(k, 21))
        img = 32 * int(r.integers(0, 1 << 12))   # img_off * C*Ho*Wo must be 32-aligned (comparison groups)
        x = workloads.maxpool_inputs((N, C, H, W), seed_cfg=int(r.integers(1, 9)))
        return f"maxpool k{k}s{stride}p{pad}", [x], \
            lambda c, s: c.maxpool2d(s[0], N, C, H, W, k, stride, pad, img_off=img), \
            lambda o, s: o.maxpool2d(s[0], N, C, H, W, k, stride, pad, img_off=img)
    if op == "softmax":
        rows, cols = int(r.integers(1, 80)), int(r.integers(1, 300))
        e, q = _exp_knobs(r), _exp_knobs(r)
        kw = dict(window=int(r.choice([25, 33, 40])), exp_t=e["t"], exp_clamp=e["clamp"], exp_window=e["window"],
                  exp_square=e["square"], recip_iters=int(r.integers(1, 13)), recip_t=q["t"],
                  recip_clamp=q["clamp"], recip_window=q["window"], recip_square=q["square"],
                  bcast=int(r.integers(0, 2)), causal=int(r.integers(0, 2)))
        x = workloads.softmax_inputs(rows, cols, seed_cfg=int(r.integers(1, 9)))
        return op, [x], lambda c, s: c.softmax(s[0], rows, cols, row_off=a32, **kw), \
            lambda o, s: o.softmax(s[0], rows, cols, row_off=a32, **kw)
    if op == "layernorm":
        rows, cols = int(r.integers(1, 64)), int(r.integers(2, 800))
        q = _exp_knobs(r)
        kw = dict(mean_mode=int(r.integers(0, 2)), rsqrt_iters=int(r.integers(1, 6)), rsqrt_t=q["t"],
                  rsqrt_clamp=q["clamp"], rsqrt_window=q["window"], rsqrt_square=q["square"],
                  bcast=int(r.integers(0, 2)))
        x = workloads.layernorm_inputs(rows, cols, seed_cfg=int(r.integers(1, 9)))
        return op, [x], lambda c, s: c.layernorm(s[0], rows, cols, row_off=a32, **kw), \
            lambda o, s: o.layernorm(s[0], rows, cols, row_off=a32, **kw)
    # matmul
    batch, M, K, N = int(r.integers(1, 4)), int(r.integers(1, 150)), int(r.integers(1, 150)), int(r.integers(1, 150))
    boff, tb = int(r.integers(0, 1 << 16)), int(r.choice([0, 16]))
    x = workloads.act_inputs(batch * M * K, seed_cfg=5, lo=-2, hi=2)
    y = workloads.act_inputs(batch * K * N, seed_cfg=6, lo=-2, hi=2)
    return f"matmul {batch}x{M}x{K}x{N}", [x, y], \
        lambda c, s: c.matmul(s[0], s[1], batch, M, K, N, batch_off=boff, trunc_bits=tb), \
        lambda o, s: o.matmul(s[0], s[1], batch, M, K, N, batch_off=boff, trunc_bits=tb)


@pytest.mark.parametrize("case", range(N_CASES))
def test_fuzz_case(m, case):
    r = np.random.default_rng([SEED, case])
    name, xs, gpu_call, orc_call = _case(r, m)
    keys = workloads.keys(int(r.integers(1, 6)))
    step = int(r.integers(0, 1 << 24))
    loopback = case % 4 == 3
    dealer = loopback and case % 8 == 7          # half the loopback cases: party 1 reads the dealer's stream
    c = m.Ctx.for_cfg(keys, mode=m.binding.MODE_PAIR_LOOPBACK) if loopback else m.Ctx.for_cfg(keys)
    circuit, engine = int(r.integers(0, 2)), int(r.integers(0, 3))
    c.set_ltz_circuit(circuit)
    c.set_matmul_engine(engine)
    o = Oracle.for_cfg(keys, step)
    # input sharing through the oracle: both sides start from the same shares
    osh = [o.share(x, owner=int(r.integers(0, 2)), off=int(r.integers(0, 1 << 20))) for x in xs]
    gsh = [tuple(torch.from_numpy(np.ascontiguousarray(p)).cuda() for p in s) for s in osh]
    c.set_step(o.step)
    if dealer:                                   # the dealer's offline pass first
        d = m.Ctx.dealer(keys, target=m.binding.MODE_PAIR_LOOPBACK)
        d.set_ltz_circuit(circuit)
        d.set_matmul_engine(engine)
        d.set_step(o.step)
        gpu_call(d, [m.Ctx.like(len(s[0])) for s in osh])
        c.set_corrections(d.dealer_stream())
    g = gpu_call(c, gsh)
    c.sync()
    if dealer:
        # (an op with no PAIR launch, e.g. trunc, leaves an empty stream: set_corrections then clears)
        assert c.corrections_left() in (0, -1), f"case {case} ({name}): dealer stream not consumed"
    ref = orc_call(o, osh)
    _same(g, ref, f"case {case} ({name}, {'loopback + dealer' if dealer else 'loopback' if loopback else 'both'})")
    assert c.step == o.step, f"case {case} ({name}): step {c.step} != oracle {o.step}"
