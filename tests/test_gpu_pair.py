"""PAIR mode on one GPU (MPC_MODE_PAIR_LOOPBACK): both parties' kernels run in one launch
and exchange every opening through the same warp-level peer-memory protocol the two-GPU
mode uses.  Cross-mode test T4: PAIR output shares are bit-identical to
MPC_MODE_BOTH's and to the oracle's on the same seeds."""
import numpy as np
import pytest

import workloads
from oracle import Oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def m():
    import paper_2511_19711_b200 as mod
    return mod


def ctxs(m, cfg=1, step=0):
    keys = workloads.keys(cfg)
    b = m.Ctx.for_cfg(keys)
    p = m.Ctx.for_cfg(keys, mode=m.binding.MODE_PAIR_LOOPBACK)
    b.set_step(step)
    p.set_step(step)
    return b, p


def eq(a, b):
    torch.cuda.synchronize()
    return torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_share_open_loopback(m):
    b, p = ctxs(m)
    x = torch.from_numpy(workloads.act_inputs(5000)).cuda()
    sb, sp = b.share(x), p.share(x)
    assert eq(sb, sp)
    rb, fb = b.open(sb)
    rp, fp = p.open(sp)
    p.sync()
    assert torch.equal(rb, rp) and torch.equal(fb, fp)


@pytest.mark.parametrize("n,off", [(1, 0), (777, 3), (100_000, 64)])
def test_mul_loopback(m, n, off):
    b, p = ctxs(m, step=7)
    x = torch.from_numpy(workloads.act_inputs(n)).cuda()
    y = torch.from_numpy(workloads.recip_inputs(n)).cuda()
    xs, ys = b.share(x), b.share(y, owner=1)
    p.set_step(b.step)
    assert eq(b.mul(xs, ys, off=off, trunc_bits=16), p.mul(xs, ys, off=off, trunc_bits=16))
    p.sync()


@pytest.mark.parametrize("w", [1, 13, 33, 34, 64])
def test_cmp_relu_loopback(m, w):
    b, p = ctxs(m, step=3)
    x = b.share(torch.from_numpy(workloads.act_inputs(4096 + 40) * 3).cuda())
    p.set_step(b.step)
    assert eq(b.cmp(x, off=64, window=w), p.cmp(x, off=64, window=w))
    assert eq(b.relu(x, off=0, window=w), p.relu(x, off=0, window=w))
    p.sync()


@pytest.mark.parametrize("t,clamp", [(8, 0), (8, 1), (2, 1), (0, 1)])
def test_exp_loopback(m, t, clamp):
    b, p = ctxs(m)
    x = b.share(torch.from_numpy(workloads.exp_inputs(3000, tail_frac=0.05)).cuda())
    p.set_step(b.step)
    assert eq(b.exp(x, off=32, t=t, clamp=clamp), p.exp(x, off=32, t=t, clamp=clamp))
    p.sync()


@pytest.mark.parametrize("kind,clamp", [("recip", 0), ("recip", 1), ("rsqrt", 0), ("rsqrt", 1)])
def test_newton_loopback(m, kind, clamp):
    b, p = ctxs(m)
    x = b.share(torch.from_numpy(workloads.rsqrt_inputs(2000)).cuda())
    p.set_step(b.step)
    assert eq(getattr(b, kind)(x, off=32, clamp=clamp), getattr(p, kind)(x, off=32, clamp=clamp))
    p.sync()


@pytest.mark.parametrize("act,form,deg", [("gelu", "poly_x", 4), ("gelu", "poly_abs", 4), ("gelu", "erf", 8),
                                          ("silu", "poly_abs", 2), ("sigmoid", "poly_x", 4), ("gelu", "relu", 0)])
def test_act_loopback(m, act, form, deg):
    b, p = ctxs(m)
    x = b.share(torch.from_numpy(workloads.act_inputs(4096 + 99)).cuda())
    p.set_step(b.step)
    kw = dict(form=form, erf_terms=deg) if form == "erf" else dict(form=form, degree=deg)
    assert eq(getattr(b, act)(x, **kw), getattr(p, act)(x, **kw))
    p.sync()


@pytest.mark.parametrize("rows,cols", [(64, 128), (45, 77), (32, 1024)])
def test_softmax_loopback(m, rows, cols):
    b, p = ctxs(m, 2)
    x = b.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
    p.set_step(b.step)
    assert eq(b.softmax(x, rows, cols, row_off=32), p.softmax(x, rows, cols, row_off=32))
    p.sync()


def test_max_pool_ln_loopback(m):
    b, p = ctxs(m, 4)
    x = b.share(torch.from_numpy(workloads.softmax_inputs(70, 9)).cuda())
    p.set_step(b.step)
    assert eq(b.max(x, 70, 9), p.max(x, 70, 9))
    N, C, H, W = 2, 16, 14, 15
    y = b.share(torch.from_numpy(workloads.maxpool_inputs((N, C, H, W))).cuda())
    p.set_step(b.step)
    assert eq(b.maxpool2d(y, N, C, H, W), p.maxpool2d(y, N, C, H, W))
    z = b.share(torch.from_numpy(workloads.layernorm_inputs(70, 768)).cuda())
    p.set_step(b.step)
    assert eq(b.layernorm(z, 70, 768, rsqrt_clamp=1), p.layernorm(z, 70, 768, rsqrt_clamp=1))
    p.sync()


def test_max_pool_cone_loopback(m):
    b, p = ctxs(m, 4)
    b.set_ltz_circuit(1)
    p.set_ltz_circuit(1)
    x = b.share(torch.from_numpy(workloads.softmax_inputs(70, 9)).cuda())
    p.set_step(b.step)
    assert eq(b.max(x, 70, 9), p.max(x, 70, 9))
    N, C, H, W = 2, 16, 14, 15
    y = b.share(torch.from_numpy(workloads.maxpool_inputs((N, C, H, W))).cuda())
    p.set_step(b.step)
    assert eq(b.maxpool2d(y, N, C, H, W), p.maxpool2d(y, N, C, H, W))
    p.sync()


def test_pair_vs_oracle_and_long_sequence(m):
    """Many consecutive ops on one PAIR context: the per-warp round counters persist across
    launches, so no op can read a previous op's stale message."""
    keys = workloads.keys(3)
    p = m.Ctx.for_cfg(keys, mode=m.binding.MODE_PAIR_LOOPBACK)
    o = Oracle.for_cfg(keys)
    n = 2048 + 32
    x = workloads.act_inputs(n)
    sp, so = p.share(torch.from_numpy(x).cuda()), o.share(x)
    for _ in range(3):
        sp = p.gelu(sp, form="poly_abs", degree=4)
        k = m.default_act("gelu", "poly_abs", degree=4)
        so = o.act(so, "gelu", "poly_abs", 4, k["B"], k["coeffs"])
        sp = p.relu(sp)
        so = o.relu(so)
    p.sync()
    assert np.array_equal(sp[0].cpu().numpy(), so[0]) and np.array_equal(sp[1].cpu().numpy(), so[1])


def test_square_ops_loopback(m):
    b, p = ctxs(m, 2)
    x = b.share(torch.from_numpy(workloads.softmax_inputs(64, 128)).cuda())
    p.set_step(b.step)
    assert eq(b.softmax(x, 64, 128, exp_square=1, recip_square=1), p.softmax(x, 64, 128, exp_square=1, recip_square=1))
    assert eq(b.square(x, trunc_bits=16), p.square(x, trunc_bits=16))
    assert eq(b.exp(x, off=0, clamp=1, square=1), p.exp(x, off=0, clamp=1, square=1))
    p.sync()


@pytest.mark.parametrize("w", [17, 21, 33, 40, 64])
def test_cone_loopback(m, w):
    b, p = ctxs(m, 1, step=3)
    b.set_ltz_circuit(1)
    p.set_ltz_circuit(1)
    x = b.share(torch.from_numpy(workloads.act_inputs(4096 * 3 + 40) * 3).cuda())
    p.set_step(b.step)
    assert eq(b.relu(x, off=0, window=w), p.relu(x, off=0, window=w))
    b2, _ = ctxs(m, 1, step=p.step)
    assert eq(b2.cmp(x, off=0, window=w), p.cmp(x, off=0, window=w))
    p.sync()


@pytest.mark.parametrize("form,deg", [("poly_abs", 4), ("poly_x", 2), ("relu", 0)])
def test_cone_act_loopback(m, form, deg):
    b, p = ctxs(m, 1, step=3)
    b.set_ltz_circuit(1)
    p.set_ltz_circuit(1)
    x = b.share(torch.from_numpy(workloads.act_inputs(4096 * 2 + 40)).cuda())
    p.set_step(b.step)
    assert eq(b.gelu(x, form=form, degree=deg), p.gelu(x, form=form, degree=deg))
    p.sync()


@pytest.mark.parametrize("w", [33, 64])
def test_cone_softmax_loopback(m, w):
    b, p = ctxs(m, 2)
    b.set_ltz_circuit(1)
    p.set_ltz_circuit(1)
    x = b.share(torch.from_numpy(workloads.softmax_inputs(96, 128)).cuda())
    p.set_step(b.step)
    assert eq(b.softmax(x, 96, 128, exp_square=1, recip_square=1, window=w),
              p.softmax(x, 96, 128, exp_square=1, recip_square=1, window=w))
    y = b.share(torch.from_numpy(workloads.act_inputs(4096 + 40)).cuda())
    p.set_step(b.step)
    assert eq(b.gelu(y, form="poly_abs", degree=4, window=w), p.gelu(y, form="poly_abs", degree=4, window=w))
    x9 = b.share(torch.from_numpy(workloads.softmax_inputs(70, 9)).cuda())
    p.set_step(b.step)
    assert eq(b.max(x9, 70, 9, window=w), p.max(x9, 70, 9, window=w))
    p.sync()


@pytest.mark.parametrize("reveal_to", [0, 1])
def test_open_to_one_party_loopback(m, reveal_to):
    """mpc_open_to (SURVEY 8(b) reveal_to): only the chosen party learns and writes rec; the
    other party sends its share, the chosen one sends zeros, and the exchange stays in lockstep
    (the next op's shares are still bit-identical to BOTH)."""
    b, p = ctxs(m, step=21)
    x = torch.from_numpy(workloads.act_inputs(5000 + 7)).cuda()
    s = b.share(x)
    rb, fb = b.open(s)
    rp, fp = p.open_to(s, reveal_to)
    p.sync()
    assert torch.equal(rb, rp) and torch.equal(fb, fp)
    p.set_step(b.step)
    assert eq(b.mul(s, s, trunc_bits=16), p.mul(s, s, trunc_bits=16))
    p.sync()
    with pytest.raises(m.MPCError):
        p.open_to(s, 2)


def test_debug_header_no_false_positive_loopback(m):
    """Debug header check in loopback: the same calls on both parties pass and change no shares."""
    b, p = ctxs(m, step=5)
    p.set_debug(True)
    x = b.share(torch.from_numpy(workloads.softmax_inputs(64, 128)).cuda())
    p.set_step(b.step)
    assert eq(b.softmax(x, 64, 128), p.softmax(x, 64, 128))
    assert eq(b.relu(x), p.relu(x))
    p.sync()


# ---- both exchange wire formats: LL (loopback default) and LL63 (PAIR default) ----
@pytest.mark.parametrize("fmt", [0, 1])
def test_exchange_formats_loopback(m, fmt):
    """Every op family in PAIR_LOOPBACK with the given wire format, bit-identical to BOTH (the
    format is transport only, reading R33): varying live-lane patterns (cone), many rounds per
    launch, consecutive launches on persistent per-slot round / tag state."""
    b, p = ctxs(m, 2, step=5)
    p.set_exchange(fmt)
    assert p.exchange == fmt
    x = b.share(torch.from_numpy(workloads.softmax_inputs(96, 128)).cuda())
    p.set_step(b.step)
    assert eq(b.softmax(x, 96, 128), p.softmax(x, 96, 128))
    assert eq(b.softmax(x, 96, 128, causal=1, exp_clamp=1), p.softmax(x, 96, 128, causal=1, exp_clamp=1))
    for circuit in (0, 1):
        b.set_ltz_circuit(circuit)
        p.set_ltz_circuit(circuit)
        for w in (21, 33, 64):
            assert eq(b.relu(x, window=w), p.relu(x, window=w))
        assert eq(b.gelu(x, form="poly_abs", degree=4), p.gelu(x, form="poly_abs", degree=4))
        assert eq(b.softmax(x, 96, 128, exp_square=1, recip_square=1, bcast=1),
                  p.softmax(x, 96, 128, exp_square=1, recip_square=1, bcast=1))
        x9 = b.share(torch.from_numpy(workloads.softmax_inputs(70, 9)).cuda())
        p.set_step(b.step)
        assert eq(b.max(x9, 70, 9), p.max(x9, 70, 9))
    b.set_ltz_circuit(0)
    p.set_ltz_circuit(0)
    y = b.share(torch.from_numpy(workloads.layernorm_inputs(40, 768)).cuda())
    p.set_step(b.step)
    assert eq(b.layernorm(y, 40, 768), p.layernorm(y, 40, 768))
    assert eq(b.layernorm(y, 40, 768, bcast=1), p.layernorm(y, 40, 768, bcast=1))
    assert eq(b.layernorm(y, 40, 768, rsqrt_clamp=1), p.layernorm(y, 40, 768, rsqrt_clamp=1))
    assert eq(b.mul_bcast(y, y, 40, 768, trunc_bits=16), p.mul_bcast(y, y, 40, 768, trunc_bits=16))
    assert eq(b.exp(y, clamp=1, square=1), p.exp(y, clamp=1, square=1))
    assert eq(b.matmul(y, y, 1, 40, 64, 40, trunc_bits=16), p.matmul(y, y, 1, 40, 64, 40, trunc_bits=16))
    assert eq(b.gelu(y, form="erf", erf_terms=8), p.gelu(y, form="erf", erf_terms=8))
    p.sync()


def test_exchange_format_is_fixed_after_first_exchange(m):
    p = m.Ctx.for_cfg(workloads.keys(1), mode=m.binding.MODE_PAIR_LOOPBACK)
    assert p.exchange == 0                      # loopback default: LL
    p.set_exchange(1)
    x = p.share(torch.from_numpy(workloads.act_inputs(64)).cuda())
    p.relu(x)
    with pytest.raises(m.MPCError):
        p.set_exchange(0)
    with pytest.raises(m.MPCError):
        p.set_exchange(2)
    p.sync()
