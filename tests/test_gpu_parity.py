"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact on every
uint64 share of both parties, on seeded inputs (DESIGN.md section 2 contract).

Small cases span several warps/tiles and a ragged tail; full BASELINE sizes compare EVERY share
against the whole-array oracle run on all host cores (tests/oracle_pool.py: 32-aligned slices
with global offsets reproduce the unsharded op exactly, the PRG being keyed by global unit).
"""
import numpy as np
import pytest

import workloads
from oracle import Oracle
from oracle import float_ref as fr

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def mpc():
    import paper_2511_19711_b200 as m
    return m


def np_(t):
    return t.cpu().numpy()


def gpu_pair(s):
    return (torch.from_numpy(np.ascontiguousarray(s[0])).cuda(), torch.from_numpy(np.ascontiguousarray(s[1])).cuda())


def same(g, o):
    a0, a1 = np_(g[0]), np_(g[1])
    assert a0.shape == o[0].shape
    bad = np.nonzero((a0 != o[0]) | (a1 != o[1]))[0]
    assert bad.size == 0, f"{bad.size} mismatching shares, first at {bad[:5]}"


def pair_ctx(mpc, cfg=1, step=0):
    keys = workloads.keys(cfg)
    c = mpc.Ctx.for_cfg(keys)
    c.set_step(step)
    return c, Oracle.for_cfg(keys, step)


# ----------------------------------------------------------------- PRG ----
@pytest.mark.parametrize("ctr,key,out", [
    ((0, 0, 0, 0), 0, (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff,) * 4, 0xffffffffffffffff, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), 0x299f31d0a4093822,
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
])
def test_device_philox_kat(mpc, ctr, key, out):
    c, _ = pair_ctx(mpc)
    unit0 = ctr[0] | (ctr[1] << 32)
    w = c.prg_fill(key, unit0, ctr[2], ctr[3], 1)
    torch.cuda.synchronize()
    got = tuple(int(v) & 0xffffffff for v in w.cpu().tolist())
    assert got == out


# ------------------------------------------------------------ share/open ----
@pytest.mark.parametrize("n", [1, 31, 33, 4113, 100_003])
@pytest.mark.parametrize("owner", [0, 1])
def test_share_open(mpc, n, owner):
    c, o = pair_ctx(mpc, step=5)
    x = workloads.act_inputs(n) * 1000
    g = c.share(torch.from_numpy(x).cuda(), owner=owner, off=7)
    r = o.share(x, owner=owner, off=7)
    same(g, r)
    x32 = x.astype(np.float32)
    g32 = c.share(torch.from_numpy(x32).cuda(), owner=owner, off=7)
    same(g32, o.share(x32.astype(np.float64), owner=owner, off=7))
    ring, f = c.open(g)
    oring, of = Oracle.open(*r)
    assert np.array_equal(np_(ring), oring) and np.array_equal(np_(f), of)
    assert c.step == o.step


# ------------------------------------------------------------- mul/trunc ----
@pytest.mark.parametrize("n,off", [(1, 0), (2, 1), (257, 3), (4096, 64), (100_001, 12345)])
@pytest.mark.parametrize("tb", [0, 16])
def test_mul(mpc, n, off, tb):
    c, o = pair_ctx(mpc, step=11)
    x = workloads.act_inputs(n)
    y = workloads.recip_inputs(n)
    gx, gy = c.share(torch.from_numpy(x).cuda()), c.share(torch.from_numpy(y).cuda(), owner=1)
    ox, oy = o.share(x), o.share(y, owner=1)
    same(c.mul(gx, gy, off=off, trunc_bits=tb), o.mul(ox, oy, off=off, trunc_bits=tb))
    same(c.trunc(gx, 16), Oracle.trunc(ox, 16))
    same(c.trunc(gy, 5), Oracle.trunc(oy, 5))


# --------------------------------------------------------------- cmp/relu ----
@pytest.mark.parametrize("w", [1, 2, 13, 33, 34, 63, 64])
def test_cmp_windows(mpc, w):
    c, o = pair_ctx(mpc, step=3)
    n = 1000
    x = workloads.act_inputs(n) * 3
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.cmp(gx, off=64, window=w), o.ltz(ox, off=64, window=w))


@pytest.mark.parametrize("n", [1, 32, 45, 4096 + 7, 65536])
def test_relu_and_cmp(mpc, n):
    c, o = pair_ctx(mpc, step=9)
    x = workloads.relu_inputs(n)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.cmp(gx, off=32), o.ltz(ox, off=32))
    same(c.relu(gx, off=0), o.relu(ox, off=0))
    assert c.step == o.step


# ------------------------------------------------------------- exp/recip ----
@pytest.mark.parametrize("t,clamp", [(8, 0), (8, 1), (4, 0), (2, 1), (0, 1), (1, 0), (0, 0)])
def test_exp(mpc, t, clamp):
    c, o = pair_ctx(mpc, step=2)
    n = 4096 + 13
    x = workloads.exp_inputs(n, tail_frac=0.05)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.exp(gx, off=96, t=t, clamp=clamp), o.exp(ox, off=96, t=t, clamp=clamp))
    assert c.step == o.step


@pytest.mark.parametrize("t", [8, 2, 0])
def test_exp_clamp_large(mpc, t):
    """n >= 2^16 runs the clamp head and the squarings as two launches (pair layout)."""
    c, o = pair_ctx(mpc, step=6)
    n = 70_000 + 5
    x = workloads.exp_inputs(n, tail_frac=0.05)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.exp(gx, off=32, t=t, clamp=1), o.exp(ox, off=32, t=t, clamp=1))
    assert c.step == o.step


@pytest.mark.parametrize("iters,t,clamp", [(10, 8, 0), (3, 8, 1), (7, 4, 0)])
def test_recip(mpc, iters, t, clamp):
    c, o = pair_ctx(mpc, step=2)
    n = 3000
    x = workloads.recip_inputs(n)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.recip(gx, off=32, iters=iters, t=t, clamp=clamp), o.recip(ox, off=32, iters=iters, t=t, clamp=clamp))


@pytest.mark.parametrize("iters,t,clamp", [(3, 8, 0), (10, 8, 1), (3, 0, 0)])
def test_rsqrt(mpc, iters, t, clamp):
    c, o = pair_ctx(mpc, step=2)
    n = 3000
    x = workloads.rsqrt_inputs(n)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.rsqrt(gx, off=32, iters=iters, t=t, clamp=clamp), o.rsqrt(ox, off=32, iters=iters, t=t, clamp=clamp))


# ------------------------------------------------------------ activations ----
ACTS = [("gelu", "poly_x", 4), ("gelu", "poly_x", 2), ("gelu", "poly_abs", 4), ("gelu", "poly_abs", 2),
        ("gelu", "relu", 0), ("gelu", "erf", 8), ("gelu", "erf", 4), ("silu", "poly_x", 4),
        ("silu", "poly_abs", 4), ("silu", "relu", 0), ("sigmoid", "poly_x", 4), ("sigmoid", "poly_x", 2),
        ("sigmoid", "relu", 0)]


@pytest.mark.parametrize("act,form,deg", ACTS)
def test_activations(mpc, act, form, deg):
    c, o = pair_ctx(mpc, step=4)
    n = 4096 + 99
    x = workloads.act_inputs(n)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    if form == "erf":
        knobs = mpc.default_act(act, "erf", erf_terms=deg)
        g = getattr(c, act)(gx, off=0, form="erf", erf_terms=deg)
        r = o.act(ox, act, "erf", 1, knobs["B"], None, deg)
    else:
        knobs = mpc.default_act(act, form, degree=deg)
        g = getattr(c, act)(gx, off=0, form=form, degree=deg)
        r = o.act(ox, act, form, knobs["degree"], knobs["B"], knobs["coeffs"] or [0.0])
    same(g, r)
    assert c.step == o.step


# -------------------------------------------------------------- row ops ----
@pytest.mark.parametrize("rows,cols", [(64, 1), (64, 2), (33, 3), (40, 9), (96, 128), (7, 200)])
def test_max(mpc, rows, cols):
    c, o = pair_ctx(mpc, 2, step=1)
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.max(gx, rows, cols, row_off=32), o.max(ox, rows, cols, row_off=32))
    assert c.step == o.step


@pytest.mark.parametrize("cols", [4, 5, 7, 16, 17])
@pytest.mark.parametrize("w", [33, 64])
def test_max_short_rows(mpc, cols, w):
    """cols <= 16 runs the warp-per-tile kernel, 17 the CTA-per-tile one: same contract."""
    c, o = pair_ctx(mpc, 2, step=3)
    rows = 200
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.max(gx, rows, cols, row_off=64, window=w), o.max(ox, rows, cols, row_off=64, window=w))
    assert c.step == o.step


@pytest.mark.parametrize("k,stride,pad", [(2, 2, 0), (3, 1, 1), (4, 2, 1)])
def test_maxpool_windows(mpc, k, stride, pad):
    N, C, H, W = 3, 8, 13, 12
    c, o = pair_ctx(mpc, 4, step=2)
    x = workloads.maxpool_inputs((N, C, H, W)) - 0.25
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    Ho, Wo = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
    img_off = 4 if (C * Ho * Wo * 4) % 32 == 0 else 0
    same(c.maxpool2d(gx, N, C, H, W, k, stride, pad, img_off=img_off),
         o.maxpool2d(ox, N, C, H, W, k, stride, pad, img_off=img_off))


def test_maxpool(mpc):
    N, C, H, W = 2, 16, 14, 15
    c, o = pair_ctx(mpc, 4, step=1)
    x = workloads.maxpool_inputs((N, C, H, W)) - 0.25
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.maxpool2d(gx, N, C, H, W, 3, 2, 1, img_off=2), o.maxpool2d(ox, N, C, H, W, 3, 2, 1, img_off=2))


@pytest.mark.parametrize("rows,cols,clamp", [(64, 128, 0), (32, 1024, 0), (45, 77, 1), (96, 128, 1)])
def test_softmax(mpc, rows, cols, clamp):
    c, o = pair_ctx(mpc, 2, step=1)
    x = workloads.softmax_inputs(rows, cols, spike=bool(clamp))
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    kw = dict(exp_clamp=clamp, recip_clamp=clamp)
    same(c.softmax(gx, rows, cols, row_off=64, **kw), o.softmax(ox, rows, cols, row_off=64, **kw))
    assert c.step == o.step


@pytest.mark.parametrize("mean_mode,iters,clamp", [(0, 3, 0), (1, 3, 1), (1, 10, 0)])
def test_layernorm(mpc, mean_mode, iters, clamp):
    rows, cols = 70, 768
    c, o = pair_ctx(mpc, 5, step=1)
    x = workloads.layernorm_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    kw = dict(mean_mode=mean_mode, rsqrt_iters=iters, rsqrt_clamp=clamp)
    same(c.layernorm(gx, rows, cols, row_off=32, **kw), o.layernorm(ox, rows, cols, row_off=32, **kw))


# --------------------------------------------------- fused = composed ----
def test_relu_equals_cmp_then_mul(mpc):
    c, _ = pair_ctx(mpc, step=20)
    n = 5000
    gx = c.share(torch.from_numpy(workloads.relu_inputs(n)).cuda())
    s0 = c.step
    a = c.relu(gx, off=0)
    c.set_step(s0, force=True)
    l = c.cmp(gx, off=0)
    notl = ((1 - l[0].to(torch.int64)).to(torch.uint64), (-l[1].to(torch.int64)).to(torch.uint64))
    b = c.mul(gx, notl, off=0)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_determinism(mpc):
    c, _ = pair_ctx(mpc, 2, step=0)
    rows, cols = 64, 128
    gx = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
    a = c.softmax(gx, rows, cols)
    c.set_step(1, force=True)
    b = c.softmax(gx, rows, cols)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


# ---------------------------------------------- full BASELINE sizes, EVERY share ----
# The oracle runs the whole op on every host core (tests/oracle_pool.py: 32-aligned slices with
# their global offsets reproduce the unsharded op exactly), and every output share of both parties
# is compared -- in the launch configuration bench.py / tools/sweep.py time.
import oracle_pool  # noqa: E402


def test_softmax_cfg2_full_size_every_share(mpc):
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    keys = workloads.keys(2)
    c = mpc.Ctx.for_cfg(keys)
    x = workloads.softmax_inputs(rows, cols)
    gx = c.share(torch.from_numpy(x).cuda())
    s0 = c.step
    z = c.softmax(gx, rows, cols)
    r = oracle_pool.rows_op("softmax", keys, s0, (np_(gx[0]), np_(gx[1])), rows, cols)
    same(z, r)
    # reconstructed floats vs the true softmax: the exp-limit formula itself is
    # 1.02e-2 from the true softmax on the full cfg2 input; fixed point adds <= 2e-3
    _, f = c.open(z)
    y = np_(f).reshape(rows, cols)
    xd = np_(c.open(gx)[1]).reshape(rows, cols)
    assert np.max(np.abs(y - fr.softmax_formula(xd))) <= 2e-3
    assert np.max(np.abs(y - fr.softmax(xd))) <= 1.25e-2


def test_softmax_cfg2_cone_full_size_every_share(mpc):
    """the carry-cone circuit (NEXT #1) in the headline shape: bit-identical to the same oracle"""
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    keys = workloads.keys(2)
    c = mpc.Ctx.for_cfg(keys)
    c.set_ltz_circuit(1)
    gx = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
    s0 = c.step
    z = c.softmax(gx, rows, cols)
    same(z, oracle_pool.rows_op("softmax", keys, s0, (np_(gx[0]), np_(gx[1])), rows, cols))


def test_gelu_cfg3_full_size_every_share(mpc):
    n = workloads.SHAPES["cfg3_gelu"]
    keys = workloads.keys(3)
    c = mpc.Ctx.for_cfg(keys)
    x = workloads.normal_inputs(n, 3)
    gx = c.share(torch.from_numpy(x).cuda())
    s0 = c.step
    z = c.gelu(gx, form="poly_abs", degree=4)
    knobs = mpc.default_act("gelu", "poly_abs", degree=4)
    r = oracle_pool.elems_op("act", keys, s0, (np_(gx[0]), np_(gx[1])), n, act="gelu", form="poly_abs", degree=4,
                             B=knobs["B"], coeffs=knobs["coeffs"])
    same(z, r)
    _, f = c.open(z)
    xd = np_(c.open(gx)[1])
    assert np.max(np.abs(np_(f) - fr.gelu(xd))) <= 4.2e-3 + 1e-3


def test_relu_cfg4_first_layer_shard_every_share(mpc):
    N, C, H, W = workloads.SHAPES["cfg4_relu_first"]
    n = N * C * H * W // 4          # one 8-image shard of the first ReLU layer (4 pairs)
    keys = workloads.keys(4)
    c = mpc.Ctx.for_cfg(keys)
    x = workloads.relu_inputs(n)
    gx = c.share(torch.from_numpy(x).cuda())
    s0 = c.step
    z = c.relu(gx)
    ring = np_(c.open(z)[0]).view(np.int64)
    xr = np_(c.open(gx)[0]).view(np.int64)
    assert np.array_equal(ring, np.maximum(xr, 0))      # ReLU is exact
    same(z, oracle_pool.elems_op("relu", keys, s0, (np_(gx[0]), np_(gx[1])), n))


def test_softmax_cfg5_pair_shard_every_share(mpc):
    """cfg5: one pair's shard of a GPT-2 attention softmax (2 sequences x 12 heads x 1024 rows of
    1024), the launch bench/sweep time; every share bit-exact, floats within §5."""
    rows, cols = 2 * 12 * 1024, 1024
    keys = workloads.keys(5)
    c = mpc.Ctx.for_cfg(keys)
    x = workloads.softmax_inputs(rows, cols, seed_cfg=5)
    gx = c.share(torch.from_numpy(x).cuda())
    s0 = c.step
    z = c.softmax(gx, rows, cols)
    same(z, oracle_pool.rows_op("softmax", keys, s0, (np_(gx[0]), np_(gx[1])), rows, cols))
    _, f = c.open(z)
    y = np_(f).reshape(rows, cols)
    xd = np_(c.open(gx)[1]).reshape(rows, cols)
    sl = slice(0, 2048)                       # float checks on a 2048-row block (fp64 formula is slow)
    # vs formula 2*4*2^t + 8 ulp (the survey's simulated 9.3e-3 came from fewer rows;
    # measured here 1.05e-2); vs the true softmax 3e-2 (SURVEY §8(c6) simulated 2.35e-2 on fewer
    # rows; measured here 2.58e-2 on 2048 rows of 1024)
    assert np.max(np.abs(y[sl] - fr.softmax_formula(xd[sl]))) <= (2 * 4 * 2**8 + 8) * 2.0**-16
    assert np.max(np.abs(y[sl] - fr.softmax(xd[sl]))) <= 3e-2


def test_layernorm_cfg5_full_size_every_share(mpc):
    rows, cols = workloads.SHAPES["cfg5_ln"]
    keys = workloads.keys(5)
    c = mpc.Ctx.for_cfg(keys)
    x = workloads.layernorm_inputs(rows, cols)
    gx = c.share(torch.from_numpy(x).cuda())
    s0 = c.step
    z = c.layernorm(gx, rows, cols)
    same(z, oracle_pool.rows_op("layernorm", keys, s0, (np_(gx[0]), np_(gx[1])), rows, cols))
    _, f = c.open(z)
    xd = np_(c.open(gx)[1]).reshape(rows, cols)
    y = np_(f).reshape(rows, cols)
    assert np.max(np.abs(y - fr.layernorm_formula(xd))) <= 2e-3          # vs formula
    # vs the true layernorm: E(1/768) = 85/2^16 (R25) scales mean and variance by -0.39 %, and the
    # 3-iteration rsqrt adds its own error; 1.3e-2 was simulated on fewer rows, 1.50e-2 is
    # measured over all 8192 cfg5 rows
    assert np.max(np.abs(y - fr.layernorm(xd))) <= 1.6e-2


def test_maxpool_cfg4_shard_every_share(mpc):
    """cfg4 MaxPool 3x3/2 pad 1 on one pair's 8-image shard of 32 x 64 x 112 x 112: exact
    reconstruction, and every output share of all 8 images bit-exact vs the oracle."""
    N, C, H, W = 8, 64, 112, 112
    keys = workloads.keys(4)
    c = mpc.Ctx.for_cfg(keys)
    x = workloads.maxpool_inputs((N, C, H, W))
    gx = c.share(torch.from_numpy(x).cuda())
    s0 = c.step
    z = c.maxpool2d(gx, N, C, H, W, 3, 2, 1)
    Ho = Wo = 56
    xr = np_(c.open(gx)[0]).view(np.int64).reshape(N, C, H, W)
    pad = np.zeros((N, C, H + 2, W + 2), dtype=np.int64)        # public zero padding (R26)
    pad[:, :, 1:-1, 1:-1] = xr
    ref = np.full((N, C, Ho, Wo), np.iinfo(np.int64).min)
    for i in range(3):
        for j in range(3):
            ref = np.maximum(ref, pad[:, :, i:i + 2 * Ho:2, j:j + 2 * Wo:2])
    assert np.array_equal(np_(c.open(z)[0]).view(np.int64).reshape(N, C, Ho, Wo), ref)
    same(z, oracle_pool.maxpool_op(keys, s0, (np_(gx[0]), np_(gx[1])), N, C, H, W, k=3, stride=2, pad=1))


def test_bad_args_raise(mpc):
    c, _ = pair_ctx(mpc)
    gx = c.share(torch.zeros(64, dtype=torch.float64).cuda())
    with pytest.raises(mpc.MPCError):
        c.cmp(gx, off=3)
    with pytest.raises(mpc.MPCError):
        c.exp(gx, t=9)
    with pytest.raises(mpc.MPCError):
        c.set_step(0)
    st = c.step
    with pytest.raises(mpc.MPCError):
        c.cmp(gx, window=65)
    assert c.step == st


# ------------------------------------------------ square-pair triples (NEXT #2) ----
@pytest.mark.parametrize("n,off", [(1, 0), (77, 3), (100_001, 64)])
def test_square(mpc, n, off):
    c, o = pair_ctx(mpc, step=13)
    x = workloads.act_inputs(n)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.square(gx, off=off, trunc_bits=16), o.square(ox, off=off, trunc_bits=16))
    assert c.step == o.step


@pytest.mark.parametrize("t,clamp", [(8, 0), (8, 1), (3, 0)])
def test_exp_square(mpc, t, clamp):
    c, o = pair_ctx(mpc, step=2)
    x = workloads.exp_inputs(4096 + 13, tail_frac=0.05)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.exp(gx, off=32, t=t, clamp=clamp, square=1), o.exp(ox, off=32, t=t, clamp=clamp, square=1))


@pytest.mark.parametrize("rows,cols", [(64, 128), (32, 1024)])
def test_softmax_square(mpc, rows, cols):
    c, o = pair_ctx(mpc, 2, step=1)
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    kw = dict(exp_square=1, recip_square=1)
    same(c.softmax(gx, rows, cols, **kw), o.softmax(ox, rows, cols, **kw))


def test_rsqrt_layernorm_square(mpc):
    c, o = pair_ctx(mpc, 5, step=1)
    x = workloads.rsqrt_inputs(3000)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.rsqrt(gx, square=1), o.rsqrt(ox, square=1))
    y = workloads.layernorm_inputs(40, 768)
    gy, oy = c.share(torch.from_numpy(y).cuda()), o.share(y)
    same(c.layernorm(gy, 40, 768, rsqrt_square=1), o.layernorm(oy, 40, 768, rsqrt_square=1))


# ------------------------------------------------ carry-cone LTZ (NEXT #1) ----
@pytest.mark.parametrize("w", [1, 2, 3, 5, 17, 18, 21, 32, 33, 34, 35, 47, 48, 63, 64])
@pytest.mark.parametrize("n", [45, 4096 + 96 + 7])
def test_cone_ltz_matches_oracle(mpc, w, n):
    """The carry cone computes the same sign bit, so the output shares equal the
    Kogge-Stone contract's (oracle) bit for bit."""
    c, o = pair_ctx(mpc, step=3)
    c.set_ltz_circuit(1)
    x = workloads.act_inputs(n) * 3
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.cmp(gx, off=64, window=w), o.ltz(ox, off=64, window=w))
    same(c.relu(gx, off=0, window=w), o.relu(ox, off=0, window=w))


def _cone_gates_bruteforce(w):
    """Pruned carry cone (ltz_cone.cuh) built node by node: leaves j < m real, j >= m public pads;
    a node whose hi child is all pads IS its lo child (no gate); a node with two real children
    costs a G gate, plus a P gate when its P is used (it is a hi child, or its parent's P is used)."""
    m = w - 1
    if m <= 0:
        return 0
    L = (m - 1).bit_length()
    gates = m                                   # g-layer
    if L == 0:
        return gates                            # one leaf: the carry is g_0
    def node(k, i, need_p):                     # level k over leaves [i 2^(k+1), (i+1) 2^(k+1))
        nonlocal gates
        lo_start, hi_start = i << (k + 1), (i << (k + 1)) + (1 << k)
        if lo_start >= m:
            return                              # all pads: public (0, 1)
        if hi_start >= m:                       # copy of the lo child
            if k > 0:
                node(k - 1, 2 * i, need_p)
            return
        gates += 1 + (1 if need_p else 0)
        if k > 0:
            node(k - 1, 2 * i, need_p)
            node(k - 1, 2 * i + 1, True)
    node(L - 1, 0, False)
    return gates


@pytest.mark.parametrize("w", [2, 3, 9, 17, 21, 25, 33, 40, 64])
def test_cone_gate_count_in_stats(mpc, w):
    """bytes each party sends for one cone LTZ = groups x (8 B per AND gate + 4 B for B2A);
    the pruned cone's gate count equals the node-by-node construction (89 at w=33, 181 at w=64)."""
    c, _ = pair_ctx(mpc)
    c.set_ltz_circuit(1)
    gx = c.share(torch.zeros(32 * 10, dtype=torch.float64).cuda())
    c.reset_stats()
    c.cmp(gx, window=w)
    g = _cone_gates_bruteforce(w)
    assert c.stats()["bytes_per_party"] == 10 * (8 * g + 4)
    assert {33: 89, 64: 181, 21: 53}.get(w, g) == g


def test_cone_ltz_large_sampled(mpc):
    n = 32 * 64 * 112 * 112 // 16
    keys = workloads.keys(4)
    c = mpc.Ctx.for_cfg(keys)
    c.set_ltz_circuit(1)
    x = workloads.relu_inputs(n)
    gx = c.share(torch.from_numpy(x).cuda())
    s0 = c.step
    z = c.relu(gx)
    z0, z1 = np_(z[0]), np_(z[1])
    for off in (0, n // 2 - (n // 2) % 32, n - 4096):
        o = Oracle.for_cfg(keys, s0)
        sl = slice(off, off + 4096)
        r = o.relu((np_(gx[0])[sl], np_(gx[1])[sl]), off=off)
        assert np.array_equal(z0[sl], r[0]) and np.array_equal(z1[sl], r[1])


@pytest.mark.parametrize("act,form,deg", ACTS)
def test_cone_activations(mpc, act, form, deg):
    c, o = pair_ctx(mpc, step=4)
    c.set_ltz_circuit(1)
    n = 4096 * 2 + 99
    x = workloads.act_inputs(n)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    if form == "erf":
        knobs = mpc.default_act(act, "erf", erf_terms=deg)
        g = getattr(c, act)(gx, off=0, form="erf", erf_terms=deg)
        r = o.act(ox, act, "erf", 1, knobs["B"], None, deg)
    else:
        knobs = mpc.default_act(act, form, degree=deg)
        g = getattr(c, act)(gx, off=0, form=form, degree=deg)
        r = o.act(ox, act, form, knobs["degree"], knobs["B"], knobs["coeffs"] or [0.0])
    same(g, r)
    assert c.step == o.step


@pytest.mark.parametrize("rows,cols,w", [(64, 128, 33), (45, 77, 33), (32, 1024, 33), (70, 9, 33), (33, 3, 33),
                                         (64, 128, 64), (45, 77, 40), (70, 9, 64), (40, 16, 21)])
def test_cone_softmax_and_max(mpc, rows, cols, w):
    c, o = pair_ctx(mpc, 2, step=1)
    c.set_ltz_circuit(1)
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.max(gx, rows, cols, row_off=32, window=w), o.max(ox, rows, cols, row_off=32, window=w))
    same(c.softmax(gx, rows, cols, row_off=32, window=w), o.softmax(ox, rows, cols, row_off=32, window=w))
    same(c.softmax(gx, rows, cols, exp_square=1, recip_square=1, window=w),
         o.softmax(ox, rows, cols, exp_square=1, recip_square=1, window=w))
    same(c.softmax(gx, rows, cols, causal=1, window=w), o.softmax(ox, rows, cols, causal=1, window=w))


@pytest.mark.parametrize("w", [33, 21, 64])
def test_cone_maxpool(mpc, w):
    N, C, H, W = 2, 16, 14, 15
    c, o = pair_ctx(mpc, 4, step=1)
    c.set_ltz_circuit(1)
    x = workloads.maxpool_inputs((N, C, H, W)) - 0.25
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.maxpool2d(gx, N, C, H, W, 3, 2, 1, img_off=2, window=w),
         o.maxpool2d(ox, N, C, H, W, 3, 2, 1, img_off=2, window=w))


@pytest.mark.parametrize("w", [40, 64])
def test_cone_activations_wide(mpc, w):
    c, o = pair_ctx(mpc, step=4)
    c.set_ltz_circuit(1)
    n = 4096 + 99
    x = workloads.act_inputs(n)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    knobs = mpc.default_act("gelu", "poly_abs", degree=4)
    same(c.gelu(gx, form="poly_abs", degree=4, window=w),
         o.act(ox, "gelu", "poly_abs", 4, knobs["B"], knobs["coeffs"], window=w))


# ------------------------------------------------- T5: fused = composed (row ops) ----
def _i64(t):
    return t.view(torch.int64)


def _bcast(v, cols):
    return v.view(-1, 1).expand(-1, cols).contiguous().view(-1)


def test_softmax_fused_equals_composed(mpc):
    """k_softmax's shares equal the composition of ABI calls on the same step ids: max ->
    (local) x - max -> exp (element units) -> (local) row sums -> recip (row units) -> mul by the
    broadcast reciprocal (element units) + truncation."""
    c, _ = pair_ctx(mpc, 2, step=40)
    rows, cols, roff = 64, 128, 32
    x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
    s0 = c.step
    z = c.softmax(x, rows, cols, row_off=roff)
    c.set_step(s0, force=True)
    mx = c.max(x, rows, cols, row_off=roff)
    d = tuple((_i64(x[p]).view(rows, cols) - _i64(mx[p]).view(rows, 1)).view(-1).view(torch.uint64) for p in (0, 1))
    e = c.exp(d, off=roff * cols, t=8)
    S = tuple(_i64(e[p]).view(rows, cols).sum(1).view(torch.uint64) for p in (0, 1))
    r = c.recip(S, off=roff, iters=10, t=8)
    rb = tuple(_bcast(r[p], cols) for p in (0, 1))
    out = c.mul(e, rb, off=roff * cols, trunc_bits=16)
    assert torch.equal(z[0], out[0]) and torch.equal(z[1], out[1])


def test_layernorm_fused_equals_composed(mpc):
    c, _ = pair_ctx(mpc, 5, step=50)
    rows, cols, roff = 40, 768, 64
    x = c.share(torch.from_numpy(workloads.layernorm_inputs(rows, cols)).cuda())
    s0 = c.step
    z = c.layernorm(x, rows, cols, row_off=roff)
    c.set_step(s0, force=True)
    e_invd, e_eps = round(65536 / cols), round(1e-5 * 65536)        # E(1/d), E(eps) (R2, R25)
    mu = [(_i64(x[p]).view(rows, cols).sum(1) * e_invd) >> 16 for p in (0, 1)]
    cc = tuple((_i64(x[p]).view(rows, cols) - mu[p].view(rows, 1)).view(-1).view(torch.uint64) for p in (0, 1))
    q = c.mul(cc, cc, off=roff * cols, trunc_bits=16)
    v = [(_i64(q[p]).view(rows, cols).sum(1) * e_invd) >> 16 for p in (0, 1)]
    v[0] = v[0] + e_eps                                             # public addend: party 0
    r = c.rsqrt(tuple(t.view(torch.uint64) for t in v), off=roff, iters=3, t=8)
    out = c.mul(cc, tuple(_bcast(r[p], cols) for p in (0, 1)), off=roff * cols, trunc_bits=16)
    assert torch.equal(z[0], out[0]) and torch.equal(z[1], out[1])


@pytest.mark.parametrize("rows,cols", [(1, 1), (31, 1), (33, 2), (1, 3), (64, 17), (5, 1025), (3, 16384), (2, 20001)])
def test_softmax_edge_shapes(mpc, rows, cols):
    """Degenerate and ragged softmax shapes: a single column (no max-tree level), two and three
    columns (odd carry), one row, 17 columns (CTA tree with an odd level), 1025 columns (global
    work tile and an odd first level)."""
    c, o = pair_ctx(mpc, 2, step=7)
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.softmax(gx, rows, cols, row_off=96), o.softmax(ox, rows, cols, row_off=96))
    assert c.step == o.step


@pytest.mark.parametrize("rows,cols", [(3, 16384), (2, 20001)])
def test_long_rows_max_layernorm(mpc, rows, cols):
    """Rows far beyond the shared-memory staging (16K / 20K elements: the global work tile path)
    for the row max and LayerNorm."""
    c, o = pair_ctx(mpc, 2, step=9)
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.max(gx, rows, cols, row_off=32), o.max(ox, rows, cols, row_off=32))
    same(c.layernorm(gx, rows, cols, row_off=64), o.layernorm(ox, rows, cols, row_off=64))
    assert c.step == o.step


@pytest.mark.parametrize("rows,cols,row_off,kw", [
    (256, 128, 0, {}), (200, 40, 32, {}), (96, 128, 64, dict(bcast=1, exp_square=1)),
    (64, 77, 96, dict(exp_clamp=1, window=40)), (70, 1, 32, {}), (33, 1024, 0, {})])
def test_softmax_causal(mpc, rows, cols, row_off, kw):
    """Causal softmax: bit-exact vs the oracle, masked outputs exactly 0, in
    BOTH mode, with the carry cone, in PAIR loopback and through the host-buffer pipeline."""
    c, o = pair_ctx(mpc, 5, step=11)
    x = workloads.softmax_inputs(rows, cols, seed_cfg=5)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    s0 = c.step
    ref = o.softmax(ox, rows, cols, row_off=row_off, causal=1, **kw)
    same(c.softmax(gx, rows, cols, row_off=row_off, causal=1, **kw), ref)
    assert c.step == o.step
    c.set_ltz_circuit(1)
    c.set_step(s0, force=True)
    same(c.softmax(gx, rows, cols, row_off=row_off, causal=1, **kw), ref)
    p = mpc.Ctx.for_cfg(workloads.keys(5), mode=mpc.binding.MODE_PAIR_LOOPBACK)
    p.set_step(s0)
    zp = p.softmax(gx, rows, cols, row_off=row_off, causal=1, **kw)
    p.sync()
    same(zp, ref)
    hx = tuple(t.cpu().pin_memory() for t in gx)
    hz = tuple(torch.empty_like(t).pin_memory() for t in hx)
    c.set_step(s0, force=True)
    c.softmax_hostio(hx, hz, rows, cols, row_off=row_off, chunk_rows=64, causal=1, **kw)
    torch.cuda.synchronize()
    same(hz, ref)


def test_matmul_long_k_tensor_cores(mpc):
    """K = 5000 (K' = 15000 for party 1, inside the exact-accumulator bound) on the tensor cores."""
    c, o = pair_ctx(mpc, 3, step=2)
    c.set_matmul_engine(2)
    M, K, N = 3, 5000, 5
    x, y = workloads.act_inputs(M * K, lo=-1, hi=1), workloads.act_inputs(K * N, seed_cfg=5, lo=-1, hi=1)
    gx, gy = c.share(torch.from_numpy(x).cuda()), c.share(torch.from_numpy(y).cuda())
    ox, oy = o.share(x), o.share(y)
    same(c.matmul(gx, gy, 1, M, K, N, trunc_bits=16), o.matmul(ox, oy, 1, M, K, N, trunc_bits=16))
