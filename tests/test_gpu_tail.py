"""Row-kernel plans and LayerNorm kernels, every share against the oracle (or the other plan on the
same call).  Covered here:
* the 32-row tiles' last round as 16-row half tiles (kernels.cuh tile_plan; off by default, measured
  slower -- MPC_TAIL_HALF=1 turns it on per call);
* the balanced softmax plan (softmax_bal_*: one range of ~rows / grid rows per CTA, any row alignment
  in the max tree) in BOTH, with the carry cone, the broadcast triple, a clamped exp, causal rows,
  in the PAIR protocol (loopback) and with the dealer's correction stream;
* the split softmax (balanced k_max + k_softmax_rest; MPC_SOFTMAX_SPLIT=1, A/B path);
* LayerNorm: k_ln_row (one warp per row), k_ln_blk (shared-memory row blocks by bulk copies) and
  k_ln_fused on the same calls.
The contract (steps, units, PRG words) does not depend on the plan.  MPC_ROW_GRID_CAP caps the grid
so that small inputs take the multi-round, half-tile and multi-block paths."""
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


def same(g, o):
    a0, a1 = g[0].cpu().numpy(), g[1].cpu().numpy()
    bad = np.nonzero((a0 != o[0]) | (a1 != o[1]))[0]
    assert bad.size == 0, f"{bad.size} mismatching shares, first at {bad[:5]}"


def ctx(m, cfg, step, mode=None):
    keys = workloads.keys(cfg)
    c = m.Ctx.for_cfg(keys) if mode is None else m.Ctx.for_cfg(keys, mode=mode)
    c.set_step(step)
    return c, Oracle.for_cfg(keys, step)


# (rows, cap): 5 tiles on 4 CTAs -> 4 full + 2 halves (the last one ragged: 150 rows); 7 on 3 -> 6 +
# 2; 5 on 2 -> 2P > ncta, no split (multi-round only); 3 tiles on 4 -> one round
PLANS = [(150, 4), (160, 4), (224, 3), (150, 2), (96, 4), (140, 4)]


@pytest.mark.parametrize("rows,cap", PLANS)
@pytest.mark.parametrize("cols", [128, 77, 9])
def test_softmax_half_tiles(m, monkeypatch, rows, cap, cols):
    monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    monkeypatch.setenv("MPC_TAIL_HALF", "1")
    monkeypatch.setenv("MPC_SOFTMAX_BAL", "0")
    c, o = ctx(m, 2, 3)
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.softmax(gx, rows, cols, row_off=32), o.softmax(ox, rows, cols, row_off=32))


@pytest.mark.parametrize("rows,cap", [(150, 4), (224, 3)])
@pytest.mark.parametrize("kw", [dict(exp_clamp=1), dict(causal=1), dict(bcast=1), dict(window=64)])
def test_softmax_half_tiles_knobs(m, monkeypatch, rows, cap, kw):
    monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    monkeypatch.setenv("MPC_TAIL_HALF", "1")
    monkeypatch.setenv("MPC_SOFTMAX_BAL", "0")
    cols = 64
    c, o = ctx(m, 2, 5)
    x = workloads.softmax_inputs(rows, cols, spike="exp_clamp" in kw)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.softmax(gx, rows, cols, row_off=64, **kw), o.softmax(ox, rows, cols, row_off=64, **kw))


@pytest.mark.parametrize("rows,cap", [(150, 4), (224, 3)])
def test_softmax_half_tiles_cone(m, monkeypatch, rows, cap):
    monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    monkeypatch.setenv("MPC_TAIL_HALF", "1")
    monkeypatch.setenv("MPC_SOFTMAX_BAL", "0")
    cols = 128
    c, o = ctx(m, 2, 7)
    c.set_ltz_circuit(1)
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.softmax(gx, rows, cols), o.softmax(ox, rows, cols))


@pytest.mark.parametrize("rows,cap", [(150, 4), (224, 3)])
@pytest.mark.parametrize("cols", [128, 33])
def test_max_half_tiles(m, monkeypatch, rows, cap, cols):
    monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    monkeypatch.setenv("MPC_TAIL_HALF", "1")
    monkeypatch.setenv("MPC_SOFTMAX_BAL", "0")
    monkeypatch.setenv("MPC_MAX_BAL", "0")
    c, o = ctx(m, 2, 1)
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.max(gx, rows, cols, row_off=32), o.max(ox, rows, cols, row_off=32))


def test_softmax_half_tiles_off_equals_on(m, monkeypatch):
    """the capped grid with half tiles equals the uncapped one share for share"""
    rows, cols = 224, 128
    c, _ = ctx(m, 2, 9)
    gx = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
    s0 = c.step
    a = c.softmax(gx, rows, cols)
    monkeypatch.setenv("MPC_ROW_GRID_CAP", "3")
    monkeypatch.setenv("MPC_TAIL_HALF", "1")
    monkeypatch.setenv("MPC_SOFTMAX_BAL", "0")
    c.set_step(s0, force=True)
    b = c.softmax(gx, rows, cols)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


@pytest.mark.parametrize("rows,cap", [(150, 4), (224, 3)])
def test_softmax_half_tiles_loopback(m, monkeypatch, rows, cap):
    """PAIR protocol in loopback: each party's CTAs follow the same plan (the cap is per party)"""
    monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    monkeypatch.setenv("MPC_TAIL_HALF", "1")
    monkeypatch.setenv("MPC_SOFTMAX_BAL", "0")
    cols = 128
    c, o = ctx(m, 2, 11, mode=m.binding.MODE_PAIR_LOOPBACK)
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    z = c.softmax(gx, rows, cols, row_off=32)
    c.sync()
    same(z, o.softmax(ox, rows, cols, row_off=32))


# ---- balanced softmax plan (BOTH: one row range of ~rows / grid rows per CTA, kernels.cuh
# softmax_bal_*): taken when the 32-row tiles need more than one round; the cap shrinks the grid ----
BAL = [(150, 4), (140, 4), (160, 4), (255, 5), (1000, 16), (129, 4)]


@pytest.mark.parametrize("rows,cap", BAL)
@pytest.mark.parametrize("cols", [128, 77, 9, 2])
def test_softmax_balanced(m, monkeypatch, rows, cap, cols):
    monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    c, o = ctx(m, 2, 13)
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.softmax(gx, rows, cols, row_off=96), o.softmax(ox, rows, cols, row_off=96))


@pytest.mark.parametrize("rows,cap", [(150, 4), (255, 5)])
@pytest.mark.parametrize("kw", [dict(causal=1), dict(exp_square=1, recip_square=1), dict(recip_iters=3, exp_t=4),
                                dict(bcast=1), dict(bcast=1, exp_square=1, recip_square=1, causal=1),
                                dict(exp_clamp=1), dict(exp_clamp=1, causal=1)])
def test_softmax_balanced_knobs(m, monkeypatch, rows, cap, kw):
    monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    cols = 64
    c, o = ctx(m, 2, 15)
    x = workloads.softmax_inputs(rows, cols, spike="exp_clamp" in kw)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.softmax(gx, rows, cols, row_off=32, **kw), o.softmax(ox, rows, cols, row_off=32, **kw))


def test_softmax_balanced_after_other_tiles(m, monkeypatch):
    """the balanced launch sets its own dynamic shared-memory size after launches of the same kernel
    with other tile sizes (a stale attribute made the first full-size run fail)"""
    c, o = ctx(m, 2, 17)
    for rows, cols in [(64, 9), (40, 77)]:
        x = workloads.softmax_inputs(rows, cols)
        gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
        same(c.softmax(gx, rows, cols), o.softmax(ox, rows, cols))
    monkeypatch.setenv("MPC_ROW_GRID_CAP", "4")
    rows, cols = 150, 128
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.softmax(gx, rows, cols), o.softmax(ox, rows, cols))


def test_softmax_balanced_equals_tiles(m, monkeypatch):
    """balanced plan = 32-row tiles, share for share, on the same call"""
    rows, cols = 1000, 128
    monkeypatch.setenv("MPC_ROW_GRID_CAP", "16")
    c, _ = ctx(m, 2, 19)
    gx = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
    s0 = c.step
    a = c.softmax(gx, rows, cols)
    monkeypatch.setenv("MPC_SOFTMAX_BAL", "0")
    c.set_step(s0, force=True)
    b = c.softmax(gx, rows, cols)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


# ---- warp-per-row LayerNorm (kernels.cuh k_ln_row, BOTH): every share vs the oracle ----
@pytest.mark.parametrize("rows,cols", [(1, 2), (3, 64), (70, 768), (45, 100), (9, 1030), (33, 2048)])
@pytest.mark.parametrize("mean_mode", [0, 1])
def test_layernorm_row_kernel(m, monkeypatch, rows, cols, mean_mode):
    monkeypatch.setenv("MPC_LN_ROW", "1")
    monkeypatch.setenv("MPC_LN_BLK", "0")
    c, o = ctx(m, 5, 2)
    x = workloads.layernorm_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    kw = dict(mean_mode=mean_mode)
    same(c.layernorm(gx, rows, cols, row_off=32, **kw), o.layernorm(ox, rows, cols, row_off=32, **kw))
    assert c.step == o.step


@pytest.mark.parametrize("kw", [dict(rsqrt_iters=10), dict(rsqrt_square=1), dict(rsqrt_t=4, rsqrt_iters=1),
                                dict(rsqrt_iters=8, rsqrt_t=8)])
def test_layernorm_row_kernel_knobs(m, monkeypatch, kw):
    monkeypatch.setenv("MPC_LN_ROW", "1")
    monkeypatch.setenv("MPC_LN_BLK", "0")
    rows, cols = 150, 768
    c, o = ctx(m, 5, 4)
    x = workloads.layernorm_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.layernorm(gx, rows, cols, row_off=64, **kw), o.layernorm(ox, rows, cols, row_off=64, **kw))


def test_layernorm_row_kernel_many_rows_per_warp(m, monkeypatch):
    """a long input gives every warp several rows (forced: the heuristic picks k_ln_fused here)"""
    monkeypatch.setenv("MPC_LN_ROW", "1")
    monkeypatch.setenv("MPC_LN_BLK", "0")
    rows, cols = 6000, 128
    c, o = ctx(m, 5, 6)
    x = workloads.layernorm_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.layernorm(gx, rows, cols), o.layernorm(ox, rows, cols))


@pytest.mark.parametrize("rows", [4700, 2368 * 2])
def test_layernorm_kernel_choice_both_exact(m, monkeypatch, rows):
    """k_ln_row and k_ln_fused on the same call: the same shares"""
    cols = 256
    c, _ = ctx(m, 5, 8)
    gx = c.share(torch.from_numpy(workloads.layernorm_inputs(rows, cols)).cuda())
    s0 = c.step
    monkeypatch.setenv("MPC_LN_ROW", "1")
    monkeypatch.setenv("MPC_LN_BLK", "0")
    a = c.layernorm(gx, rows, cols)
    monkeypatch.setenv("MPC_LN_ROW", "0")
    c.set_step(s0, force=True)
    b = c.layernorm(gx, rows, cols)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


# ---- LayerNorm on shared-memory row blocks (ln_blk.cuh k_ln_blk, BOTH): every share vs the oracle ----
@pytest.mark.parametrize("rows,cols", [(1, 2), (7, 64), (70, 768), (45, 100), (9, 1030), (33, 2048), (5, 3072),
                                       (13, 4000)])
@pytest.mark.parametrize("cap", ["0", "3"])
def test_layernorm_blocks(m, monkeypatch, rows, cols, cap):
    """RB = 8 / 4 / 2 / 1 rows per block by width (4000: no block fits, another kernel); cap 3: several
    blocks per CTA through both buffers; ragged last blocks"""
    if cap != "0":
        monkeypatch.setenv("MPC_ROW_GRID_CAP", cap)
    c, o = ctx(m, 5, 12)
    x = workloads.layernorm_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    for mm in (0, 1):
        same(c.layernorm(gx, rows, cols, row_off=32, mean_mode=mm), o.layernorm(ox, rows, cols, row_off=32, mean_mode=mm))
    assert c.step == o.step


@pytest.mark.parametrize("kw", [dict(rsqrt_iters=10), dict(rsqrt_square=1), dict(rsqrt_t=4, rsqrt_iters=1),
                                dict(rsqrt_iters=8, rsqrt_t=8), dict(eps=0.5)])
def test_layernorm_blocks_knobs(m, monkeypatch, kw):
    monkeypatch.setenv("MPC_ROW_GRID_CAP", "5")
    rows, cols = 150, 768
    c, o = ctx(m, 5, 14)
    x = workloads.layernorm_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.layernorm(gx, rows, cols, row_off=64, **kw), o.layernorm(ox, rows, cols, row_off=64, **kw))


@pytest.mark.parametrize("rows,cols", [(8192, 768), (3001, 256)])
def test_layernorm_blocks_equal_fused(m, monkeypatch, rows, cols):
    """k_ln_blk and k_ln_fused on the same call: the same shares"""
    c, _ = ctx(m, 5, 16)
    gx = c.share(torch.from_numpy(workloads.layernorm_inputs(rows, cols)).cuda())
    s0 = c.step
    a = c.layernorm(gx, rows, cols)
    monkeypatch.setenv("MPC_LN_BLK", "0")
    monkeypatch.setenv("MPC_LN_ROW", "0")
    c.set_step(s0, force=True)
    b = c.layernorm(gx, rows, cols)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


# ---- balanced softmax plan in the PAIR protocol (loopback) and with the dealer's stream ----
@pytest.mark.parametrize("rows,cap,cols", [(150, 4, 128), (1000, 16, 128), (255, 5, 77), (64, 0, 128),
                                           (12288, 0, 128), (340, 4, 128), (150, 4, 1024)])
@pytest.mark.parametrize("bcast", [0, 1])
def test_softmax_balanced_pair_loopback(m, monkeypatch, rows, cap, cols, bcast):
    """both parties' CTA c run the same row range and exchange sequence: bit-identical to BOTH"""
    if cap:
        monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    keys = workloads.keys(2)
    b = m.Ctx.for_cfg(keys)
    p = m.Ctx.for_cfg(keys, mode=m.binding.MODE_PAIR_LOOPBACK)
    b.set_step(23)
    p.set_step(23)
    x = b.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
    p.set_step(b.step)
    zb = b.softmax(x, rows, cols, row_off=32, bcast=bcast)
    zp = p.softmax(x, rows, cols, row_off=32, bcast=bcast)
    p.sync()
    torch.cuda.synchronize()
    assert torch.equal(zb[0], zp[0]) and torch.equal(zb[1], zp[1])
    if rows <= 1000:
        o = Oracle.for_cfg(keys, 23)
        ox = o.share(workloads.softmax_inputs(rows, cols))
        same(zp, o.softmax(ox, rows, cols, row_off=32, bcast=bcast))


@pytest.mark.parametrize("rows,cap", [(150, 4), (1000, 16), (340, 4)])
def test_softmax_balanced_dealer_stream(m, monkeypatch, rows, cap):
    """the dealer's offline pass runs party 1's balanced kernel with the same grid: party 1 consumes
    exactly the stream and the shares equal BOTH's"""
    monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    cols = 128
    keys = workloads.keys(2)
    b = m.Ctx.for_cfg(keys)
    p = m.Ctx.for_cfg(keys, mode=m.binding.MODE_PAIR_LOOPBACK)
    d = m.Ctx.dealer(keys, target=m.binding.MODE_PAIR_LOOPBACK)
    for c in (b, p, d):
        c.set_step(5)
    xs = b.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
    p.set_step(b.step)
    d.set_step(b.step)
    zb = b.softmax(xs, rows, cols)
    d.softmax(m.Ctx.like(rows * cols), rows, cols)
    p.set_corrections(d.dealer_stream())
    zp = p.softmax(xs, rows, cols)
    p.sync()
    assert p.corrections_left() == 0
    torch.cuda.synchronize()
    assert torch.equal(zb[0], zp[0]) and torch.equal(zb[1], zp[1])


# ---- split softmax: balanced k_max launch + k_softmax_rest (3 CTAs per SM); MPC_SOFTMAX_SPLIT=1 ----
@pytest.mark.parametrize("rows,cap,cols", [(150, 4, 128), (1000, 0, 128), (255, 5, 78), (12288, 0, 128), (64, 0, 2)])
def test_softmax_split(m, monkeypatch, rows, cap, cols):
    monkeypatch.setenv("MPC_SOFTMAX_SPLIT", "1")
    if cap:
        monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    c, o = ctx(m, 2, 25)
    x = workloads.softmax_inputs(rows, cols)
    gx = c.share(torch.from_numpy(x).cuda())
    s0 = c.step
    a = c.softmax(gx, rows, cols, row_off=32)
    monkeypatch.setenv("MPC_SOFTMAX_SPLIT", "0")
    c.set_step(s0, force=True)
    b = c.softmax(gx, rows, cols, row_off=32)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    if rows <= 1000:
        ox = o.share(x)
        same(a, o.softmax(ox, rows, cols, row_off=32))


@pytest.mark.parametrize("rows,cap,cols", [(150, 4, 128), (1000, 16, 128), (255, 5, 77), (96, 0, 64)])
@pytest.mark.parametrize("causal", [0, 1])
def test_softmax_balanced_cone(m, monkeypatch, rows, cap, cols, causal):
    """the carry-cone max tree (NEXT #1) on the balanced plan: groups offset at range boundaries"""
    if cap:
        monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    c, o = ctx(m, 2, 27)
    c.set_ltz_circuit(1)
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.softmax(gx, rows, cols, row_off=32, causal=causal), o.softmax(ox, rows, cols, row_off=32, causal=causal))


def test_layernorm_unaligned_shares(m):
    """share arrays that start 8 bytes past a 16-byte boundary (cp.async.bulk cannot read them): the
    row-block kernel is not taken, the result is still the oracle's"""
    rows, cols = 33, 768
    c, o = ctx(m, 5, 30)
    x = workloads.layernorm_inputs(rows, cols)
    gx = c.share(torch.from_numpy(np.concatenate([[0.0], x.ravel()])).cuda())
    gv = (gx[0][1:], gx[1][1:])
    assert gv[0].data_ptr() % 16 == 8
    ov = (o.share(np.concatenate([[0.0], x.ravel()])))
    ox = (ov[0][1:], ov[1][1:])
    same(c.layernorm(gv, rows, cols), o.layernorm(ox, rows, cols))


@pytest.mark.parametrize("rows,cap,cols", [(150, 4, 1024), (300, 0, 1024), (255, 5, 300), (64, 0, 200),
                                           (340, 4, 1024), (370, 4, 256)])
@pytest.mark.parametrize("kw", [dict(), dict(causal=1), dict(bcast=1)])
def test_softmax_balanced_wide_rows(m, monkeypatch, rows, cap, cols, kw):
    """rows wider than the shared-memory work area (cols > 192): the balanced plan with its level
    buffers in a per-CTA global work area and the triple tables in shared memory (340 / 370 rows on 4
    CTAs: 86 / 94 rows per CTA, three tables and three reciprocal-chain warps)"""
    if cap:
        monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    c, o = ctx(m, 2, 29)
    x = workloads.softmax_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.softmax(gx, rows, cols, row_off=64, **kw), o.softmax(ox, rows, cols, row_off=64, **kw))


def test_softmax_balanced_wide_equals_tiles(m, monkeypatch):
    rows, cols = 2000, 1024
    c, _ = ctx(m, 2, 31)
    gx = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
    s0 = c.step
    a = c.softmax(gx, rows, cols)
    monkeypatch.setenv("MPC_SOFTMAX_BAL_WIDE", "0")
    c.set_step(s0, force=True)
    b = c.softmax(gx, rows, cols)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


@pytest.mark.parametrize("rows,cap,cols", [(150, 4, 128), (1000, 0, 128), (255, 5, 77), (12288, 0, 128), (3, 0, 33),
                                           (200, 0, 17)])
def test_max_balanced(m, monkeypatch, rows, cap, cols):
    """the standalone row max on the balanced plan (k_max with one range per CTA) = the 32-row tiles and
    the oracle"""
    if cap:
        monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    c, o = ctx(m, 2, 33)
    x = workloads.softmax_inputs(rows, cols)
    gx = c.share(torch.from_numpy(x).cuda())
    s0 = c.step
    a = c.max(gx, rows, cols, row_off=32)
    monkeypatch.setenv("MPC_MAX_BAL", "0")
    c.set_step(s0, force=True)
    b = c.max(gx, rows, cols, row_off=32)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    if rows <= 1000:
        same(a, o.max(o.share(x), rows, cols, row_off=32))


@pytest.mark.parametrize("rows,cap,cols", [(1000, 4, 128), (777, 3, 77), (32768, 0, 128), (5000, 8, 2)])
def test_balanced_rounds(m, monkeypatch, rows, cap, cols):
    """more than 64 rows per CTA: k equal rounds of ranges per CTA (nrange = k x grid), softmax and the
    standalone max; equal to the 32-row tiles and (small cases) the oracle"""
    if cap:
        monkeypatch.setenv("MPC_ROW_GRID_CAP", str(cap))
    c, o = ctx(m, 2, 35)
    x = workloads.softmax_inputs(rows, cols)
    gx = c.share(torch.from_numpy(x).cuda())
    s0 = c.step
    a = c.softmax(gx, rows, cols, row_off=32)
    am = c.max(gx, rows, cols, row_off=32)
    monkeypatch.setenv("MPC_SOFTMAX_BAL", "0")
    monkeypatch.setenv("MPC_MAX_BAL", "0")
    c.set_step(s0, force=True)
    b = c.softmax(gx, rows, cols, row_off=32)
    bm = c.max(gx, rows, cols, row_off=32)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    assert torch.equal(am[0], bm[0]) and torch.equal(am[1], bm[1])
    if rows <= 1000:
        ox = o.share(x)
        same(a, o.softmax(ox, rows, cols, row_off=32))
