"""Pins for the oracle's SURVEY §8(f) NEXT #2 variants beyond square-pair triples:
the broadcast triple (softmax's / layernorm's e * bcast(r) with one opening of r per row,
DESIGN.md 2.8) and power-basis polynomials.

Broadcast triple: the product must be the exact wrapping ring product x_ij * y_i for
ANY sharing (closed form, Python big ints), keyed by global element / row units (shard
invariance), one step per call.  Power basis: the polynomial value within the fixed-
point bound derived below, exact outside the segment, same step count as Horner.
"""
import json
import os

import numpy as np
import pytest

import workloads
from oracle import Oracle, encode
from oracle import float_ref as fr

COEFFS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "fixtures",
                                     "coeffs.json")))["fits"]
ULP = 2.0 ** -16
M64 = (1 << 64) - 1


def O(cfg=1, step=0):
    return Oracle.for_cfg(workloads.keys(cfg), step)


def dec(s):
    return Oracle.open(*s)[1]


def ring(s):
    return Oracle.open(*s)[0].view(np.int64)


def rand_shares(vals, seed):
    g = np.random.default_rng(seed)
    r = g.integers(0, 2**64, len(vals), dtype=np.uint64, endpoint=False)
    v = np.array([v & M64 for v in vals], dtype=np.uint64)
    return v - r, r


def rec(s):
    return [int(a) + int(b) & M64 for a, b in zip(s[0], s[1])]


# ------------------------------------------------------------ broadcast triple ----
def test_mul_bcast_is_wrapping_product():
    rows, cols = 7, 13
    g = np.random.default_rng(11)
    xv = [int(v) for v in g.integers(0, 2**64, rows * cols, dtype=np.uint64, endpoint=False)]
    yv = [int(v) for v in g.integers(0, 2**64, rows, dtype=np.uint64, endpoint=False)]
    o = O(5, step=3)
    z = o.mul_bcast(rand_shares(xv, 1), rand_shares(yv, 2), rows, cols, off=64, row_off=5)
    assert rec(z) == [(xv[i] * yv[i // cols]) & M64 for i in range(rows * cols)]
    assert o.step == 4


def test_mul_bcast_edge_values_and_trunc():
    # 1.0 * 1.0 (S:438's example at scale 2^16) and -1.5 * 2.0, truncated by 16
    o = O()
    y = rand_shares([encode(1.0), encode(2.0)], 5)
    x4 = rand_shares([encode(1.0), encode(-1.5) & M64, encode(2.25), encode(0.5)], 4)
    z = o.mul_bcast(x4, y, 2, 2, trunc_bits=16)
    got = ring(z)
    want = np.array([1.0, -1.5, 4.5, 1.0]) * 65536
    assert np.all((got == want) | (got == want - 1))


def test_mul_bcast_shard_invariance():
    # one call over 64 rows == two calls over rows [0,32) and [32,64) with their offsets
    rows, cols = 64, 10
    x = rand_shares(list(range(1, rows * cols + 1)), 7)
    y = rand_shares([3 * r + 1 for r in range(rows)], 8)
    full = O(2, 9).mul_bcast(x, y, rows, cols, off=320, row_off=32)
    h = rows // 2 * cols
    a = O(2, 9).mul_bcast((x[0][:h], x[1][:h]), (y[0][:32], y[1][:32]), 32, cols, off=320, row_off=32)
    b = O(2, 9).mul_bcast((x[0][h:], x[1][h:]), (y[0][32:], y[1][32:]), 32, cols, off=320 + h, row_off=64)
    assert np.array_equal(full[0], np.concatenate([a[0], b[0]]))
    assert np.array_equal(full[1], np.concatenate([a[1], b[1]]))


def test_mul_bcast_differs_from_expanded_triple_but_same_value():
    # a different protocol (its own output shares), the same reconstruction
    rows, cols = 4, 8
    x = rand_shares([5 * i + 3 for i in range(rows * cols)], 12)
    y = rand_shares([7, 11, 13, 17], 13)
    yb = (np.repeat(y[0], cols), np.repeat(y[1], cols))
    zb = O(1, 2).mul_bcast(x, y, rows, cols)
    ze = O(1, 2).mul(x, yb)
    assert rec(zb) == rec(ze)
    assert not np.array_equal(zb[0], ze[0])


@pytest.mark.parametrize("rows,cols,tol_true", [(64, 128, 1.1e-2), (32, 1024, 2.6e-2)])
def test_softmax_bcast(rows, cols, tol_true):
    o = O(2)
    s = o.share(workloads.softmax_inputs(rows, cols))
    xd = dec(s).reshape(rows, cols)
    y = dec(o.softmax(s, rows, cols, bcast=1)).reshape(rows, cols)
    assert np.max(np.abs(y - fr.softmax_formula(xd))) <= 2 * 4 * 256 * ULP + 8 * ULP
    assert np.max(np.abs(y - fr.softmax(xd))) <= tol_true
    # same step ids as the expanded product (one step), different output shares
    o2 = O(2)
    s2 = o2.share(workloads.softmax_inputs(rows, cols))
    o2.softmax(s2, rows, cols)
    assert o2.step == o.step


def test_softmax_bcast_golden_and_shift_invariance():
    o = O(2)
    y = dec(o.softmax(o.share([[0.0, 0.0]]), 1, 2, bcast=1))
    assert np.max(np.abs(y - 0.5)) <= 1e-2
    rows, cols = 32, 64
    s = O(2).share(workloads.softmax_inputs(rows, cols))
    a = O(2, 100).softmax(s, rows, cols, bcast=1)
    c = np.uint64(encode(-2.5) & M64)
    b = O(2, 100).softmax((s[0] + c, s[1]), rows, cols, bcast=1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_layernorm_bcast():
    rows, cols = 64, 768
    o = O(5)
    s = o.share(workloads.layernorm_inputs(rows, cols))
    xd = dec(s).reshape(rows, cols)
    y = dec(o.layernorm(s, rows, cols, bcast=1)).reshape(rows, cols)
    assert np.max(np.abs(y - fr.layernorm_formula(xd))) <= 2e-3
    assert np.max(np.abs(y - fr.layernorm(xd))) <= 1.3e-2


# ---------------------------------------------------------------- power basis ----
def power_tol(v, c, d, abs_form):
    """Fixed-point bound of POWER: v2 = MT(v,v) errs by <= 2 ulp, v3 = MT(v2,v)
    by |v| * 2 + 2, v4 = MT(v2,v2) by 2 |v2| * 2 + 2; pmulF(v^k, c_k) adds |c_k| err_k +
    1 (its truncation) + 0.5 |v|^k (E(c_k) rounding); + 1 for addP's encoding of c_0,
    + 2 for the |x|-form's 0.5 x term and the masked sum's truncation-free products."""
    v = np.abs(v)
    err = {1: 0.0, 2: 2.0, 3: 2.0 * v + 2.0, 4: 4.0 * v * v + 2.0}
    t = np.ones_like(v) * (1.0 + (2.0 if abs_form else 0.0))
    for k in range(1, d + 1):
        t = t + abs(c[k]) * err[k] + 1.0 + 0.5 * v ** k
    return t * ULP


@pytest.mark.parametrize("fit", [f for f in COEFFS if f["form"] in ("poly_x", "poly_abs") and f["degree"] >= 1],
                         ids=lambda f: f"{f['op']}-{f['form']}-{f['degree']}")
def test_power_basis_vs_formula_and_true(fit):
    o = O()
    B, d, c = fit["interval"][1], fit["degree"], fit["coefficients"]
    s = o.share(workloads.act_inputs(4096))
    xd = dec(s)
    y = dec(o.act(s, fit["op"], fit["form"], d, B, c, basis=1))
    f = fr.act_formula(xd, fit["op"], fit["form"], d, B, c)
    v = np.abs(xd) if fit["form"] == "poly_abs" else xd
    mid = (xd >= -B) & (xd < B)
    assert np.all(np.abs(y - f)[mid] <= power_tol(v, c, d, fit["form"] == "poly_abs")[mid])
    true = fr.TRUE_ACT[fit["op"]](xd)
    assert np.max(np.abs(y - true)) <= fit["max_abs_error"] + np.max(power_tol(np.array([B]), c, d, True))
    # outside [-B, B) exact, as for Horner
    xr, yr = ring(s), ring(o.act(s, fit["op"], fit["form"], d, B, c, basis=1))
    hi, lo = xd >= B + 1e-3, xd < -B - 1e-3
    top = 65536 if fit["op"] == "sigmoid" else xr[hi]
    assert np.all(yr[hi] == top) and np.all(yr[lo] == 0)


def test_power_basis_steps_and_degree1():
    fit = [f for f in COEFFS if f["op"] == "gelu" and f["form"] == "poly_x" and f["degree"] == 4][0]
    x = workloads.act_inputs(256)
    oh, op = O(), O()
    sh, sp = oh.share(x), op.share(x)
    oh.act(sh, "gelu", "poly_x", 4, fit["interval"][1], fit["coefficients"])
    op.act(sp, "gelu", "poly_x", 4, fit["interval"][1], fit["coefficients"], basis=1)
    assert oh.step == op.step                                  # d-1 product steps either way
    # degree 1: POWER and HORNER are the same arithmetic (h = addP(pmulF(v, c1), c0))
    c1 = [0.25, 0.5]
    a = O(1, 5).act(sh, "gelu", "poly_x", 1, 5.0, c1)
    b = O(1, 5).act(sh, "gelu", "poly_x", 1, 5.0, c1, basis=1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_power_basis_brute_force_small_ring_values():
    # every fixed-point input on a coarse grid of [-4, 4): the power-basis quartic
    # matches the exact rational polynomial of the ENCODED input within the bound
    c = [0.1, -0.2, 0.3, -0.05, 0.01]
    xs = np.arange(-4.0, 4.0, 1.0 / 64)
    o = O()
    s = o.share(xs)
    y = dec(o.act(s, "gelu", "poly_x", 4, 1000.0, c, basis=1))
    xd = dec(s)
    exact = sum(ck * xd ** k for k, ck in enumerate(c))
    assert np.all(np.abs(y - exact) <= power_tol(xd, c, 4, False))
