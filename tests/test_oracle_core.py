"""Pins for the oracle's PRG, share algebra, Beaver, truncation and LTZ.

Each test checks the oracle against something other than itself: published
known-answer vectors, Python big-integer arithmetic (closed forms), brute force
over small ranges, printed SPEC/PAPER values (tests/golden/spec_examples.json),
and statistical properties the paper states.
"""
import json
import os

import numpy as np
import pytest

import workloads
from oracle import Oracle, encode, ltz_gate_count, philox, trunc_wrap_trials

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
M64 = (1 << 64) - 1
KEYS = workloads.keys(1)


def O(step=0):
    return Oracle.for_cfg(KEYS, step)


def shares_of(vals, seed=7):
    """Arbitrary sharings of given ring values: x0 uniform, x1 = v - x0 (mod 2^64)."""
    vals = [int(v) & M64 for v in vals]
    g = np.random.default_rng(seed)
    x0 = g.integers(0, 2**64, len(vals), dtype=np.uint64, endpoint=False)
    x1 = np.array([(v - int(a)) & M64 for v, a in zip(vals, x0)], dtype=np.uint64)
    return x0, x1


def rec(s):
    return [(int(a) + int(b)) & M64 for a, b in zip(s[0], s[1])]


def signed(v):
    v &= M64
    return v - (1 << 64) if v >> 63 else v


# ---------------------------------------------------------------- Philox ----
@pytest.mark.parametrize("vec", GOLD["philox4x32_10_kat"]["vectors"])
def test_philox_kat(vec):
    ctr = [int(h, 16) for h in vec["ctr"]]
    key = [int(h, 16) for h in vec["key"]]
    assert philox(ctr, key) == tuple(int(h, 16) for h in vec["out"])


# ---------------------------------------------------------- share / open ----
def test_encode_examples():
    assert encode(GOLD["encode_1p5"]["x"]) == GOLD["encode_1p5"]["ring"]
    # round-half-even (reading R2) vs Python's round(), an independent implementation
    for c in [0.5 / 65536, 1.5 / 65536, -2.5 / 65536, 1e-5, -3.14159, 12345.678, 2.0**30]:
        assert encode(c) == round(c * 65536)


def test_share_reconstructs_exactly():
    x = workloads.rng(1, 99).uniform(-2.0**31, 2.0**31, 10_000)
    o = O()
    s = o.share(x, owner=0)
    assert rec(s) == [round(v * 65536) & M64 for v in x]
    s1 = o.share(x, owner=1)
    assert rec(s1) == [round(v * 65536) & M64 for v in x]
    assert o.step == 2
    # the non-owner's share is the mask r, which differs between steps
    assert not np.array_equal(s[1], s1[0])


def test_open_decode():
    s = shares_of([98304, (-98304) & M64, 1])
    ring, f = Oracle.open(*s)
    assert list(ring) == [98304, (-98304) & M64, 1]
    assert list(f) == [1.5, -1.5, 1.0 / 65536]


# --------------------------------------------------------------- Beaver ----
def test_beaver_is_wrapping_product():
    g = np.random.default_rng(3)
    xv = [int(v) for v in g.integers(0, 2**64, 1000, dtype=np.uint64, endpoint=False)]
    yv = [int(v) for v in g.integers(0, 2**64, 1000, dtype=np.uint64, endpoint=False)]
    o = O(5)
    z = o.mul(shares_of(xv, 1), shares_of(yv, 2), off=64)
    assert rec(z) == [(a * b) & M64 for a, b in zip(xv, yv)]
    assert o.step == 6


def test_beaver_one_times_one():
    gb = GOLD["beaver_one_times_one"]
    o = O()
    z = o.mul(shares_of([gb["x"]]), shares_of([gb["y"]], 3))
    assert rec(z) == [gb["product"]]
    zt = Oracle.trunc(z, 16)
    assert rec(zt)[0] in (gb["trunc"], gb["trunc"] - 1)


def test_beaver_output_depends_on_unit_and_step():
    o = O()
    x, y = shares_of([5, 6, 7, 8]), shares_of([1, 2, 3, 4], 9)
    a = o.mul(x, y)
    o.step = 0
    b = o.mul(x, y)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])  # deterministic
    c = o.mul(x, y)                                                    # next step
    assert not np.array_equal(a[0], c[0])
    o.step = 0
    d = o.mul(x, y, off=2)                                             # other units
    assert not np.array_equal(a[0], d[0])
    assert rec(a) == rec(c) == rec(d)


# ----------------------------------------------------------- truncation ----
def test_trunc_examples():
    o = O()
    s = o.share([GOLD["trunc_1p5"]["x"]])
    z = Oracle.trunc(s, 16)
    assert signed(rec(z)[0]) in GOLD["trunc_1p5"]["ok"]


def test_trunc_floor_or_floor_minus_one():
    g = np.random.default_rng(11)
    xs = [int(v) for v in g.integers(-2**40, 2**40, 5000)]
    s = shares_of(xs, 4)
    for k in (1, 8, 16):
        z = Oracle.trunc(s, k)
        for v, r in zip(xs, rec(z)):
            assert signed(r) in (v >> k, (v >> k) - 1)


def test_trunc_small_ring_wrap_rate():
    gd = GOLD["trunc_small_ring"]
    bad = trunc_wrap_trials(gd["N"], gd["k"], gd["x"], gd["trials"])
    rate = bad / gd["trials"]
    assert abs(rate - gd["rate"]) <= gd["tol"], rate
    bad = trunc_wrap_trials(gd["N"], gd["k"], -gd["x"], gd["trials"])
    assert abs(bad / gd["trials"] - gd["rate"]) <= gd["tol"]


def test_trunc_no_wraps_at_64():
    # no wraps in 10^6 trials for |x| <= 2^32 at N = 64 (probability ~2^-32)
    assert trunc_wrap_trials(64, 16, 2**32, 1_000_000) == 0
    assert trunc_wrap_trials(64, 16, -2**32, 1_000_000) == 0


# ------------------------------------------------------------------ LTZ ----
def test_ltz_examples():
    ge = GOLD["ltz_examples"]
    for w in (64, 33):
        z = O().ltz(shares_of([v * 65536 for v in ge["x"]]), window=w)
        assert rec(z) == ge["ltz"]


def test_ltz_random_w64_matches_sign():
    g = np.random.default_rng(21)
    xs = [int(v) for v in g.integers(0, 2**64, 10_000, dtype=np.uint64, endpoint=False)]
    z = O(3).ltz(shares_of(xs, 5), off=0, window=64)
    assert rec(z) == [v >> 63 for v in xs]


def test_ltz_window33_correct_inside_window():
    g = np.random.default_rng(22)
    xs = [int(v) for v in g.integers(-2**32, 2**32, 4096)]
    xs += [-2**32, 2**32 - 1, -1, 0, 1]
    z = O().ltz(shares_of(xs, 6), window=33)
    assert rec(z) == [1 if v < 0 else 0 for v in xs]


def test_ltz_is_bit_w_minus_1_for_every_window():
    # brute force of the definition: rec(b) = bit (w-1) of rec(x) for every x, every w
    g = np.random.default_rng(23)
    for w in range(1, 65):
        xs = [int(v) for v in g.integers(0, 2**64, 96, dtype=np.uint64, endpoint=False)]
        z = O(w).ltz(shares_of(xs, w), off=32 * w, window=w)
        assert rec(z) == [(v >> (w - 1)) & 1 for v in xs], w


@pytest.mark.parametrize("w", [13, 33, 64])
def test_ltz_brute_force_small_range(w):
    xs = list(range(-2**12, 2**12))
    z = O().ltz(shares_of(xs, 8), window=w)
    assert rec(z) == [1 if v < 0 else 0 for v in xs]


def test_ltz_edge_sharings():
    # edge shares: one share zero, shares near 2^63, all-ones
    vals, x0s = [], []
    for v in [0, 1, -1, 2**31, -2**31, 2**32 - 1, -2**32]:
        for a in [0, 1, M64, 1 << 63, (1 << 63) - 1, 1 << 32, v & M64]:
            vals.append(v & M64); x0s.append(a)
    x0 = np.array(x0s, dtype=np.uint64)
    x1 = np.array([(v - a) & M64 for v, a in zip(vals, x0s)], dtype=np.uint64)
    for w in (33, 64):
        z = O().ltz((x0, x1), window=w)
        assert rec(z) == [(v >> (w - 1)) & 1 for v in vals]


def test_ltz_gate_counts_and_byte_ratio():
    g = GOLD["ltz_gate_counts"]
    assert ltz_gate_count(33) == g["w33"]
    assert ltz_gate_count(64) == g["w64"]
    # bytes per element per party: (2 G(w) + 1) bits  (2 words per gate + 1 B2A bit)
    ratio = (2 * ltz_gate_count(33) + 1) / (2 * ltz_gate_count(64) + 1)
    assert abs(ratio / g["spec_ratio"] - 1) <= 0.05


def test_relu_exact():
    xs = list(range(-3000, 3000, 7)) + [2**31, -2**31]
    z = O().relu(shares_of(xs, 9), window=33)
    assert [signed(v) for v in rec(z)] == [max(v, 0) for v in xs]


def test_relu_is_ltz_then_mul():
    # fused = composed: relu uses steps (s: LTZ, s+1: BM(x, 1 - ltz))
    xs = list(range(-100, 100))
    x = shares_of(xs, 10)
    a = O(40).relu(x, off=32)
    o = O(40)
    l0, l1 = o.ltz(x, off=32)
    nl = ((1 - l0.astype(object)) & M64).astype(np.uint64), ((-l1.astype(object)) & M64).astype(np.uint64)
    b = o.mul(x, nl, off=32)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_shard_invariance_ltz_and_mul():
    xs = [int(v) for v in np.random.default_rng(5).integers(-2**30, 2**30, 256)]
    x = shares_of(xs, 11)
    full = O(7).ltz(x, off=0)
    lo = O(7).ltz((x[0][:128], x[1][:128]), off=0)
    hi = O(7).ltz((x[0][128:], x[1][128:]), off=128)
    assert np.array_equal(full[0], np.concatenate([lo[0], hi[0]]))
    assert np.array_equal(full[1], np.concatenate([lo[1], hi[1]]))
    fm = O(7).mul(x, x)
    hm = O(7).mul((x[0][100:], x[1][100:]), (x[0][100:], x[1][100:]), off=100)
    assert np.array_equal(fm[0][100:], hm[0]) and np.array_equal(fm[1][100:], hm[1])


# ------------------------------------------------ square-pair triples (NEXT #2) ----
def test_square_is_wrapping_square():
    g = np.random.default_rng(31)
    xv = [int(v) for v in g.integers(0, 2**64, 1000, dtype=np.uint64, endpoint=False)]
    o = O(9)
    z = o.square(shares_of(xv, 12), off=5)
    assert rec(z) == [(a * a) & M64 for a in xv]
    assert o.step == 10
    # differs from the Beaver product's shares (different triple) but reconstructs the same
    zb = O(9).mul(shares_of(xv, 12), shares_of(xv, 12), off=5)
    assert rec(zb) == rec(z) and not np.array_equal(zb[0], z[0])
