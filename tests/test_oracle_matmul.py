"""Pins for the oracle's Beaver matrix multiplication over Z_2^64 (SURVEY §8(f) NEXT #3,
DESIGN.md 2.10): for ANY sharing the reconstruction is the exact wrapping ring product
rec(X) @ rec(Y) mod 2^64 (computed here with Python integers, the definition of the ring
product); units are global (batch shard invariance); truncation within one ulp of the
floor; fixed-point encodings decode to the float matmul within the truncation bound."""
import numpy as np
import pytest

import workloads
from oracle import Oracle, encode

M64 = (1 << 64) - 1


def O(cfg=1, step=0):
    return Oracle.for_cfg(workloads.keys(cfg), step)


def shares(vals, seed):
    g = np.random.default_rng(seed)
    v = np.array([int(x) & M64 for x in vals], dtype=np.uint64)
    r = g.integers(0, 2**64, v.size, dtype=np.uint64, endpoint=False)
    return v - r, r


def rec(s):
    return [(int(a) + int(b)) & M64 for a, b in zip(s[0], s[1])]


def ring_matmul(X, Y, M, K, N):
    return [sum(X[m * K + k] * Y[k * N + n] for k in range(K)) & M64 for m in range(M) for n in range(N)]


@pytest.mark.parametrize("batch,M,K,N", [(1, 1, 1, 1), (1, 3, 5, 4), (2, 7, 9, 3), (3, 2, 16, 5)])
def test_matmul_is_wrapping_ring_product(batch, M, K, N):
    g = np.random.default_rng(100 + M * K * N)
    X = [int(v) for v in g.integers(0, 2**64, batch * M * K, dtype=np.uint64, endpoint=False)]
    Y = [int(v) for v in g.integers(0, 2**64, batch * K * N, dtype=np.uint64, endpoint=False)]
    o = O(2, step=5)
    z = o.matmul(shares(X, 1), shares(Y, 2), batch, M, K, N, batch_off=3)
    want = []
    for b in range(batch):
        want += ring_matmul(X[b * M * K:(b + 1) * M * K], Y[b * K * N:(b + 1) * K * N], M, K, N)
    assert rec(z) == want
    assert o.step == 6


def test_matmul_batch_shard_invariance():
    batch, M, K, N = 4, 3, 6, 2
    X = shares(list(range(1, batch * M * K + 1)), 3)
    Y = shares([7 * i + 1 for i in range(batch * K * N)], 4)
    full = O(1, 9).matmul(X, Y, batch, M, K, N, batch_off=10)
    h, hk = 2 * M * K, 2 * K * N
    a = O(1, 9).matmul((X[0][:h], X[1][:h]), (Y[0][:hk], Y[1][:hk]), 2, M, K, N, batch_off=10)
    b = O(1, 9).matmul((X[0][h:], X[1][h:]), (Y[0][hk:], Y[1][hk:]), 2, M, K, N, batch_off=12)
    assert np.array_equal(full[0], np.concatenate([a[0], b[0]]))
    assert np.array_equal(full[1], np.concatenate([a[1], b[1]]))


def test_matmul_shares_depend_on_step_and_offset_not_value():
    X = shares([1, 2, 3, 4], 5)
    Y = shares([5, 6, 7, 8], 6)
    a = O(1, 1).matmul(X, Y, 1, 2, 2, 2)
    b = O(1, 2).matmul(X, Y, 1, 2, 2, 2)
    c = O(1, 1).matmul(X, Y, 1, 2, 2, 2, batch_off=1)
    assert rec(a) == rec(b) == rec(c) == [19, 22, 43, 50]
    assert not np.array_equal(a[0], b[0]) and not np.array_equal(a[0], c[0])


def test_matmul_fixed_point_and_truncation():
    # encoded floats: the truncated product decodes to the float matmul of the encodings within 2 ulp
    M, K, N = 5, 12, 4
    g = np.random.default_rng(7)
    xf = g.uniform(-3, 3, (M, K))
    yf = g.uniform(-3, 3, (K, N))
    o = O(3)
    X, Y = o.share(xf), o.share(yf)
    zt = o.matmul(X, Y, 1, M, K, N, trunc_bits=16)
    xd = Oracle.open(*X)[1].reshape(M, K)
    yd = Oracle.open(*Y)[1].reshape(K, N)
    got = Oracle.open(*zt)[1].reshape(M, N)
    assert np.max(np.abs(got - xd @ yd)) <= 2 * 2.0 ** -16        # floor, or floor - 1 (share wrap)
    # exact: the untruncated product is the exact ring product of the encodings
    z = O(3, 1).matmul(X, Y, 1, M, K, N)
    ex = np.array(ring_matmul(rec(X), rec(Y), M, K, N), dtype=np.uint64)
    assert np.array_equal(Oracle.open(*z)[0], ex)
    t = Oracle.open(*O(3, 1).matmul(X, Y, 1, M, K, N, trunc_bits=16))[0].view(np.int64)
    fl = ex.view(np.int64) >> 16
    assert np.all((t == fl) | (t == fl - 1))


def test_matmul_identity_and_zero():
    M = 4
    eye = [encode(1.0) if i == j else 0 for i in range(M) for j in range(M)]
    Yv = [encode(v) & M64 for v in np.linspace(-2, 2, M * 3)]
    o = O()
    z = o.matmul(shares(eye, 8), shares(Yv, 9), 1, M, M, 3, trunc_bits=16)
    r = np.array(rec(z), dtype=np.uint64).view(np.int64)
    want = np.array(Yv, dtype=np.uint64).view(np.int64)
    assert np.all((r == want) | (r == want - 1))
    z0 = O().matmul(shares([0] * 6, 1), shares([5] * 6, 2), 1, 2, 3, 2)
    assert rec(z0) == [0, 0, 0, 0]
