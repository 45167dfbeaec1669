"""Oracle pins for the causal softmax variant (reading R24c): rows are the
T x T score blocks of causal attention (T = cols), global row g attends to columns j <= g mod T.

Pinned against: the float causal softmax written with -inf masking (a different definition of
the same function), exact zeros in the masked outputs, bit-identity with the dense softmax on
rows whose position is T - 1 (nothing masked) and for T = 1, and the one-entry rows (position 0)
reconstructing to 1 within the Newton-Raphson tolerance.
"""
import numpy as np
import pytest

import workloads
from oracle import Oracle

ULP = 2.0 ** -16


def O(step=0):
    return Oracle.for_cfg(workloads.keys(5), step)


def dec(s):
    return Oracle.open(*s)[1]


def causal_mask(rows, cols, row_off):
    pos = (row_off + np.arange(rows)) % cols
    return np.arange(cols)[None, :] > pos[:, None]


def float_causal_softmax(x, mask):
    z = np.where(mask, -np.inf, x)
    z = z - z.max(axis=1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=1, keepdims=True)


@pytest.mark.parametrize("rows,cols,row_off", [(64, 64, 0), (80, 40, 32), (96, 128, 64)])
def test_causal_softmax_vs_float(rows, cols, row_off):
    o = O()
    s = o.share(workloads.softmax_inputs(rows, cols, seed_cfg=5))
    xd = dec(s).reshape(rows, cols)
    z = o.softmax(s, rows, cols, row_off=row_off, causal=1)
    mask = causal_mask(rows, cols, row_off)
    y = dec(z).reshape(rows, cols)
    assert np.max(np.abs(y - float_causal_softmax(xd, mask))) <= 1.1e-2
    # masked outputs are the public zero: both shares exactly 0
    z0, z1 = (np.asarray(p).reshape(rows, cols) for p in z)
    assert not np.any(z0[mask]) and not np.any(z1[mask])
    assert np.max(np.abs(y.sum(1) - 1)) <= 3e-2


def test_causal_last_position_rows_equal_dense():
    rows, cols, row_off = 96, 32, 32
    x = workloads.softmax_inputs(rows, cols, seed_cfg=5)
    o = O(3)
    s = o.share(x)
    a = O(4).softmax(s, rows, cols, row_off=row_off, causal=1)
    b = O(4).softmax(s, rows, cols, row_off=row_off)
    full = (row_off + np.arange(rows)) % cols == cols - 1          # nothing masked
    a0, a1, b0, b1 = (np.asarray(p).reshape(rows, cols) for p in (*a, *b))
    assert full.sum() == 3
    assert np.array_equal(a0[full], b0[full]) and np.array_equal(a1[full], b1[full])
    assert not np.array_equal(a0[~full], b0[~full])


def test_causal_one_column_equals_dense():
    rows = 70
    x = workloads.softmax_inputs(rows, 1, seed_cfg=5)
    o = O()
    s = o.share(x)
    a = O(2).softmax(s, rows, 1, row_off=32, causal=1)
    b = O(2).softmax(s, rows, 1, row_off=32)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_causal_first_position_is_one():
    rows, cols = 64, 48
    o = O()
    s = o.share(workloads.softmax_inputs(rows, cols, seed_cfg=5) * 3)
    y = dec(o.softmax(s, rows, cols, row_off=0, causal=1)).reshape(rows, cols)
    first = np.arange(rows) % cols == 0
    assert np.all(np.abs(y[first, 0] - 1.0) <= 1e-2)
    assert np.all(y[first, 1:] == 0.0)


def test_causal_same_steps_as_dense():
    rows, cols = 40, 24
    o1, o2 = O(7), O(7)
    s = O().share(workloads.softmax_inputs(rows, cols, seed_cfg=5))
    o1.softmax(s, rows, cols, causal=1)
    o2.softmax(s, rows, cols)
    assert o1.step == o2.step
