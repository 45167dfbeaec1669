"""The sliced all-cores oracle runs (tests/oracle_pool.py) reproduce the whole-array oracle
exactly: the PRG is keyed by global unit, so 32-aligned row / element / image
slices with their global offsets are the unsharded op.  This is what lets the GPU parity tests
compare every share of the full BASELINE-size configs."""
import numpy as np

import workloads
from oracle import Oracle
import oracle_pool as op


def test_rows_op_softmax_layernorm_max():
    keys = workloads.keys(2)
    rows, cols = 160, 40
    o = Oracle.for_cfg(keys, 7)
    x = o.share(workloads.softmax_inputs(rows, cols))
    for name, kw in (("softmax", {}), ("layernorm", dict(mean_mode=1)), ("max", {}), ("softmax", dict(causal=1))):
        ref = getattr(Oracle.for_cfg(keys, 7), name)(x, rows, cols, row_off=64, **kw)
        got = op.rows_op(name, keys, 7, x, rows, cols, row_off=64, block=32, nproc=3, **kw)
        assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1]), name


def test_elems_op_relu_act():
    keys = workloads.keys(3)
    n = 1000
    o = Oracle.for_cfg(keys, 3)
    x = o.share(workloads.act_inputs(n))
    ref = Oracle.for_cfg(keys, 3).relu(x, off=96)
    got = op.elems_op("relu", keys, 3, x, n, off=96, block=64, nproc=3)
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])
    ref = Oracle.for_cfg(keys, 3).act(x, "gelu", "erf", 1, 2.5, None, 8, off=32)
    got = op.elems_op("act", keys, 3, x, n, off=32, block=96, nproc=2, act="gelu", form="erf", degree=1, B=2.5,
                      erf_terms=8)
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])


def test_maxpool_op_by_image():
    keys = workloads.keys(4)
    N, C, H, W = 3, 2, 8, 8        # C * 4 * 4 = 32 outputs per image: image offsets stay 32-aligned
    o = Oracle.for_cfg(keys, 5)
    x = o.share(workloads.maxpool_inputs((N, C, H, W)))
    ref = Oracle.for_cfg(keys, 5).maxpool2d(x, N, C, H, W, img_off=2)
    got = op.maxpool_op(keys, 5, x, N, C, H, W, img_off=2, nproc=2)
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])
