"""Host logic of bench.py's CPU baselines (no GPU): the all-cores oracle timing splits cfg2 into
32-row-aligned slices whose results are exactly the whole op (PRG keyed by global row), and the
process pool returns one wall time per repetition."""
import os
import sys

import numpy as np

import workloads
from oracle import Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_row_slices_reproduce_the_whole_softmax():
    rows, cols = 96, 128
    x = workloads.softmax_inputs(rows, cols)
    keys = workloads.keys(2)
    o = Oracle.for_cfg(keys)
    whole = o.softmax(o.share(x), rows, cols)
    parts = [[], []]
    for a, b in ((0, 32), (32, 96)):
        ob = Oracle.for_cfg(keys)
        z = ob.softmax(ob.share(x[a:b], off=a * cols), b - a, cols, row_off=a)
        for p in (0, 1):
            parts[p].append(np.asarray(z[p]))
    for p in (0, 1):
        assert np.array_equal(np.concatenate(parts[p]), np.asarray(whole[p]))


def test_all_cores_pool_times_each_rep():
    import bench
    dts, used = bench._oracle_softmax_all_cores(128, 2, reps=2)
    assert used == 2 and len(dts) == 2 and all(d > 0 for d in dts)
