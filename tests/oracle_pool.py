"""Whole-array oracle runs on every host core (test infrastructure; imports oracle/ only).

The PRG is keyed by global unit, so an op over rows [r0, r1) with row_off = r0
(or elements [e0, e1) with off = e0, or images [i0, i1) with img_off = i0) reproduces exactly
that slice of the unsharded op.  These helpers split a full BASELINE-size input into such slices,
run the plain-C oracle on them in a fork pool (one process per core; the input arrays are shared
copy-on-write) and concatenate the output shares -- so the GPU parity tests compare EVERY share of
the full-size configs, not samples."""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

from oracle import Oracle

_G: dict = {}


def cores() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


def _work(task):
    kind, a, b = task
    g = _G
    o = Oracle.for_cfg(g["keys"], g["step"])
    x0, x1, kw = g["x0"], g["x1"], g["kw"]
    if kind == "rows":
        C = g["cols"]
        z = getattr(o, g["op"])((x0[a * C:b * C], x1[a * C:b * C]), b - a, C, row_off=g["row_off"] + a, **kw)
    elif kind == "elems":
        z = getattr(o, g["op"])((x0[a:b], x1[a:b]), off=g["off"] + a, **kw)
    else:                                            # images of an NCHW maxpool
        C, H, W = g["chw"]
        per = C * H * W
        z = o.maxpool2d((x0[a * per:b * per], x1[a * per:b * per]), b - a, C, H, W, img_off=g["img_off"] + a, **kw)
    return a, z[0], z[1]


def _run(tasks, nproc):
    nproc = min(nproc or cores(), len(tasks))
    if nproc <= 1:
        res = [_work(t) for t in tasks]
    else:
        with mp.get_context("fork").Pool(nproc) as pool:
            res = pool.map(_work, tasks, chunksize=1)
    res.sort(key=lambda r: r[0])
    return np.concatenate([r[1] for r in res]), np.concatenate([r[2] for r in res])


def rows_op(op, keys, step, x, rows, cols, row_off=0, block=None, nproc=None, **kw):
    """op in {softmax, layernorm, max}: the whole rows x cols op, sliced in 32-row-aligned blocks."""
    _G.clear()
    _G.update(keys=keys, step=step, x0=np.ascontiguousarray(x[0]), x1=np.ascontiguousarray(x[1]), kw=kw, op=op,
              cols=cols, row_off=row_off)
    n = nproc or cores()
    block = block or max(32, ((rows + 4 * n - 1) // (4 * n) + 31) // 32 * 32)
    return _run([("rows", a, min(rows, a + block)) for a in range(0, rows, block)], n)


def elems_op(op, keys, step, x, n, off=0, block=None, nproc=None, **kw):
    """element-wise op (relu, act, exp, ...) over n elements, sliced in 32-aligned blocks."""
    _G.clear()
    _G.update(keys=keys, step=step, x0=np.ascontiguousarray(x[0]), x1=np.ascontiguousarray(x[1]), kw=kw, op=op,
              off=off)
    p = nproc or cores()
    block = block or max(32, ((n + 4 * p - 1) // (4 * p) + 31) // 32 * 32)
    return _run([("elems", a, min(n, a + block)) for a in range(0, n, block)], p)


def maxpool_op(keys, step, x, N, C, H, W, img_off=0, nproc=None, **kw):
    """maxpool2d over N images, one image per task (C*Ho*Wo output rows per image; img_off must
    keep the global output row offset a multiple of 32, as the op requires)."""
    _G.clear()
    _G.update(keys=keys, step=step, x0=np.ascontiguousarray(x[0]), x1=np.ascontiguousarray(x[1]), kw=kw,
              chw=(C, H, W), img_off=img_off)
    return _run([("pool", a, a + 1) for a in range(N)], nproc)
