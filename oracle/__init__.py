"""CPU oracle for the 2-party nonlinear-operator path (arxiv 2511.19711).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this package.  The product
package paper_2511_19711_b200 never imports it, and it never imports the
product package.  The arithmetic lives in oracle/oracle.c (plain scalar C,
both parties simulated in lockstep, one schedule step at a time); this module
only builds it with gcc and marshals numpy arrays.  Float references of the
approximation formulas (fp64 numpy) are in oracle/float_ref.py.

Every function is pinned by tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc -O2 (no intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        # -fwrapv: signed int64 arithmetic wraps like the ring Z_2^64 (no UB on overflow)
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fwrapv", "-D_GNU_SOURCE", "-shared", "-fPIC",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None
u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
I64 = ctypes.c_int64
INT = ctypes.c_int
DBL = ctypes.c_double


class _Ctx(ctypes.Structure):
    _fields_ = [("key_share", ctypes.c_uint64), ("key_p0", ctypes.c_uint64),
                ("key_p1", ctypes.c_uint64), ("step", ctypes.c_uint64)]


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        CP = ctypes.POINTER(_Ctx)
        L.orc_philox4x32_10.argtypes = [ctypes.POINTER(ctypes.c_uint32)] * 3
        L.orc_encode.argtypes = [DBL]; L.orc_encode.restype = I64
        L.orc_share.argtypes = [CP, f64p, INT, u64p, u64p, I64, I64]
        L.orc_open.argtypes = [u64p, u64p, I64, ctypes.c_void_p, ctypes.c_void_p, INT]
        L.orc_mul.argtypes = [CP, u64p, u64p, u64p, u64p, u64p, u64p, I64, I64, INT]
        L.orc_trunc.argtypes = [u64p, u64p, u64p, u64p, I64, INT]
        L.orc_ltz.argtypes = [CP, u64p, u64p, u64p, u64p, I64, I64, INT]
        L.orc_relu.argtypes = [CP, u64p, u64p, u64p, u64p, I64, I64, INT]
        L.orc_square.argtypes = [CP, u64p, u64p, u64p, u64p, I64, I64, INT]
        L.orc_exp.argtypes = [CP, u64p, u64p, u64p, u64p, I64, I64, INT, INT, INT, INT]
        L.orc_recip.argtypes = [CP, u64p, u64p, u64p, u64p, I64, I64, INT, INT, INT, INT, INT]
        L.orc_rsqrt.argtypes = [CP, u64p, u64p, u64p, u64p, I64, I64, INT, INT, INT, INT, INT]
        L.orc_act.argtypes = [CP, u64p, u64p, u64p, u64p, I64, I64, INT, INT, INT, DBL,
                              ctypes.c_void_p, INT, INT, INT]
        L.orc_mul_bcast.argtypes = [CP, u64p, u64p, u64p, u64p, u64p, u64p, I64, I64, I64, I64, INT]
        L.orc_matmul.argtypes = [CP, u64p, u64p, u64p, u64p, u64p, u64p, I64, I64, I64, I64, I64, INT]
        L.orc_max.argtypes = [CP, u64p, u64p, u64p, u64p, I64, I64, I64, INT]
        L.orc_maxpool2d.argtypes = [CP, u64p, u64p, u64p, u64p, INT, INT, INT, INT, INT, INT, INT,
                                    I64, INT]
        L.orc_softmax.argtypes = [CP, u64p, u64p, u64p, u64p, I64, I64, I64, INT,
                                  INT, INT, INT, INT, INT, INT, INT, INT, INT, INT, INT]
        L.orc_layernorm.argtypes = [CP, u64p, u64p, u64p, u64p, I64, I64, I64, DBL, INT,
                                    INT, INT, INT, INT, INT, INT]
        L.orc_ltz_gate_count.argtypes = [INT]; L.orc_ltz_gate_count.restype = INT
        L.orc_plain_exp.argtypes = [f64p, f64p, I64, INT, INT, INT]
        L.orc_plain_max.argtypes = [f64p, f64p, I64, I64, INT]
        L.orc_plain_recip.argtypes = [f64p, f64p, I64, INT, INT, INT, INT]
        L.orc_plain_rsqrt.argtypes = [f64p, f64p, I64, INT, INT, INT, INT]
        L.orc_plain_act.argtypes = [f64p, f64p, I64, INT, INT, INT, DBL, ctypes.c_void_p, INT, INT, INT]
        L.orc_plain_softmax.argtypes = [f64p, f64p, I64, I64, INT, INT, INT, INT, INT, INT, INT, INT, INT]
        L.orc_plain_layernorm.argtypes = [f64p, f64p, I64, I64, DBL, INT, INT, INT, INT, INT]
        L.orc_max_levels.argtypes = [I64]; L.orc_max_levels.restype = INT
        L.orc_trunc_wrap_trials.argtypes = [INT, INT, I64, I64, ctypes.c_uint64]
        L.orc_trunc_wrap_trials.restype = I64
        _lib = L
    return _lib


def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return tuple(int(v) for v in o)


def encode(c: float) -> int:
    return int(lib().orc_encode(float(c)))


def ltz_gate_count(w: int) -> int:
    return int(lib().orc_ltz_gate_count(w))


def max_levels(cols: int) -> int:
    return int(lib().orc_max_levels(cols))


def trunc_wrap_trials(N: int, k: int, x: int, trials: int, key: int = 0x7A11) -> int:
    return int(lib().orc_trunc_wrap_trials(N, k, x, trials, key))


def _u(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _pair(n):
    return np.empty(n, np.uint64), np.empty(n, np.uint64)


class Oracle:
    """Lockstep two-party simulator with the same step accounting as mpc_ctx."""

    def __init__(self, key_share: int, key_p0: int, key_p1: int, step: int = 0):
        self.c = _Ctx(key_share, key_p0, key_p1, step)

    @classmethod
    def for_cfg(cls, keys: dict, step: int = 0):
        return cls(keys["key_share"], keys["key_p0"], keys["key_p1"], step)

    @property
    def step(self) -> int:
        return int(self.c.step)

    @step.setter
    def step(self, v: int):
        self.c.step = v

    def share(self, x, owner=0, off=0):
        x = np.ascontiguousarray(x, dtype=np.float64).ravel()
        s0, s1 = _pair(x.size)
        lib().orc_share(ctypes.byref(self.c), x, owner, s0, s1, x.size, off)
        return s0, s1

    @staticmethod
    def open(s0, s1, scale_bits=16):
        s0, s1 = _u(s0), _u(s1)
        ring = np.empty(s0.size, np.uint64)
        f = np.empty(s0.size, np.float64)
        lib().orc_open(s0, s1, s0.size, ring.ctypes.data, f.ctypes.data, scale_bits)
        return ring, f

    def mul(self, x, y, off=0, trunc_bits=0):
        (x0, x1), (y0, y1) = map(lambda p: (_u(p[0]), _u(p[1])), (x, y))
        z0, z1 = _pair(x0.size)
        lib().orc_mul(ctypes.byref(self.c), x0, x1, y0, y1, z0, z1, x0.size, off, trunc_bits)
        return z0, z1

    def mul_bcast(self, x, y, rows, cols, off=0, row_off=0, trunc_bits=0):
        """z[r, j] = x[r, j] * y[r] with a broadcast triple."""
        (x0, x1), (y0, y1) = map(lambda p: (_u(p[0]), _u(p[1])), (x, y))
        z0, z1 = _pair(rows * cols)
        lib().orc_mul_bcast(ctypes.byref(self.c), x0, x1, y0, y1, z0, z1, rows, cols, off, row_off, trunc_bits)
        return z0, z1

    def matmul(self, x, y, batch, M, K, N, batch_off=0, trunc_bits=0):
        """Z[b] = X[b] (M x K) @ Y[b] (K x N) with a matrix Beaver triple."""
        (x0, x1), (y0, y1) = map(lambda p: (_u(p[0]), _u(p[1])), (x, y))
        z0, z1 = _pair(batch * M * N)
        lib().orc_matmul(ctypes.byref(self.c), x0, x1, y0, y1, z0, z1, batch, M, K, N, batch_off, trunc_bits)
        return z0, z1

    @staticmethod
    def trunc(x, bits=16):
        x0, x1 = _u(x[0]), _u(x[1])
        z0, z1 = _pair(x0.size)
        lib().orc_trunc(x0, x1, z0, z1, x0.size, bits)
        return z0, z1

    def _un(self, fn, x, *args):
        x0, x1 = _u(x[0]), _u(x[1])
        z0, z1 = _pair(x0.size)
        fn(ctypes.byref(self.c), x0, x1, z0, z1, x0.size, *args)
        return z0, z1

    def ltz(self, x, off=0, window=33):
        return self._un(lib().orc_ltz, x, off, window)

    def relu(self, x, off=0, window=33):
        return self._un(lib().orc_relu, x, off, window)

    def square(self, x, off=0, trunc_bits=0):
        return self._un(lib().orc_square, x, off, trunc_bits)

    def exp(self, x, off=0, t=8, clamp=0, window=33, square=0):
        return self._un(lib().orc_exp, x, off, t, clamp, window, square)

    def recip(self, x, off=0, iters=10, t=8, clamp=0, window=33, square=0):
        return self._un(lib().orc_recip, x, off, iters, t, clamp, window, square)

    def rsqrt(self, x, off=0, iters=3, t=8, clamp=0, window=33, square=0):
        return self._un(lib().orc_rsqrt, x, off, iters, t, clamp, window, square)

    ACT = {"gelu": 0, "silu": 1, "sigmoid": 2}
    FORM = {"poly_x": 0, "poly_abs": 1, "relu": 2, "erf": 3}

    def act(self, x, act="gelu", form="poly_x", degree=4, B=5.0, coeffs=None, erf_terms=8,
            off=0, window=33, basis=0):
        c = np.ascontiguousarray(coeffs if coeffs is not None else [0.0], dtype=np.float64)
        return self._un(lib().orc_act, x, off, self.ACT[act], self.FORM[form], degree, float(B),
                        c.ctypes.data, erf_terms, window, basis)

    def max(self, x, rows, cols, row_off=0, window=33):
        x0, x1 = _u(x[0]), _u(x[1])
        z0, z1 = _pair(rows)
        lib().orc_max(ctypes.byref(self.c), x0, x1, z0, z1, rows, cols, row_off, window)
        return z0, z1

    def maxpool2d(self, x, N, C, H, W, k=3, stride=2, pad=1, img_off=0, window=33):
        Ho = (H + 2 * pad - k) // stride + 1
        Wo = (W + 2 * pad - k) // stride + 1
        x0, x1 = _u(x[0]), _u(x[1])
        z0, z1 = _pair(N * C * Ho * Wo)
        lib().orc_maxpool2d(ctypes.byref(self.c), x0, x1, z0, z1, N, C, H, W, k, stride, pad,
                            img_off, window)
        return z0, z1

    def softmax(self, x, rows, cols, row_off=0, window=33, exp_t=8, exp_clamp=0, exp_window=33,
                recip_iters=10, recip_t=8, recip_clamp=0, recip_window=33, exp_square=0, recip_square=0,
                bcast=0, causal=0):
        x0, x1 = _u(x[0]), _u(x[1])
        z0, z1 = _pair(rows * cols)
        lib().orc_softmax(ctypes.byref(self.c), x0, x1, z0, z1, rows, cols, row_off, window,
                          exp_t, exp_clamp, exp_window, exp_square, recip_iters, recip_t, recip_clamp,
                          recip_window, recip_square, bcast, int(causal))
        return z0, z1

    def layernorm(self, x, rows, cols, row_off=0, eps=1e-5, mean_mode=0, rsqrt_iters=3,
                  rsqrt_t=8, rsqrt_clamp=0, rsqrt_window=33, rsqrt_square=0, bcast=0):
        x0, x1 = _u(x[0]), _u(x[1])
        z0, z1 = _pair(rows * cols)
        lib().orc_layernorm(ctypes.byref(self.c), x0, x1, z0, z1, rows, cols, row_off, eps,
                            mean_mode, rsqrt_iters, rsqrt_t, rsqrt_clamp, rsqrt_window, rsqrt_square, bcast)
        return z0, z1


class Plain:
    """Plaintext-ring schedules (the auto-tuner's non-MPC evaluator): each
    schedule of DESIGN.md 2.5 on one int64 ring value per element (scale 2^16), floor
    truncation, LTZ_w = bit (w-1).  Float64 in, float64 out (decoded ring values)."""

    @staticmethod
    def _x(x):
        return np.ascontiguousarray(x, dtype=np.float64).ravel()

    @classmethod
    def exp(cls, x, t=8, clamp=0, window=33):
        x = cls._x(x); y = np.empty_like(x)
        lib().orc_plain_exp(x, y, x.size, t, int(clamp), window)
        return y

    @classmethod
    def recip(cls, x, iters=10, t=8, clamp=0, window=33):
        x = cls._x(x); y = np.empty_like(x)
        lib().orc_plain_recip(x, y, x.size, iters, t, int(clamp), window)
        return y

    @classmethod
    def rsqrt(cls, x, iters=3, t=8, clamp=0, window=33):
        x = cls._x(x); y = np.empty_like(x)
        lib().orc_plain_rsqrt(x, y, x.size, iters, t, int(clamp), window)
        return y

    @classmethod
    def act(cls, x, act="gelu", form="poly_x", degree=4, B=5.0, coeffs=None, erf_terms=8, window=33, basis=0):
        x = cls._x(x); y = np.empty_like(x)
        c = np.ascontiguousarray(coeffs if coeffs is not None else [0.0], dtype=np.float64)
        lib().orc_plain_act(x, y, x.size, Oracle.ACT[act], Oracle.FORM[form], degree, float(B), c.ctypes.data,
                            erf_terms, window, basis)
        return y

    @classmethod
    def max(cls, x, rows, cols, window=33):
        x = cls._x(x); y = np.empty(rows, np.float64)
        lib().orc_plain_max(x, y, rows, cols, window)
        return y

    @classmethod
    def softmax(cls, x, rows, cols, window=33, exp_t=8, exp_clamp=0, exp_window=33, recip_iters=10, recip_t=8,
                recip_clamp=0, recip_window=33, causal=0):
        x = cls._x(x); y = np.empty_like(x)
        lib().orc_plain_softmax(x, y, rows, cols, window, exp_t, int(exp_clamp), exp_window, recip_iters, recip_t,
                                int(recip_clamp), recip_window, int(causal))
        return y

    @classmethod
    def layernorm(cls, x, rows, cols, eps=1e-5, mean_mode=0, rsqrt_iters=3, rsqrt_t=8, rsqrt_clamp=0,
                  rsqrt_window=33):
        x = cls._x(x); y = np.empty_like(x)
        lib().orc_plain_layernorm(x, y, rows, cols, float(eps), mean_mode, rsqrt_iters, rsqrt_t, int(rsqrt_clamp),
                                  rsqrt_window)
        return y
