"""fp64 references for the oracle (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Two kinds of reference, used by the tolerance tests:
  * the approximation FORMULA evaluated in float64 (isolates fixed-point error):
    exp-limit, Newton-Raphson reciprocal / rsqrt,
    segment polynomials, erf series (reading R21),
    max-stabilised softmax (P:604 footnote), layernorm;
  * the TRUE function (np.exp, 1/x, 1/sqrt(x), GELU via erf, SiLU, sigmoid).
"""
from __future__ import annotations

import math

import numpy as np

try:
    from scipy.special import erf as _erf
except Exception:  # pragma: no cover
    _erf = np.vectorize(math.erf)


# ---- true functions --------------------------------------------------------
def gelu(x):
    return 0.5 * x * (1.0 + _erf(x / math.sqrt(2.0)))


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def silu(x):
    return x * sigmoid(x)


TRUE_ACT = {"gelu": gelu, "silu": silu, "sigmoid": sigmoid}


def softmax(x):
    z = x - x.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


def layernorm(x, eps=1e-5):
    mu = x.mean(axis=-1, keepdims=True)
    v = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(v + eps)


# ---- approximation formulas in float64 -----------------------------------------
def exp_limit(x, t=8, clamp=False):
    """(1 + x/2^t)^(2^t), optionally zeroed below -2^t."""
    x = np.asarray(x, dtype=np.float64)
    y = 1.0 + x / 2.0 ** t
    if clamp:
        y = y * (x >= -(2.0 ** t))
    for _ in range(t):
        y = y * y
    return y


def recip_nr(x, iters=10, t=8, clamp=False):
    y = 3.0 * exp_limit(0.5 - x, t, clamp) + 0.003
    for _ in range(iters):
        y = y * (2.0 - x * y)
    return y


def rsqrt_nr(x, iters=3, t=8, clamp=False):
    y = 2.2 * exp_limit(-(x / 2.0 + 0.2), t, clamp) + 0.2
    for _ in range(iters):
        y = y * (3.0 - x * y * y) * 0.5
    return y


def erf_coeffs(K):
    out, fact = [], 1.0
    for k in range(K):
        if k > 0:
            fact *= k
        out.append((-1.0 if k & 1 else 1.0) / (fact * (2 * k + 1)))
    return out


def act_formula(x, act="gelu", form="poly_x", degree=4, B=5.0, coeffs=None, erf_terms=8):
    """Plaintext value of the segment approximation (reading R21)."""
    x = np.asarray(x, dtype=np.float64)
    if form == "relu" or degree == 0:
        if act == "sigmoid":
            return (x >= 0).astype(np.float64)
        return np.maximum(x, 0.0)
    if form == "poly_x":
        inner = np.polyval(list(coeffs)[::-1], x)
    elif form == "poly_abs":
        inner = 0.5 * x + np.polyval(list(coeffs)[::-1], np.abs(x))
    elif form == "erf":
        z = x / math.sqrt(2.0)
        a = erf_coeffs(erf_terms)
        S = np.polyval(a[::-1], z * z)
        inner = 0.5 * x * (1.0 + 2.0 / math.sqrt(math.pi) * z * S)
    else:
        raise ValueError(form)
    mid = (x >= -B) & (x < B)
    tail = (x >= B) * (1.0 if act == "sigmoid" else x)
    return np.where(mid, inner, 0.0) + tail


def softmax_formula(x, t=8, clamp=False, iters=10, rt=8, rclamp=False):
    m = x.max(axis=-1, keepdims=True)
    e = exp_limit(x - m, t, clamp)
    S = e.sum(axis=-1, keepdims=True)
    return e * recip_nr(S, iters, rt, rclamp)


def layernorm_formula(x, eps=1e-5, iters=3, t=8, clamp=False, mean_mode=0):
    """mean_mode 0 multiplies by the ENCODED public constant 1/d (Sec-PubFloat Mul,
    S:384: round(2^16/d)/2^16, reading R25); mean_mode 1 divides by d exactly."""
    d = x.shape[-1]
    inv_d = round(65536.0 / d) / 65536.0 if mean_mode == 0 else 1.0 / d
    eps = round(eps * 65536.0) / 65536.0
    mu = x.sum(axis=-1, keepdims=True) * inv_d
    c = x - mu
    v = (c * c).sum(axis=-1, keepdims=True) * inv_d + eps
    return c * rsqrt_nr(v, iters, t, clamp)
