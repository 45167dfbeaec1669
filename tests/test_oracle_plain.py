"""Pins for the oracle's PLAINTEXT-ring schedules (oracle.Plain, oracle.c orc_plain_*): the
auto-tuner's non-MPC evaluator, which the GPU
evaluator mpc_plain_eval must match bit for bit (tests/test_gpu_tuner.py).

Each schedule is pinned against something other than itself:
  * the fp64 approximation FORMULA within the fixed-point budget of DESIGN.md section 5;
  * the TRUE function within the approximation's stated error (R15-R21 readings);
  * the MPC oracle (two parties, Beaver / LTZ / per-share truncation, pinned in
    test_oracle_core / test_oracle_approx): the plaintext run differs from the reconstructed MPC
    result only by the per-share truncation of each product, so within the same budget;
  * exact identities: degree 0 = ReLU / unit step, t = 0 + clamp = ReLU(1 + x) (R14), exact
    segment tails, exact row maxima, constant LayerNorm rows -> 0, bit-identical softmax under a
    public shift (and LayerNorm mean_mode 1 under a shift), causal masked outputs exactly 0 and
    unmasked last-position rows identical to the dense op.
"""
import json
import os

import numpy as np
import pytest

import workloads
from oracle import Oracle, Plain, encode
from oracle import float_ref as fr

COEFFS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "fixtures",
                                     "coeffs.json")))["fits"]
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
ULP = 2.0 ** -16


def q(x):
    """inputs on the 2^-16 grid, so E(x) = x * 2^16 exactly and float references see the same x"""
    return np.array([encode(v) for v in np.ravel(x)], dtype=np.float64) / 65536.0


def mpc(cfg=1):
    return Oracle.for_cfg(workloads.keys(cfg))


def dec(s):
    return Oracle.open(*s)[1]


def horner_tol(v, d, abs_form=False):
    v = np.abs(v)
    t = 0.5 * v ** d + sum(2.5 * v ** k for k in range(d))
    return (t + (2 if abs_form else 0) + 1) * ULP


# ------------------------------------------------------------------ exp ----
@pytest.mark.parametrize("t,clamp", [(8, 0), (8, 1), (6, 0), (4, 1), (2, 1), (1, 0), (0, 0)])
def test_plain_exp_vs_formula_and_mpc(t, clamp):
    x = q(workloads.exp_inputs(4096, tail_frac=0.05 if clamp else 0.0))
    y = Plain.exp(x, t, clamp)
    f = fr.exp_limit(x, t, clamp)
    m = np.ones_like(x, bool) if clamp else x >= -(2.0 ** t)
    tol = 4 * 2 ** t * ULP * np.maximum(1.0, np.abs(f))
    assert np.all(np.abs(y - f)[m] <= tol[m])
    o = mpc()
    ym = dec(o.exp(o.share(x), t=t, clamp=clamp))
    assert np.all(np.abs(y - ym)[m] <= tol[m])


def test_plain_exp_t0_clamp_is_relu_of_1_plus_x_exactly():
    x = q(np.concatenate([np.linspace(-3, 3, 1201), [-1.0, -2.0, -0.5]]))
    assert np.array_equal(Plain.exp(x, 0, 1), np.maximum(0.0, 1.0 + x))
    assert np.array_equal(Plain.exp(x, 0, 0), 1.0 + x)


def test_plain_exp_golden():
    g = GOLD["exp_t8_xm1"]
    assert abs(Plain.exp([g["x"]], g["t"])[0] - g["value"]) <= 4 * 256 * ULP
    d = GOLD["exp_t8_xm600_diverges"]
    assert abs(Plain.exp([d["x"]], d["t"], 1)[0]) == 0.0           # clamped: exactly zero


# ---------------------------------------------------------- Newton-Raphson ----
def test_plain_recip():
    x = q(workloads.recip_inputs(4096))
    y = Plain.recip(x, 10)
    assert np.all(np.abs(y - fr.recip_nr(x, 10)) <= 4 * ULP * (1 + 1 / x) + 1e-12)
    assert np.max(np.abs(y - 1 / x) * x) <= 1e-2 + 4 * ULP * (1 + x).max()
    o = mpc()
    ym = dec(o.recip(o.share(x), iters=10))
    assert np.all(np.abs(y - ym) <= 8 * ULP * (1 + 1 / x))
    # R17: recip(1.0) needs >= 7 iterations; error decreasing in iters
    assert abs(Plain.recip([1.0], 7)[0] - 1) <= 1e-4 and abs(Plain.recip([1.0], 1)[0] - 1) > 0.5


@pytest.mark.parametrize("iters,tol_ulp", [(3, 64), (10, 16)])
def test_plain_rsqrt(iters, tol_ulp):
    x = q(np.exp(np.random.default_rng(3).uniform(np.log(0.25), np.log(16), 4096)))
    y = Plain.rsqrt(x, iters)
    f = fr.rsqrt_nr(x, iters)
    assert np.all(np.abs(y - f) <= tol_ulp * ULP * np.maximum(1, f))
    o = mpc()
    ym = dec(o.rsqrt(o.share(x), iters=iters))
    assert np.all(np.abs(y - ym) <= 2 * tol_ulp * ULP * np.maximum(1, f))
    g = GOLD["rsqrt_4"]
    assert abs(Plain.rsqrt([g["x"]], g["iters"])[0] - g["value"]) <= g["tol"]


# ---------------------------------------------------------- segment polys ----
@pytest.mark.parametrize("fit", [f for f in COEFFS if f["form"] != "erf"],
                         ids=lambda f: f"{f['op']}-{f['form']}-{f['degree']}")
@pytest.mark.parametrize("basis", [0, 1])
def test_plain_poly(fit, basis):
    B = fit["interval"][1]
    x = q(workloads.act_inputs(4096))
    y = Plain.act(x, fit["op"], fit["form"], fit["degree"], B, fit["coefficients"], basis=basis)
    f = fr.act_formula(x, fit["op"], fit["form"], fit["degree"], B, fit["coefficients"])
    tol = horner_tol(x, fit["degree"], fit["form"] == "poly_abs")
    if basis:
        tol = tol + 8 * (1 + np.abs(x) ** 2) * ULP * sum(abs(c) for c in fit["coefficients"])
    assert np.all(np.abs(y - f) <= tol)
    # exact tails outside [-B, B): x (or 1) above, 0 below
    hi, lo = x >= B, x < -B
    assert np.all(y[hi] == (1.0 if fit["op"] == "sigmoid" else x[hi])) and np.all(y[lo] == 0)
    o = mpc()
    ym = dec(o.act(o.share(x), fit["op"], fit["form"], fit["degree"], B, fit["coefficients"], basis=basis))
    assert np.all(np.abs(y - ym) <= 2 * tol)


@pytest.mark.parametrize("K", [4, 8])
def test_plain_erf(K):
    B = 2.5
    x = q(workloads.act_inputs(4096))
    y = Plain.act(x, "gelu", "erf", 1, B, None, K)
    f = fr.act_formula(x, "gelu", "erf", 1, B, None, K)
    z2 = np.minimum(x * x / 2, B * B / 2)
    tol = horner_tol(z2, K - 1) * (1 + np.abs(x)) + 8 * ULP
    assert np.all(np.abs(y - f) <= tol)
    o = mpc()
    assert np.all(np.abs(y - dec(o.act(o.share(x), "gelu", "erf", 1, B, None, K))) <= 2 * tol)


def test_plain_degree0_exact():
    x = q(np.linspace(-4, 4, 801))
    for act in ("gelu", "silu"):
        assert np.array_equal(Plain.act(x, act, "relu"), np.maximum(x, 0.0))
        assert np.array_equal(Plain.act(x, act, "poly_x", 0, 5.0, [0.0]), np.maximum(x, 0.0))
    assert np.array_equal(Plain.act(x, "sigmoid", "poly_x", 0, 5.0, [0.0]), (x >= 0).astype(np.float64))


# ------------------------------------------------------------------ max ----
@pytest.mark.parametrize("cols", [1, 2, 3, 7, 9, 128, 1000])
def test_plain_max_exact(cols):
    x = q(workloads.softmax_inputs(40, cols))
    assert np.array_equal(Plain.max(x, 40, cols), x.reshape(40, cols).max(1))


# -------------------------------------------------------------- softmax ----
@pytest.mark.parametrize("rows,cols,tol_true", [(64, 128, 1.1e-2), (16, 1024, 3e-2), (40, 77, 1.1e-2)])
def test_plain_softmax(rows, cols, tol_true):
    x = q(workloads.softmax_inputs(rows, cols))
    y = Plain.softmax(x, rows, cols).reshape(rows, cols)
    X = x.reshape(rows, cols)
    assert np.max(np.abs(y - fr.softmax_formula(X))) <= 2 * 4 * 256 * ULP + 8 * ULP
    assert np.max(np.abs(y - fr.softmax(X))) <= tol_true
    o = mpc(2)
    ym = dec(o.softmax(o.share(x), rows, cols)).reshape(rows, cols)
    assert np.max(np.abs(y - ym)) <= 2 * (2 * 4 * 256 * ULP + 8 * ULP)


def test_plain_softmax_shift_invariance_and_golden():
    rows, cols = 32, 64
    x = q(workloads.softmax_inputs(rows, cols))
    assert np.array_equal(Plain.softmax(x, rows, cols), Plain.softmax(x + 3.25, rows, cols))
    g = GOLD["softmax_00"]
    assert np.max(np.abs(Plain.softmax(g["x"], 1, 2) - g["out"])) <= 1e-2


def test_plain_softmax_causal():
    T, rows = 64, 128
    x = q(workloads.softmax_inputs(rows, T))
    y = Plain.softmax(x, rows, T, causal=1).reshape(rows, T)
    X = x.reshape(rows, T)
    pos = np.arange(rows)[:, None] % T
    masked = np.arange(T)[None, :] > pos
    assert np.all(y[masked] == 0.0)
    ref = fr.softmax(np.where(masked, -np.inf, X))
    assert np.max(np.abs(y - ref)) <= 1.1e-2
    dense = Plain.softmax(x, rows, T).reshape(rows, T)
    last = (np.arange(rows) % T) == T - 1
    assert np.array_equal(y[last], dense[last])


def test_plain_softmax_clamp_variant():
    rows, cols = 32, 128
    x = q(workloads.softmax_inputs(rows, cols, spike=True))
    y = Plain.softmax(x, rows, cols, exp_clamp=1).reshape(rows, cols)
    assert np.max(np.abs(y - fr.softmax(x.reshape(rows, cols)))) <= 1.1e-2


# ------------------------------------------------------------ layernorm ----
@pytest.mark.parametrize("mean_mode,iters", [(0, 3), (1, 3), (1, 10)])
def test_plain_layernorm(mean_mode, iters):
    rows, cols = 64, 768
    x = q(workloads.layernorm_inputs(rows, cols))
    X = x.reshape(rows, cols)
    y = Plain.layernorm(x, rows, cols, mean_mode=mean_mode, rsqrt_iters=iters).reshape(rows, cols)
    assert np.max(np.abs(y - fr.layernorm_formula(X, iters=iters, mean_mode=mean_mode))) <= 2e-3
    tol_true = 1.6e-2 if mean_mode == 0 else (8e-3 if iters == 3 else 1e-3)
    assert np.max(np.abs(y - fr.layernorm(X))) <= tol_true
    o = mpc(5)
    ym = dec(o.layernorm(o.share(x), rows, cols, mean_mode=mean_mode, rsqrt_iters=iters)).reshape(rows, cols)
    assert np.max(np.abs(y - ym)) <= 4e-3


def test_plain_layernorm_exact_identities():
    # constant rows: c = 0 exactly when the mean is exact -- floor division (mode 1), or mode 0
    # with d a power of two (E(1/256) = 256 exactly; E(1/768) = 85 carries R25's -0.39 %)
    x = np.tile(np.array([[0.75], [-1.25], [3.0]]), (1, 768))
    assert np.all(Plain.layernorm(x, 3, 768, mean_mode=1) == 0.0)
    assert np.all(Plain.layernorm(x[:, :256], 3, 256, mean_mode=0) == 0.0)
    xs = q(workloads.layernorm_inputs(8, 768))
    a = Plain.layernorm(xs, 8, 768, mean_mode=1)
    b = Plain.layernorm(xs + 2.5, 8, 768, mean_mode=1)     # floor((S + d E(c)) / d) = mu + E(c)
    assert np.array_equal(a, b)
