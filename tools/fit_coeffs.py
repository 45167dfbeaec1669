"""Least-squares fits of the segment polynomials -> fixtures/coeffs.json.

SPEC.md S:239 decision: coefficients are NOT copied from BOLT (the paper does
not print them); they are least-squares fits on a dense grid,
stored with the max abs error over the whole real line (inside the segment:
polynomial error; outside: asymptote error).  Forms:
  poly_x   : f(x) ~ P(x)                 on [-B, B]   (SPEC S:193 literal form)
  poly_abs : f(x) ~ 0.5 x + P(|x|)       on [-B, B]   (BOLT structure, P:737;
             valid for GELU and SiLU, whose f(x) - x/2 is even)
Coefficients are low -> high.  Run:  python tools/fit_coeffs.py
"""
from __future__ import annotations

import json
import math
import os

import numpy as np

from scipy.special import erf

# The fixture is an input of BOTH sides (knob values passed through the ABI), so this tool is
# self-contained: it imports nothing from oracle/ (test infrastructure) or from the product.
TRUE_ACT = {
    "gelu": lambda x: 0.5 * x * (1.0 + erf(x / math.sqrt(2.0))),
    "silu": lambda x: x * (1.0 / (1.0 + np.exp(-x))),
    "sigmoid": lambda x: 1.0 / (1.0 + np.exp(-x)),
}


def act_formula(x, act, form, degree, B, coeffs=None, erf_terms=8):
    """Segment approximation in float64: inside [-B, B) the form's polynomial (x-form S:193,
    |x|-form P:737) or the erf Maclaurin series (reading R21); outside the asymptote."""
    if form == "poly_x":
        inner = np.polyval(list(coeffs)[::-1], x)
    elif form == "poly_abs":
        inner = 0.5 * x + np.polyval(list(coeffs)[::-1], np.abs(x))
    else:
        z2 = x * x / 2.0
        S, fact = np.zeros_like(x), 1.0
        for k in range(erf_terms):
            fact = fact * k if k > 0 else 1.0
            S = S + ((-1.0) ** k / (fact * (2 * k + 1))) * z2 ** k
        inner = 0.5 * x * (1.0 + 2.0 / math.sqrt(math.pi) * (x / math.sqrt(2.0)) * S)
    mid = (x >= -B) & (x < B)
    tail = (x >= B) * (1.0 if act == "sigmoid" else x)
    return np.where(mid, inner, 0.0) + tail


FITS = [
    # (act, form, degree, B)
    ("gelu", "poly_x", 4, 5.0), ("gelu", "poly_x", 2, 5.0),
    ("gelu", "poly_abs", 4, 3.0), ("gelu", "poly_abs", 2, 3.0),
    ("silu", "poly_x", 4, 5.0), ("silu", "poly_x", 2, 5.0),
    ("silu", "poly_abs", 4, 5.0), ("silu", "poly_abs", 2, 5.0),
    ("sigmoid", "poly_x", 4, 5.0), ("sigmoid", "poly_x", 2, 5.0),
]


def fit(act, form, degree, B):
    f = TRUE_ACT[act]
    if form == "poly_x":
        xs = np.linspace(-B, B, 20001)
        c = np.polynomial.polynomial.polyfit(xs, f(xs), degree)
    else:
        xs = np.linspace(0.0, B, 20001)
        c = np.polynomial.polynomial.polyfit(xs, f(xs) - 0.5 * xs, degree)
    c = [float(v) for v in c]
    grid = np.linspace(-B - 4.0, B + 4.0, 200001)
    err = float(np.max(np.abs(act_formula(grid, act, form, degree, B, c) - f(grid))))
    return c, err


def main():
    out = []
    for act, form, d, B in FITS:
        c, err = fit(act, form, d, B)
        out.append({"op": act, "form": form, "degree": d, "interval": [-B, B],
                    "coefficients": c, "max_abs_error": err})
        print(f"{act:8s} {form:9s} deg {d}  B={B}: max|err| = {err:.4g}")
    for K, B in ((4, 2.5), (6, 2.5), (8, 2.5)):
        grid = np.linspace(-B - 4.0, B + 4.0, 200001)
        err = float(np.max(np.abs(act_formula(grid, "gelu", "erf", 1, B, None, K)
                                  - TRUE_ACT["gelu"](grid))))
        out.append({"op": "gelu", "form": "erf", "erf_terms": K, "interval": [-B, B],
                    "coefficients": None, "max_abs_error": err})
        print(f"gelu     erf       K={K}  B={B}: max|err| = {err:.4g}")
    relu_err = float(np.max(np.abs(np.maximum(grid, 0) - TRUE_ACT["gelu"](grid))))
    print(f"gelu relu: {relu_err:.4g}")
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "fixtures", "coeffs.json")
    with open(path, "w") as fh:
        json.dump({"source": "tools/fit_coeffs.py (least squares, SPEC S:239 decision)",
                   "fits": out}, fh, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
