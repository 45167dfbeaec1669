"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no encoding, no sharing, no PRG):
it only draws float activations with the shapes and value distributions of the
paper's workloads and names
the PRG keys each config uses.  Both the oracle side and the CUDA side consume
the same arrays, which is what makes bit-exact parity checkable.

Shapes come from BASELINE.json `configs`:
  cfg1  exp / reciprocal / GELU on 4096 elements, both parties on one device
  cfg2  BERT-base attention softmax 8x12x128x128            (PAPER.md P:735 defaults)
  cfg3  BERT-base FFN GELU 8x128x3072
  cfg4  ResNet-50 ReLU / MaxPool at batch 32               (first layer 32x64x112x112)
  cfg5  GPT-2 small softmax 1024-token, GELU, LayerNorm 768
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 2511_19711

# PRG keys per config (SURVEY.md §8(d) "PRG keys"): K_s share-mask key,
# K_0 / K_1 dealer->party keys.  64-bit each.
def keys(cfg: int) -> dict:
    return {
        "key_share": (0x5EED0000 << 32) | cfg,
        "key_p0": (0xDEA10000 << 32) | cfg,
        "key_p1": (0xDEA11111 << 32) | cfg,
    }


def rng(cfg: int, stream: int = 0) -> np.random.Generator:
    return np.random.default_rng(SEED_BASE + cfg + 1000 * stream)


SHAPES = {
    "cfg1_elems": 4096,
    "cfg2_softmax": (8 * 12 * 128, 128),        # rows x cols
    "cfg3_gelu": 8 * 128 * 3072,
    "cfg4_relu_first": (32, 64, 112, 112),
    "cfg4_maxpool_in": (32, 64, 112, 112),
    "cfg5_softmax": (8 * 12 * 1024, 1024),
    "cfg5_gelu": 8 * 1024 * 3072,
    "cfg5_ln": (8 * 1024, 768),
}


def exp_inputs(n: int, seed_cfg: int = 1, tail_frac: float = 0.0) -> np.ndarray:
    """U[-10, 2] plus an optional tail slice U[-600, -512] (cfg1)."""
    g = rng(seed_cfg, 1)
    x = g.uniform(-10.0, 2.0, n)
    k = int(n * tail_frac)
    if k:
        x[-k:] = g.uniform(-600.0, -512.0, k)
    return x


def recip_inputs(n: int, seed_cfg: int = 1, lo: float = 0.05, hi: float = 128.0) -> np.ndarray:
    """log-uniform on [lo, hi] (cfg1; softmax row sums live in [1, 50])."""
    g = rng(seed_cfg, 2)
    return np.exp(g.uniform(np.log(lo), np.log(hi), n))


def rsqrt_inputs(n: int, seed_cfg: int = 1, lo: float = 0.25, hi: float = 16.0) -> np.ndarray:
    g = rng(seed_cfg, 3)
    return np.exp(g.uniform(np.log(lo), np.log(hi), n))


def act_inputs(n: int, seed_cfg: int = 1, lo: float = -8.0, hi: float = 8.0) -> np.ndarray:
    """GELU/SiLU/Sigmoid inputs U[-8, 8] (cfg1)."""
    g = rng(seed_cfg, 4)
    return g.uniform(lo, hi, n)


def normal_inputs(n: int, seed_cfg: int, sigma: float = 2.0, stream: int = 5) -> np.ndarray:
    """N(0, sigma^2): attention scores / FFN pre-activations (cfg2, cfg3, cfg5)."""
    g = rng(seed_cfg, stream)
    return g.normal(0.0, sigma, n)


def softmax_inputs(rows: int, cols: int, seed_cfg: int = 2, sigma: float = 2.0,
                   spike: bool = False) -> np.ndarray:
    """Attention scores N(0, sigma^2); optional +6 spike on one position per row."""
    g = rng(seed_cfg, 6)
    x = g.normal(0.0, sigma, (rows, cols))
    if spike:
        pos = g.integers(0, cols, rows)
        x[np.arange(rows), pos] += 6.0
    return x


def layernorm_inputs(rows: int, cols: int, seed_cfg: int = 5) -> np.ndarray:
    """Rows N(mu_r, sigma_r^2), mu_r ~ U[-1,1], sigma_r ~ U[0.5, 4] (cfg5)."""
    g = rng(seed_cfg, 7)
    mu = g.uniform(-1.0, 1.0, (rows, 1))
    sd = g.uniform(0.5, 4.0, (rows, 1))
    return mu + sd * g.normal(0.0, 1.0, (rows, cols))


def relu_inputs(n: int, seed_cfg: int = 4) -> np.ndarray:
    g = rng(seed_cfg, 8)
    return g.normal(0.0, 1.0, n)


def maxpool_inputs(shape, seed_cfg: int = 4) -> np.ndarray:
    """Post-ReLU activations (MaxPool follows ReLU in ResNet, reading R26)."""
    g = rng(seed_cfg, 9)
    return np.maximum(g.normal(0.0, 1.0, shape), 0.0)


def random_ring(n: int, seed: int) -> np.ndarray:
    """Uniform u64 values (for share-algebra / Beaver / LTZ property tests)."""
    g = np.random.default_rng(seed)
    return g.integers(0, 2**64, n, dtype=np.uint64, endpoint=False)
