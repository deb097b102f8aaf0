"""Oracles for the applications built on the hot path -- TEST
INFRASTRUCTURE ONLY (only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
use it).  Plain numpy written from the definitions in the paper; nothing here calls the CUDA
path, and none of it uses the Karatsuba split.

    difference_pmf   P(X - Y = d) for independent X, Y in {0,1}^D (PAPER.md 35-38, 147-149),
                     by its definition: every pair (i, j) adds x[i] y[j] to the cell of the
                     digit-wise difference d = i - j, stored at k = sum_b (d_b + 1) 3^b.
    carries          out[m] = sum_{k : sum_b k_b 2^b = m} z[k] -- performing the carries of
                     the carry-free convolution (PAPER.md 354-373: (2,1,2) -> 12).
    conv1d_carryfree_then_carries
                     carries(Algorithm 1 on the bit-axis embedding), PAPER.md 354-373.
    maxconv_exact    max_{i + j = k} x[i] y[j] (the (x, max) semiring, PAPER.md 341-346), brute
                     force over all pairs.
    maxconv_pnorm    mx my (sum_{i+j=k} (x[i]/mx)^p (y[j]/my)^p)^(1/p), the p-norm estimate of
                     PAPER.md 341-352, from Algorithm 1 on the scaled powers.
"""
from __future__ import annotations

import numpy as np

from . import conv as _conv  # Algorithm 1 (gather form), oracle/hc_oracle.c


def _tern_table(D: int) -> np.ndarray:
    """T(i) = sum_b bit_b(i) 3^b for all i < 2^D (PAPER.md 109-112)."""
    t = np.zeros(1, dtype=np.int64)
    for b in range(D):
        t = np.concatenate([t, t + 3 ** b])
    return t


def difference_pmf(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """z[k] = sum_{i, j : i_b - j_b = k_b - 1 for all b} x[i] y[j]; pairs in i-major order."""
    n = x.shape[0]
    D = n.bit_length() - 1
    T = _tern_table(D)
    ones = sum(3 ** b for b in range(D))  # digit offset +1 on every axis
    z = np.zeros(3 ** D, dtype=x.dtype)
    for i in range(n):
        k = T[i] - T + ones  # d = i - j digit-wise, shifted to {0,1,2}
        np.add.at(z, k, x[i] * y)
    return z


def carry_values(D: int) -> np.ndarray:
    """val(k) = sum_b k_b 2^b for every ternary index k < 3^D."""
    v = np.zeros(1, dtype=np.int64)
    for b in range(D):
        v = np.concatenate([v, v + (1 << b), v + (2 << b)])
    return v


def carries(z: np.ndarray, D: int) -> np.ndarray:
    """out[m] = sum_{k : val(k) = m} z[k], m < 2^(D+1) - 1, cells added in ascending k."""
    out = np.zeros((2 << D) - 1, dtype=z.dtype)
    np.add.at(out, carry_values(D), z)
    return out


def conv1d_carryfree_then_carries(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    D = x.shape[0].bit_length() - 1
    return carries(_conv(x, y), D)


def maxconv_exact(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    n = x.shape[0]
    D = n.bit_length() - 1
    T = _tern_table(D)
    z = np.full(3 ** D, -np.inf if x.dtype.kind == "f" else np.iinfo(x.dtype).min, dtype=x.dtype)
    for i in range(n):
        np.maximum.at(z, T[i] + T, x[i] * y)
    return z


def maxconv_pnorm(x: np.ndarray, y: np.ndarray, p: float) -> np.ndarray:
    mx, my = float(x.max()), float(y.max())
    xp = (x / mx) ** p if mx > 0 else np.zeros_like(x)
    yp = (y / my) ** p if my > 0 else np.zeros_like(y)
    s = _conv(xp, yp)
    return np.where(s > 0, mx * my * np.power(np.maximum(s, 0.0), 1.0 / p), 0.0)
