"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only draws the inputs x, y of the
BASELINE.json configs (DESIGN.md §3 "input recipe").  Both the oracle and the CUDA path
consume the same host arrays produced here, so no random-number code is duplicated.

Generator: counter-based splitmix64.  Element ``idx`` of stream ``stream`` under ``seed``
is ``mix(seed * G + (stream << 40) + idx + 1)`` with G the 64-bit golden-ratio constant
and ``mix`` the splitmix64 finaliser, so values do not depend on generation order.
Streams: x uses ``2*b``, y uses ``2*b + 1`` (b = batch index, 0 for single pairs).
"""
from __future__ import annotations

import numpy as np

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# BASELINE.json configs (names used by tests and bench.py)
CONFIGS = {
    "c1_d10_i64": dict(D=10, dtype="int64", dist="uniform", lo=0, hi=9, seed=1001, batch=1),
    "c2_b65536_d8_i64": dict(D=8, dtype="int64", dist="uniform", lo=0, hi=255, seed=1002, batch=65536),
    "c3_d16_i64": dict(D=16, dtype="int64", dist="uniform", lo=0, hi=(1 << 16) - 1, seed=1003, batch=1),
    "c4_d20_f64": dict(D=20, dtype="float64", dist="exp_norm", seed=1004, batch=1),
    "c5_d22_f64": dict(D=22, dtype="float64", dist="exp_norm", seed=1005, batch=1),
}


def splitmix64(seed: int, stream: int, n: int, start: int = 0) -> np.ndarray:
    """n counter-based 64-bit draws (uint64) for (seed, stream), indices start..start+n-1."""
    with np.errstate(over="ignore"):
        ctr = np.arange(start, start + n, dtype=np.uint64) + np.uint64(1)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) * _G + (np.uint64(stream) << np.uint64(40)) + ctr
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_int(seed: int, stream: int, n: int, lo: int, hi: int) -> np.ndarray:
    """int64 uniform on [lo, hi] (inclusive) via r % (hi-lo+1); bias <= (hi-lo)/2^64."""
    r = splitmix64(seed, stream, n)
    span = np.uint64(hi - lo + 1)
    return (r % span).astype(np.int64) + np.int64(lo)


def exp_normalized(seed: int, stream: int, n: int) -> np.ndarray:
    """fp64 i.i.d. Exponential(1) via -log1p(-u), u = (r >> 11) * 2^-53, then divided by
    the array's sum (BASELINE.json config 4: 'probability masses ... normalized to sum 1')."""
    r = splitmix64(seed, stream, n)
    u = (r >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    x = -np.log1p(-u)
    return x / x.sum()


def draw(dist: str, seed: int, stream: int, n: int, lo: int = 0, hi: int = 9) -> np.ndarray:
    if dist == "uniform":
        return uniform_int(seed, stream, n, lo, hi)
    if dist == "exp_norm":
        return exp_normalized(seed, stream, n)
    if dist == "uniform01":
        r = splitmix64(seed, stream, n)
        return (r >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    raise ValueError(dist)


def make_pair(D: int, dtype: str, dist: str, seed: int, lo: int = 0, hi: int = 9):
    n = 1 << D
    x = draw(dist, seed, 0, n, lo, hi)
    y = draw(dist, seed, 1, n, lo, hi)
    return x.astype(dtype), y.astype(dtype)


def make_batched(B: int, D: int, dtype: str, dist: str, seed: int, lo: int = 0, hi: int = 9):
    """[B, 2^D] pairs; batch b uses streams 2b (x) and 2b+1 (y)."""
    n = 1 << D
    x = np.empty((B, n), dtype=dtype)
    y = np.empty((B, n), dtype=dtype)
    if dist == "uniform":
        # vectorised: one draw per (b, i) with stream folded into the counter
        for b in range(B):
            x[b] = uniform_int(seed, 2 * b, n, lo, hi)
            y[b] = uniform_int(seed, 2 * b + 1, n, lo, hi)
    else:
        for b in range(B):
            x[b] = draw(dist, seed, 2 * b, n, lo, hi)
            y[b] = draw(dist, seed, 2 * b + 1, n, lo, hi)
    return x, y


def make_batched_fast(B: int, D: int, lo: int, hi: int, seed: int):
    """Same values as make_batched(..., 'uniform', ...) but vectorised over batches."""
    n = 1 << D
    with np.errstate(over="ignore"):
        b = np.arange(B, dtype=np.uint64)[:, None]
        ctr = np.arange(n, dtype=np.uint64)[None, :] + np.uint64(1)
        out = []
        for parity in (0, 1):
            stream = b * np.uint64(2) + np.uint64(parity)
            z = np.uint64(seed) * _G + (stream << np.uint64(40)) + ctr
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z = z ^ (z >> np.uint64(31))
            out.append((z % np.uint64(hi - lo + 1)).astype(np.int64) + np.int64(lo))
    return out[0], out[1]


def config_inputs(name: str):
    """x, y for a named BASELINE.json config (batched configs return [B, 2^D])."""
    c = CONFIGS[name]
    if c["batch"] > 1:
        return make_batched_fast(c["batch"], c["D"], c["lo"], c["hi"], c["seed"])
    return make_pair(c["D"], c["dtype"], c["dist"], c["seed"], c.get("lo", 0), c.get("hi", 9))


def all_ones(D: int, dtype="int64"):
    n = 1 << D
    return np.ones(n, dtype=dtype), np.ones(n, dtype=dtype)


def separable_factors(D: int, seed: int, lo: int = 1, hi: int = 2):
    """Per-axis length-2 factors (a_d, b_d) with integer entries in [lo, hi]."""
    fx = uniform_int(seed, 100, 2 * D, lo, hi).reshape(D, 2)
    fy = uniform_int(seed, 101, 2 * D, lo, hi).reshape(D, 2)
    return fx, fy


def tensor_product(f: np.ndarray) -> np.ndarray:
    """x[i] = prod_b f[b, bit_b(i)]  (bit b of the flat index is axis b)."""
    D = f.shape[0]
    x = np.ones(1, dtype=f.dtype)
    for b in range(D):
        # new axis b is the next more significant bit: x_new[i + 2^b * t] = x[i] * f[b, t]
        x = np.concatenate([x * f[b, 0], x * f[b, 1]])
    return x
