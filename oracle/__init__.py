"""Oracle for hypercube convolution -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_1608_00206_b200``) never imports it and shares no code with it.

It wraps ``hc_oracle.c``: the paper's naive Algorithm 1 of the
convolution definition on bit-indexed flat arrays, fp64 and int64
(uint64 wrap-around).  See the C file's header for the exact contract of each function.

Pins (tests/test_oracle_pins.py) tie it to what the paper and the mathematics fix: the
D=1 form (PAPER.md 174-176, 259-261), a hand-derived D=2 example, the all-ones closed
form, separable inputs (the axis-peeling identity, PAPER.md 153-164), deltas including
the carry-free example 7,5 -> (2,1,2) (PAPER.md 359-365), mass conservation, the
generating-function identity mod a prime, and a multi-index brute force for D <= 4.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile hc_oracle.c with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int
        I64 = ctypes.c_int64
        U64 = ctypes.c_uint64
        L.orc_ternary_of_binary.argtypes = [U64]
        L.orc_ternary_of_binary.restype = U64
        L.orc_pow3.argtypes = [I]
        L.orc_pow3.restype = U64
        L.orc_max_threads.restype = I
        for dt in ("f64", "i64"):
            getattr(L, f"orc_conv_scatter_{dt}").argtypes = [I, P, P, P]
            getattr(L, f"orc_conv_gather_{dt}").argtypes = [I, P, P, P, I]
            getattr(L, f"orc_conv_cells_{dt}").argtypes = [I, P, P, P, I64, P, I]
            getattr(L, f"orc_conv_batched_{dt}").argtypes = [I, I, P, P, P, I]
        L.orc_conv_batched_cells_i64.argtypes = [I, P, P, P, P, I64, P, I]
        _lib = L
    return _lib


def _dt(a: np.ndarray) -> str:
    if a.dtype == np.float64:
        return "f64"
    if a.dtype == np.int64:
        return "i64"
    raise TypeError(f"oracle supports float64 and int64, got {a.dtype}")


def _check(x: np.ndarray, y: np.ndarray) -> int:
    x = np.asarray(x)
    y = np.asarray(y)
    if x.dtype != y.dtype or x.ndim != 1 or y.shape != x.shape:
        raise ValueError("x, y must be 1-D arrays of equal length and dtype")
    n = x.shape[0]
    D = n.bit_length() - 1
    if n < 2 or (1 << D) != n:
        raise ValueError("length must be 2^D with D >= 1")
    return D


def ternary_of_binary(i: int) -> int:
    return int(lib().orc_ternary_of_binary(i))


def conv_scatter(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Algorithm 1 literally: z <- 0; for i: for j: z[i+j] += x[i]*y[j] (single thread)."""
    D = _check(x, y)
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    z = np.empty(3 ** D, dtype=x.dtype)
    getattr(lib(), f"orc_conv_scatter_{_dt(x)}")(D, x.ctypes.data, y.ctypes.data, z.ctypes.data)
    return z


def conv(x: np.ndarray, y: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """Gather form of Algorithm 1 (bitwise identical to conv_scatter), OpenMP over cells."""
    D = _check(x, y)
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    z = np.empty(3 ** D, dtype=x.dtype)
    getattr(lib(), f"orc_conv_gather_{_dt(x)}")(D, x.ctypes.data, y.ctypes.data, z.ctypes.data, nthreads)
    return z


def conv_cells(x: np.ndarray, y: np.ndarray, ks, nthreads: int = 0) -> np.ndarray:
    """z[k] for the listed flat output indices only (sampled parity)."""
    D = _check(x, y)
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    ks = np.ascontiguousarray(np.asarray(ks, dtype=np.uint64))
    out = np.empty(ks.shape[0], dtype=x.dtype)
    getattr(lib(), f"orc_conv_cells_{_dt(x)}")(D, x.ctypes.data, y.ctypes.data, ks.ctypes.data,
                                               ks.shape[0], out.ctypes.data, nthreads)
    return out


def conv_batched(x: np.ndarray, y: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """x, y of shape [B, 2^D] -> z of shape [B, 3^D] (row-major batches)."""
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    if x.ndim != 2 or x.shape != y.shape or x.dtype != y.dtype:
        raise ValueError("x, y must be [B, 2^D] arrays of equal shape and dtype")
    B, n = x.shape
    D = n.bit_length() - 1
    if (1 << D) != n or D < 1:
        raise ValueError("row length must be 2^D")
    z = np.empty((B, 3 ** D), dtype=x.dtype)
    getattr(lib(), f"orc_conv_batched_{_dt(x)}")(B, D, x.ctypes.data, y.ctypes.data, z.ctypes.data, nthreads)
    return z


def conv_batched_cells_i64(x: np.ndarray, y: np.ndarray, bs, ks, nthreads: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    B, n = x.shape
    D = n.bit_length() - 1
    bs = np.ascontiguousarray(np.asarray(bs, dtype=np.uint64))
    ks = np.ascontiguousarray(np.asarray(ks, dtype=np.uint64))
    out = np.empty(ks.shape[0], dtype=np.int64)
    lib().orc_conv_batched_cells_i64(D, x.ctypes.data, y.ctypes.data, bs.ctypes.data, ks.ctypes.data,
                                     ks.shape[0], out.ctypes.data, nthreads)
    return out


def max_threads() -> int:
    return int(lib().orc_max_threads())
