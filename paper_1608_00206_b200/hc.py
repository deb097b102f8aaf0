"""Thin ctypes binding over libhc.so (include/hc.h).  Argument marshalling only: every step
of the convolution runs in the CUDA kernels behind the C ABI.  torch supplies device
memory and streams; nothing here computes on the host, and there is no fallback: a
missing or unloadable libhc.so raises at import time.
"""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HC_LIB") or os.path.join(_HERE, "libhc.so")  # HC_LIB: development variants
HEADER = os.path.join(os.path.dirname(_HERE), "include", "hc.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libhc.so not built at {LIB_PATH}; run `python -m paper_1608_00206_b200.build` "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

HC_INT64, HC_FP64 = 0, 1
STATUS = {0: "HC_OK", 1: "HC_ERR_INVALID_DIM", 2: "HC_ERR_DTYPE", 3: "HC_ERR_NULL", 4: "HC_ERR_ALIGN",
          5: "HC_ERR_DEVICE", 6: "HC_ERR_CAPACITY", 7: "HC_ERR_CUDA", 9: "HC_ERR_SHARD"}

_P = ctypes.c_void_p
_I = ctypes.c_int
_U64 = ctypes.c_uint64
_lib.hc_status_str.argtypes = [_I]
_lib.hc_status_str.restype = ctypes.c_char_p
_lib.hc_in_len.argtypes = [_I]
_lib.hc_in_len.restype = _U64
_lib.hc_out_len.argtypes = [_I]
_lib.hc_out_len.restype = _U64
_lib.hc_plan_create.argtypes = [ctypes.POINTER(_P), _I, _I, _I, _I]
_lib.hc_plan_destroy.argtypes = [_P]
_lib.hc_shard_info.argtypes = [_P, _I, ctypes.POINTER(_U64), ctypes.POINTER(_U64)]
_lib.hc_shard_range.argtypes = [_I, _I, _I, ctypes.POINTER(_U64), ctypes.POINTER(_U64)]
_lib.hc_convolve.argtypes = [_P, _P, _P, _P, _P]
_lib.hc_convolve_sharded.argtypes = [_P, _P, _P, _P, _P]
_lib.hc_convolve_batched.argtypes = [_I, _I, _I, _P, _P, _P, _P]
_lib.hc_convolve_host.argtypes = [_P, _P, _P, _P, _P]
_lib.hc_ep_range.argtypes = [_I, _I, _I, _I] + [ctypes.POINTER(_U64)] * 4
_lib.hc_ep_create.argtypes = [ctypes.POINTER(_P), _I, _I, _I, _I, _I]
_lib.hc_ep_destroy.argtypes = [_P]
_lib.hc_ep_local.argtypes = [_P, _P, _P, _P, _P]
_lib.hc_ep_finish.argtypes = [_P, _P, _P, _P]
_lib.hc_ep_finish_peer.argtypes = [_P, ctypes.POINTER(_P), _P, _P]
_lib.hc_convolve_difference.argtypes = [_P, _P, _P, _P, _P]
_lib.hc_carries_work_len.argtypes = [_I]
_lib.hc_carries_work_len.restype = _U64
_lib.hc_apply_carries.argtypes = [_I, _I, _P, _P, _P, _P]
_lib.hc_conv1d.argtypes = [_P, _P, _P, _P, _P, _P, _P]
_lib.hc_maxconv_pnorm.argtypes = [_P, _P, _P, _P, ctypes.c_double, _I, _P]
_lib.hc_launch_count.restype = _U64
_lib.hc_prof_enable.argtypes = [_I]
_lib.hc_prof_read.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_U64)]


class HCError(RuntimeError):
    def __init__(self, code: int, where: str = ""):
        self.code = code
        super().__init__(f"{where}: {STATUS.get(code, code)} ({_lib.hc_status_str(code).decode()})")


def _ok(code: int, where: str):
    if code != 0:
        raise HCError(code, where)


def exported_symbols():
    """Names declared in include/hc.h (the test suite checks libhc.so exports each)."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(hc_[a-z0-9_]+)\s*\(", text)))


def in_len(D: int) -> int:
    return int(_lib.hc_in_len(D))


def out_len(D: int) -> int:
    return int(_lib.hc_out_len(D))


def shard_range(D: int, ngpu: int, rank: int):
    """Host-only: [z_begin, z_end) owned by `rank` of `ngpu` (hc_shard_range)."""
    b, e = _U64(), _U64()
    _ok(_lib.hc_shard_range(D, ngpu, rank, ctypes.byref(b), ctypes.byref(e)), "hc_shard_range")
    return int(b.value), int(e.value)


def _dtype_code(dtype) -> int:
    s = str(dtype)
    if s.endswith("int64"):
        return HC_INT64
    if s.endswith("float64"):
        return HC_FP64
    raise TypeError(f"hypercube convolution supports int64 and float64, got {dtype}")


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _dev(t, n, dtype_code, name):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    import torch
    cur = torch.cuda.current_device()
    if t.device.index != cur:
        raise ValueError(f"{name} is on {t.device} but the current device is cuda:{cur} "
                         "(plans and launches use the current device)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.numel() != n:
        raise ValueError(f"{name} must have {n} elements, got {t.numel()}")
    if _dtype_code(t.dtype) != dtype_code:
        raise TypeError(f"{name} dtype {t.dtype} does not match the plan")
    return ctypes.c_void_p(t.data_ptr())


class Plan:
    """hc_plan_create(D, dtype, ngpu, rank)."""

    def __init__(self, D: int, dtype="float64", ngpu: int = 1, rank: int = 0):
        self.D, self.ngpu, self.rank = D, ngpu, rank
        self.dtype_code = _dtype_code(dtype)
        h = _P()
        _ok(_lib.hc_plan_create(ctypes.byref(h), D, self.dtype_code, ngpu, rank), "hc_plan_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _lib.hc_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def shard_info(self, rank=None):
        b, e = _U64(), _U64()
        _ok(_lib.hc_shard_info(self._h, self.rank if rank is None else rank, ctypes.byref(b), ctypes.byref(e)),
            "hc_shard_info")
        return int(b.value), int(e.value)

    def convolve(self, x, y, z, stream=None):
        n, m = in_len(self.D), out_len(self.D)
        _ok(_lib.hc_convolve(self._h, _dev(x, n, self.dtype_code, "x"), _dev(y, n, self.dtype_code, "y"),
                             _dev(z, m, self.dtype_code, "z"), _P(_stream_ptr(stream))), "hc_convolve")
        return z

    def convolve_sharded(self, x, y, z_shard, stream=None):
        n = in_len(self.D)
        b, e = self.shard_info()
        _ok(_lib.hc_convolve_sharded(self._h, _dev(x, n, self.dtype_code, "x"), _dev(y, n, self.dtype_code, "y"),
                                     _dev(z_shard, e - b, self.dtype_code, "z_shard"), _P(_stream_ptr(stream))),
            "hc_convolve_sharded")
        return z_shard

    def convolve_difference(self, x, y, z, stream=None):
        """hc_convolve_difference: z[k] = P(X - Y = k - 1) digit-wise."""
        n, m = in_len(self.D), out_len(self.D)
        _ok(_lib.hc_convolve_difference(self._h, _dev(x, n, self.dtype_code, "x"), _dev(y, n, self.dtype_code, "y"),
                                        _dev(z, m, self.dtype_code, "z"), _P(_stream_ptr(stream))),
            "hc_convolve_difference")
        return z

    def maxconv_pnorm(self, x, y, z, p: float, round_to_int: bool = False, stream=None):
        """hc_maxconv_pnorm: p-norm estimate of max_{i+j=k} x[i] y[j]."""
        n, m = in_len(self.D), out_len(self.D)
        _ok(_lib.hc_maxconv_pnorm(self._h, _dev(x, n, self.dtype_code, "x"), _dev(y, n, self.dtype_code, "y"),
                                  _dev(z, m, self.dtype_code, "z"), float(p), 1 if round_to_int else 0,
                                  _P(_stream_ptr(stream))), "hc_maxconv_pnorm")
        return z

    def convolve_host(self, x_host, y_host, z_host, stream=None):
        """Host (CPU, ideally pinned) tensors; copies in, computes, copies this rank's share out."""
        n = in_len(self.D)
        b, e = self.shard_info()
        for t, want, name in ((x_host, n, "x"), (y_host, n, "y"), (z_host, e - b, "z")):
            if t.is_cuda or not t.is_contiguous() or t.numel() != want or _dtype_code(t.dtype) != self.dtype_code:
                raise ValueError(f"{name}: need a contiguous host tensor of {want} {self.dtype_code} elements")
        _ok(_lib.hc_convolve_host(self._h, _P(x_host.data_ptr()), _P(y_host.data_ptr()), _P(z_host.data_ptr()),
                                  _P(_stream_ptr(stream))), "hc_convolve_host")
        return z_host


def convolve_batched(x, y, z, stream=None):
    """x, y: [B, 2^D] CUDA tensors; z: [B, 3^D]."""
    if x.dim() != 2 or x.shape != y.shape:
        raise ValueError("x, y must be [B, 2^D]")
    B, n = x.shape
    D = n.bit_length() - 1
    if (1 << D) != n:
        raise ValueError("row length must be 2^D")
    code = _dtype_code(x.dtype)
    _ok(_lib.hc_convolve_batched(B, D, code, _dev(x, B * n, code, "x"), _dev(y, B * n, code, "y"),
                                 _dev(z, B * out_len(D), code, "z"), _P(_stream_ptr(stream))),
        "hc_convolve_batched")
    return z


def convolve(x, y, z=None, stream=None):
    """One-shot convenience: plan + hc_convolve on CUDA tensors x, y (2^D each)."""
    import torch
    n = x.numel()
    D = n.bit_length() - 1
    if z is None:
        z = torch.empty(3 ** D, dtype=x.dtype, device=x.device)
    Plan(D, x.dtype).convolve(x, y, z, stream)
    return z


def carries_work_len(D: int) -> int:
    return int(_lib.hc_carries_work_len(D))


def apply_carries(D: int, z, out, work=None, stream=None):
    """hc_apply_carries: out[m] = sum_{k: sum_b k_b 2^b = m} z[k]."""
    import torch
    code = _dtype_code(z.dtype)
    wl = carries_work_len(D)
    if wl and work is None:
        work = torch.empty(wl, dtype=z.dtype, device=z.device)
    wp = _dev(work, wl, code, "work") if wl else _P(0)
    _ok(_lib.hc_apply_carries(D, code, _dev(z, out_len(D), code, "z"), _dev(out, (2 << D) - 1, code, "out"), wp,
                              _P(_stream_ptr(stream))), "hc_apply_carries")
    return out


def conv1d(x, y, out=None, plan=None, stream=None, z_work=None):
    """Ordinary 1-D convolution of two length-2^D CUDA vectors through the carry-free
    (hypercube) convolution and the carries (hc_conv1d, PAPER.md 354-373); int64 with
    D >= 13 fuses the carries into the slab engine."""
    import torch
    n = x.numel()
    D = n.bit_length() - 1
    if n < 2 or (1 << D) != n:
        raise ValueError(f"conv1d: x must have length 2^D with D >= 1, got {n}")
    if y.numel() != n:
        raise ValueError(f"conv1d: y has {y.numel()} elements, x has {n}")
    code = _dtype_code(x.dtype)
    plan = plan or Plan(D, x.dtype)
    if plan.D != D or plan.dtype_code != code:
        raise ValueError(f"conv1d: plan is (D={plan.D}, dtype code {plan.dtype_code}), inputs are "
                         f"(D={D}, dtype code {code})")
    fused = code == HC_INT64 and D >= 13  # no z: plan-owned ring of slab buffers
    if z_work is None and not fused:
        z_work = torch.empty(3 ** D, dtype=x.dtype, device=x.device)
    if out is None:
        out = torch.empty((2 << D) - 1, dtype=x.dtype, device=x.device)
    wl = carries_work_len(D)
    work = None if (fused or wl == 0) else torch.empty(wl, dtype=x.dtype, device=x.device)
    # fused: z_work (if given) holds the pass-1 tiles in place; else the plan's slab ring
    zp = _P(0) if z_work is None else _dev(z_work, 3 ** D, code, "z_work")
    _ok(_lib.hc_conv1d(plan._h, _dev(x, n, code, "x"), _dev(y, n, code, "y"), zp,
                       _dev(out, (2 << D) - 1, code, "out"), _P(work.data_ptr()) if work is not None else _P(0),
                       _P(_stream_ptr(stream))), "hc_conv1d")
    return out


def ep_range(D: int, k: int, ngpu: int, rank: int):
    """Host-only (hc_ep_range): ((e_begin, e_end), (col_begin, col_end)) of `rank`."""
    v = [_U64() for _ in range(4)]
    _ok(_lib.hc_ep_range(D, k, ngpu, rank, *[ctypes.byref(t) for t in v]), "hc_ep_range")
    return (int(v[0].value), int(v[1].value)), (int(v[2].value), int(v[3].value))


class EPPlan:
    """Evaluation-point variant of the multi-GPU split (hc_ep_*; BASELINE north_star (4)).

    local(x, y, w): w[(e - e_begin), :] = conv_{D-k}(forward_top(x)[e], forward_top(y)[e]);
    exchange (ep_exchange, NCCL send/recv); finish(wt, z): interpolation over the top axes."""

    def __init__(self, D: int, k: int, dtype="float64", ngpu: int = 1, rank: int = 0):
        self.D, self.k, self.ngpu, self.rank = D, k, ngpu, rank
        self.dtype_code = _dtype_code(dtype)
        (self.e0, self.e1), (self.c0, self.c1) = ep_range(D, k, ngpu, rank)
        self.npoints, self.ncols_total = 3 ** k, 3 ** (D - k)
        h = _P()
        _ok(_lib.hc_ep_create(ctypes.byref(h), D, k, self.dtype_code, ngpu, rank), "hc_ep_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _lib.hc_ep_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def local(self, x, y, w, stream=None):
        n = in_len(self.D)
        _ok(_lib.hc_ep_local(self._h, _dev(x, n, self.dtype_code, "x"), _dev(y, n, self.dtype_code, "y"),
                             _dev(w, (self.e1 - self.e0) * self.ncols_total, self.dtype_code, "w"),
                             _P(_stream_ptr(stream))), "hc_ep_local")
        return w

    def finish_peer(self, w_ranks, z, stream=None):
        """hc_ep_finish_peer: interpolation reading every rank's w directly
        (w_ranks: one device tensor per rank -- peer-mapped buffers on a multi-GPU node)."""
        if len(w_ranks) != self.ngpu:
            raise ValueError("need one w buffer per rank")
        arr = (_P * self.ngpu)(*[_P(t.data_ptr()) for t in w_ranks])
        m = self.npoints * (self.c1 - self.c0)
        _ok(_lib.hc_ep_finish_peer(self._h, arr, _dev(z, m, self.dtype_code, "z"), _P(_stream_ptr(stream))),
            "hc_ep_finish_peer")
        return z

    def finish(self, wt, z, stream=None):
        m = self.npoints * (self.c1 - self.c0)
        _ok(_lib.hc_ep_finish(self._h, _dev(wt, m, self.dtype_code, "wt"), _dev(z, m, self.dtype_code, "z"),
                              _P(_stream_ptr(stream))), "hc_ep_finish")
        return z


def ep_exchange(w, wt, D: int, k: int, rank: int, world: int, dist=None):
    """The all-to-all of the evaluation-point variant: rank g holds w[e - e_begin_g, :] for
    its points; afterwards wt[e, :] = w_of_owner(e)[e, col_begin_rank : col_end_rank] for all
    3^k points.  Point-to-point NCCL (or gloo) sends of contiguous row segments in one
    batch.  world == 1: a device copy."""
    ranges = [ep_range(D, k, world, r) for r in range(world)]
    (e0, e1), (c0, c1) = ranges[rank]
    if world == 1 or dist is None:
        wt.view(e1 - e0, c1 - c0).copy_(w.view(e1 - e0, -1)[:, c0:c1])
        return wt
    if w.is_cuda and dist.get_backend() == "gloo":
        # gloo's point-to-point is CPU-only: stage through host memory (testing several ranks
        # on one device); NCCL exchanges the device buffers directly
        wt_h = wt.cpu()
        ep_exchange(w.cpu(), wt_h, D, k, rank, world, dist)
        wt.copy_(wt_h)
        return wt
    wv = w.view(e1 - e0, -1)
    wtv = wt.view(3 ** k, c1 - c0)
    ops = []
    for h in range(world):
        (_, _), (hc0, hc1) = ranges[h]
        (he0, he1), _ = ranges[h]
        if h == rank:
            wtv[e0:e1].copy_(wv[:, c0:c1])
            continue
        for e in range(e0, e1):
            ops.append(dist.P2POp(dist.isend, wv[e - e0, hc0:hc1].contiguous(), h))
        for e in range(he0, he1):
            ops.append(dist.P2POp(dist.irecv, wtv[e], h))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return wt


def ep_peer_buffers(w, rank: int, world: int, dist=None):
    """f3: every rank's hc_ep_local output as a device tensor this process can read -- its own
    buffer, and CUDA IPC mappings of the others' (torch tensor reductions; lazy peer access,
    i.e. NVLink reads on a multi-GPU node).  Call once per buffer; the mappings stay valid
    while the owners keep their tensors."""
    if world == 1 or dist is None:
        return [w]
    from torch.multiprocessing.reductions import reduce_tensor
    mine = reduce_tensor(w)
    objs = [None] * world
    dist.all_gather_object(objs, mine)
    return [w if r == rank else f(*a) for r, (f, a) in enumerate(objs)]


def launch_count() -> int:
    return int(_lib.hc_launch_count())


def prof_enable(on: bool = True):
    _lib.hc_prof_enable(1 if on else 0)


def prof_reset():
    _lib.hc_prof_reset()


def prof_read(name: str):
    ms = ctypes.c_double()
    n = _U64()
    _ok(_lib.hc_prof_read(name.encode(), ctypes.byref(ms), ctypes.byref(n)), "hc_prof_read")
    return float(ms.value), int(n.value)
