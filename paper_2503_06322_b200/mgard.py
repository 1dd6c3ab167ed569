"""MGARD reduction path on B200: the drop-in for hpdr/mgard (codec.py, transform.py,
quantize.py).  Every function runs on the GPU through libhpdr_b200.so; there is no CPU
fallback.

Signatures, blob layout and exception classes follow the reference:
  mgard_compress(u, eb_rel, dict_size=4096, adapter=None, cache=None, value_range=None) -> bytes
      (codec.py:25-56)
  mgard_decompress(data, adapter=None, cache=None) -> TensorData          (codec.py:59-113)
  decompose / recompose (transform.py:287-348), quantize / dequantize (quantize.py:50-125)
plus the north-star wrapper compress(data, error_bound, norm) / decompress(blob).
``adapter`` is accepted and ignored (the reference's CPU execution adapters have no role
on the device); ``device=`` selects the GPU.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib, hostmem
from ._lib import check, dims_arg, lib
from .context import Context, ContextCache, ContextKey
from .errors import CorruptStreamError, ValidationError
from .hierarchy import Hierarchy, build_hierarchy
from .tensor import DTYPE_CODES, DTYPE_FROM_CODE, DType, TensorData

DEFAULT_DICT_SIZE = 4096   # quantize.py:19


@dataclass
class CoefficientSet:
    """Multilevel coefficients in finest-grid order (transform.py:32-42)."""

    dims: tuple
    values: np.ndarray
    level_counts: list
    u_min: float
    u_max: float
    source_dtype: DType = DType.F64


@dataclass
class QuantizedSet:
    """quantize.py:34-47."""

    dims: tuple
    keys: np.ndarray
    outlier_idx: np.ndarray
    outlier_bins: np.ndarray
    coarse_values: np.ndarray
    bin_width: float
    eb_abs: float
    dict_size: int
    u_min: float
    u_max: float
    total_levels: int
    source_dtype: DType = DType.F64


# ----------------------------------------------------------------------------- helpers
def _native(cache: ContextCache | None, key: ContextKey | None, device: int | None, obj=None):
    if cache is not None and key is not None:
        # a CUDA tensor argument runs on its own GPU; otherwise device=, else the cache's device
        dev = device
        if dev is None and getattr(getattr(obj, "device", None), "type", None) == "cuda":
            dev = _lib.default_device(obj)
        return cache.acquire(key, device=dev).native
    return _lib.default_context(device, obj)


def _as_input(u):
    """(address, dims, dtype code, keep-alive) of a TensorData / ndarray / torch tensor."""
    if isinstance(u, TensorData):
        if u.dtype not in (DType.F32, DType.F64):
            raise ValidationError(f"lossy compression needs F32/F64, got {u.dtype}")
        return u.values.ctypes.data, u.dims, DTYPE_CODES[u.dtype], u.values
    if isinstance(u, np.ndarray):
        if u.dtype not in (np.float32, np.float64):
            raise ValidationError(f"lossy compression needs F32/F64, got {u.dtype}")
        arr = np.ascontiguousarray(u)
        if arr.ndim < 1 or arr.ndim > 4:
            raise ValidationError(f"rank {arr.ndim} outside 1..4")
        return arr.ctypes.data, tuple(arr.shape), 0 if arr.dtype == np.float32 else 1, arr
    if hasattr(u, "data_ptr") and hasattr(u, "is_contiguous"):   # torch.Tensor (host, pinned or CUDA)
        import torch

        if u.dtype not in (torch.float32, torch.float64):
            raise ValidationError(f"lossy compression needs F32/F64, got {u.dtype}")
        t = u.contiguous()
        if t.dim() < 1 or t.dim() > 4:
            raise ValidationError(f"rank {t.dim()} outside 1..4")
        return int(t.data_ptr()), tuple(t.shape), 0 if t.dtype == torch.float32 else 1, t
    raise ValidationError(f"unsupported input type {type(u)}")


def _dims_ok(dims):
    dims = tuple(int(d) for d in dims)
    if not dims:
        raise ValidationError("dims must be non-empty")
    if len(dims) > 4:
        raise ValidationError(f"rank {len(dims)} exceeds maximum 4")
    if any(d < 1 for d in dims):
        raise ValidationError(f"every extent must be >= 1, got {dims}")
    return dims


# ----------------------------------------------------------------------------- codec
# blob size of the last call per (context, dims, dtype, eb_rel, dict_size, mode): the next result's
# bytes object is created (and first-touched) from it while the GPU works
_SIZE_HINTS: dict = {}


def mgard_compress(u, eb_rel: float, dict_size: int = DEFAULT_DICT_SIZE, adapter=None,
                   cache: ContextCache | None = None, value_range=None, *, device: int | None = None,
                   out=None):
    """Decompose, quantize against the error bound and entropy-code the keys on the GPU.

    Returns ``bytes`` identical to the reference blob.  With ``out`` (a host numpy uint8
    array, pinned or not, or a CUDA tensor) the blob is written there and its length is
    returned instead.
    """
    addr, dims, code, keep = _as_input(u)
    dims = _dims_ok(dims)
    hostmem.register_input(keep)   # a reused large ndarray is page-locked (DMA without staging)
    key = None
    if cache is not None:
        key = ContextKey.make("mgard", dims, DTYPE_FROM_CODE[code].value, eb_rel=float(eb_rel),
                              dict_size=int(dict_size))
    ctx = _native(cache, key, device, u if getattr(u, "is_cuda", False) else out)
    has = value_range is not None
    r0, r1 = (float(value_range[0]), float(value_range[1])) if has else (0.0, 0.0)
    n = C.c_uint64()
    if out is None:
        # a fresh `bytes` (codec.py:56), created once the size is known so that the blob streams
        # into it behind the payload encode
        hkey = (id(ctx), tuple(dims), code, float(eb_rel), int(dict_size), has)
        sink = _lib.BytesSink(_SIZE_HINTS.get(hkey, 0))
        try:
            check(lib().hpdr_mgard_compress_alloc(ctx.handle, C.c_void_p(addr), code, len(dims), dims_arg(dims),
                                                  float(eb_rel), int(dict_size), int(has), r0, r1, sink.fn, None,
                                                  C.byref(n)))
        finally:
            del keep
            blob = sink.take()
        if len(_SIZE_HINTS) > 64:
            _SIZE_HINTS.clear()
        _SIZE_HINTS[hkey] = int(n.value)
        return blob
    out_addr, out_cap = _lib.ptr(out), int(out.nbytes)
    check(lib().hpdr_mgard_compress(ctx.handle, C.c_void_p(addr), code, len(dims), dims_arg(dims),
                                    float(eb_rel), int(dict_size), int(has), r0, r1,
                                    C.c_void_p(out_addr) if out_addr else None, out_cap, C.byref(n)))
    del keep
    if n.value > out_cap:
        check(lib().hpdr_mgard_fetch(ctx.handle, C.c_void_p(out_addr), out_cap))
    return int(n.value)


def blob_info(data) -> tuple:
    """(dtype, dims) parsed from a blob header without decoding it."""
    buf = np.frombuffer(memoryview(data), dtype=np.uint8)
    dt, rk = C.c_int(), C.c_int()
    dims = (C.c_uint64 * 4)()
    check(lib().hpdr_mgard_peek(C.c_void_p(buf.ctypes.data if buf.size else 0), buf.size, C.byref(dt),
                                C.byref(rk), dims))
    return dt.value, tuple(int(dims[i]) for i in range(min(rk.value, 4))), rk.value


def mgard_decompress(data, adapter=None, cache: ContextCache | None = None, *, device: int | None = None,
                     out=None) -> TensorData:
    """Decode, dequantize and recompose on the GPU (codec.py:59-113).  ``data`` may also be a
    CUDA uint8 tensor (a device-resident blob, read in place) or a host uint8 tensor."""
    if hasattr(data, "numpy") and hasattr(data, "data_ptr") and not getattr(data, "is_cuda", False):
        data = data.numpy()   # host torch tensor (pinned or not): a zero-copy numpy view
    if getattr(data, "is_cuda", False):
        addr, size = int(data.data_ptr()), int(data.numel() * data.element_size())
        buf = data[: min(size, 128)].cpu().numpy().view(np.uint8)   # header only
    else:
        buf = np.frombuffer(memoryview(data), dtype=np.uint8)
        addr, size = (buf.ctypes.data if buf.size else 0), buf.size
    code, dims, rank = blob_info(buf)
    ctx = _native(None, None, device, data if getattr(data, "is_cuda", False) else out)
    if cache is not None and code in DTYPE_FROM_CODE and 1 <= rank <= 4:
        # the reference keys the context by the stored eb_rel / dict_size (codec.py:88-93)
        hdr = 1 + 8 * rank
        eb_rel = float(np.frombuffer(buf[hdr + 1:hdr + 9].tobytes(), "<f8")[0]) if buf.size >= hdr + 13 else 0.0
        dsz = int(np.frombuffer(buf[hdr + 9:hdr + 13].tobytes(), "<u4")[0]) if buf.size >= hdr + 13 else 0
        key = ContextKey.make("mgard", dims, DTYPE_FROM_CODE[code].value, eb_rel=eb_rel, dict_size=dsz)
        ctx = _native(cache, key, device, data if getattr(data, "is_cuda", False) else out)
    dt = DTYPE_FROM_CODE.get(code, DType.F64)
    n_elem = int(np.prod(dims)) if dims and 1 <= rank <= 4 else 0
    if out is None:
        res = hostmem.empty(dims if (1 <= rank <= 4 and all(d >= 1 for d in dims)) else (max(n_elem, 1),),
                            dt.np_dtype)
    else:
        res = out
    check(lib().hpdr_mgard_decompress(ctx.handle, C.c_void_p(addr), size, C.c_void_p(_lib.ptr(res)),
                                      int(res.nbytes)))
    if out is not None:
        return out
    return TensorData(dims, dt, res)


# ----------------------------------------------------------------------------- north-star API
def _abs_mapping(error_bound: float):
    """Absolute L-inf bound e as (eb_rel, value_range) with eb_rel*(hi-lo) == e exactly."""
    e = float(error_bound)
    if not (e > 0 and math.isfinite(e)):
        raise ValidationError(f"error_bound must be positive and finite, got {error_bound}")
    k = 0
    while e / 2.0 ** k >= 1.0:
        k += 1
    return e / 2.0 ** k, (0.0, 2.0 ** k)


def compress(data, error_bound: float, norm: str = "linf", mode: str = "abs",
             dict_size: int = DEFAULT_DICT_SIZE, *, device: int | None = None, cache=None, out=None):
    """compress(data, error_bound, norm) of the north star.

    ``mode="abs"`` bounds max|x - x'| by ``error_bound``; ``mode="rel"`` by
    ``error_bound * (max(x) - min(x))``.  ``norm="l2"`` uses the same quantizer (RMS <= max
    <= eb), so the blob stays reference-compatible.
    """
    if norm not in ("linf", "l2", "inf", "Linf", "L2"):
        raise ValidationError(f"unknown norm {norm!r}")
    if mode == "rel":
        return mgard_compress(data, error_bound, dict_size, cache=cache, device=device, out=out)
    if mode != "abs":
        raise ValidationError(f"mode must be 'abs' or 'rel', got {mode!r}")
    eb_rel, vr = _abs_mapping(error_bound)
    return mgard_compress(data, eb_rel, dict_size, cache=cache, value_range=vr, device=device, out=out)


def decompress(blob, *, device: int | None = None, out=None):
    """decompress(blob) of the north star: the reconstructed array."""
    r = mgard_decompress(blob, device=device, out=out)
    return r if out is not None else r.values


# ----------------------------------------------------------------------------- stages
def decompose(u, h: Hierarchy | None = None, adapter=None, ctx: Context | None = None,
              *, device: int | None = None) -> CoefficientSet:
    """transform.py:287-323 on the GPU."""
    addr, dims, code, keep = _as_input(u)
    dims = _dims_ok(dims)
    if h is not None and tuple(h.dims) != dims:
        raise ValidationError(f"dims {dims} do not match hierarchy {h.dims}")
    h = h or build_hierarchy(dims)
    nat = ctx.native if ctx is not None else _lib.default_context(device)
    coef = np.empty(dims, dtype=np.float64)
    mn, mx = C.c_double(), C.c_double()
    check(lib().hpdr_decompose(nat.handle, C.c_void_p(addr), code, len(dims), dims_arg(dims),
                               C.c_void_p(coef.ctypes.data), C.byref(mn), C.byref(mx)))
    del keep
    return CoefficientSet(dims, coef, h.level_element_counts(), mn.value, mx.value, DTYPE_FROM_CODE[code])


def recompose(c: CoefficientSet, h: Hierarchy | None = None, adapter=None, ctx: Context | None = None,
              *, device: int | None = None) -> np.ndarray:
    """transform.py:326-348 on the GPU."""
    dims = _dims_ok(c.dims)
    if h is not None and tuple(h.dims) != dims:
        raise ValidationError(f"dims {dims} do not match hierarchy {h.dims}")
    nat = ctx.native if ctx is not None else _lib.default_context(device)
    vals = np.ascontiguousarray(c.values, dtype=np.float64)
    out = np.empty(dims, dtype=np.float64)
    check(lib().hpdr_recompose(nat.handle, C.c_void_p(vals.ctypes.data), len(dims), dims_arg(dims),
                               C.c_void_p(out.ctypes.data)))
    return out


def quantize(c: CoefficientSet, h: Hierarchy | None = None, eb_rel: float = 1e-3,
             dict_size: int = DEFAULT_DICT_SIZE, value_range=None, *, device: int | None = None) -> QuantizedSet:
    """quantize.py:50-98 on the GPU."""
    dims = _dims_ok(c.dims)
    vals = np.ascontiguousarray(c.values, dtype=np.float64)
    n = vals.size
    nat = _lib.default_context(device)
    keys = np.empty(n, np.uint32)
    oidx = np.empty(n, np.uint64)
    obins = np.empty(n, np.int64)
    cv = np.empty(16, np.float64)
    no, nco = C.c_uint64(), C.c_uint64()
    eb_abs, binw = C.c_double(), C.c_double()
    lv = C.c_uint32()
    has = value_range is not None
    r0, r1 = (float(value_range[0]), float(value_range[1])) if has else (0.0, 0.0)
    check(lib().hpdr_quantize(nat.handle, C.c_void_p(vals.ctypes.data), len(dims), dims_arg(dims),
                              float(c.u_min), float(c.u_max), float(eb_rel), int(dict_size), int(has), r0, r1,
                              C.c_void_p(keys.ctypes.data), C.c_void_p(oidx.ctypes.data),
                              C.c_void_p(obins.ctypes.data), C.byref(no), C.c_void_p(cv.ctypes.data),
                              C.byref(nco), C.byref(eb_abs), C.byref(binw), C.byref(lv)))
    vmin, vmax = (c.u_min, c.u_max) if not has else (r0, r1)
    return QuantizedSet(dims, keys, oidx[: no.value].copy(), obins[: no.value].copy(), cv[: nco.value].copy(),
                        binw.value, eb_abs.value, int(dict_size), vmin, vmax, int(lv.value), c.source_dtype)


def dequantize(q: QuantizedSet, h: Hierarchy | None = None, *, device: int | None = None) -> CoefficientSet:
    """quantize.py:101-125 on the GPU (same kernels as the fused decode path)."""
    dims = _dims_ok(q.dims)
    h = h or build_hierarchy(dims)
    keys = np.ascontiguousarray(q.keys, dtype=np.uint32).reshape(-1)
    nat = _lib.default_context(device)
    out = np.empty(dims, np.float64)
    oidx = np.ascontiguousarray(q.outlier_idx, dtype=np.uint64)
    obins = np.ascontiguousarray(q.outlier_bins, dtype=np.int64)
    cv = np.ascontiguousarray(q.coarse_values, dtype=np.float64)
    check(lib().hpdr_dequantize(nat.handle, C.c_void_p(keys.ctypes.data), keys.size, len(dims), dims_arg(dims),
                                int(q.dict_size), float(q.bin_width), C.c_void_p(oidx.ctypes.data),
                                C.c_void_p(obins.ctypes.data), oidx.size, C.c_void_p(cv.ctypes.data), cv.size,
                                C.c_void_p(out.ctypes.data)))
    return CoefficientSet(dims, out, h.level_element_counts(), q.u_min, q.u_max, q.source_dtype)


__all__ = ["CoefficientSet", "QuantizedSet", "Hierarchy", "build_hierarchy", "mgard_compress",
           "mgard_decompress", "compress", "decompress", "decompose", "recompose", "quantize", "dequantize",
           "blob_info", "DEFAULT_DICT_SIZE", "CorruptStreamError"]
