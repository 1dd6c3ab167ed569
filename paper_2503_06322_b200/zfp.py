"""Fixed-rate block coder on the GPU: drop-in for the reference's ``hpdr.zfp``
(hpdr/zfp.py:270-353).

Streams are byte-identical to the reference's: ``"<BBB"`` rank, dtype code, rate, the dims as
u64, then every 4^d block packed into exactly ``1 + e_bits + rate*4^d`` bits.  All block work
(gather with edge replication, common exponent, reversible lifting, negabinary bit planes) runs in
``k_zfp_encode`` / ``k_zfp_decode`` of libhpdr_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib, hostmem
from ._lib import check, dims_arg, lib
from .errors import ValidationError
from .tensor import DTYPE_CODES, DTYPE_FROM_CODE, DType, TensorData

BLOCK_SIDE = 4       # zfp.py:30
MAX_BLOCK_RANK = 3   # zfp.py:31
E_BITS = {DType.F32: 8, DType.F64: 11}
Q_BITS = {DType.F32: 32, DType.F64: 64}


def compressed_size(dims, dtype: DType, rate: int) -> int:
    """Exact stream size in bytes for the fix-rate contract (zfp.py:270-278)."""
    dims = tuple(int(d) for d in dims)
    if dtype not in Q_BITS:
        raise ValidationError(f"fix-rate compression needs F32/F64, got {dtype}")
    size = C.c_uint64()
    check(lib().hpdr_zfp_compressed_size(DTYPE_CODES[dtype], len(dims), dims_arg(dims), int(rate), C.byref(size)))
    return int(size.value)


def _as_field(u):
    """(address, dims, dtype code, keep-alive) of a TensorData / ndarray / torch tensor."""
    if isinstance(u, TensorData):
        if u.dtype not in Q_BITS:
            raise ValidationError(f"fix-rate compression needs F32/F64, got {u.dtype}")
        return u.values.ctypes.data, u.dims, DTYPE_CODES[u.dtype], u.values
    if isinstance(u, np.ndarray):
        if u.dtype not in (np.float32, np.float64):
            raise ValidationError(f"fix-rate compression needs F32/F64, got {u.dtype}")
        arr = np.ascontiguousarray(u)
        return arr.ctypes.data, tuple(arr.shape), 0 if arr.dtype == np.float32 else 1, arr
    if hasattr(u, "data_ptr") and hasattr(u, "is_contiguous"):   # torch.Tensor (host, pinned or CUDA)
        import torch

        if u.dtype not in (torch.float32, torch.float64):
            raise ValidationError(f"fix-rate compression needs F32/F64, got {u.dtype}")
        t = u.contiguous()
        return int(t.data_ptr()), tuple(t.shape), 0 if t.dtype == torch.float32 else 1, t
    raise ValidationError(f"unsupported input type {type(u)}")


def zfp_compress(u, rate: int, adapter=None, *, device: int | None = None, out=None):
    """zfp_compress (zfp.py:281-308).  ``adapter`` is accepted and ignored.  Returns ``bytes``; with
    ``out`` (host uint8 array, pinned or not, or a CUDA uint8 tensor) the stream is written there
    and its length returned."""
    addr, dims, code, keep = _as_field(u)
    dims = tuple(int(d) for d in dims)
    if not dims:
        raise ValidationError("dims must be non-empty")
    hostmem.register_input(keep)
    ctx = _lib.default_context(device, u if getattr(u, "is_cuda", False) else out)
    n = C.c_uint64()
    if out is None:
        size = compressed_size(dims, DTYPE_FROM_CODE[code], rate) if len(dims) <= MAX_BLOCK_RANK else 0
        b, p = _lib.new_bytes(size) if size else (b"", 0)
        check(lib().hpdr_zfp_compress(ctx.handle, C.c_void_p(addr), code, len(dims), dims_arg(dims), int(rate),
                                      C.c_void_p(p) if p else None, size, C.byref(n)))
        del keep
        return b
    check(lib().hpdr_zfp_compress(ctx.handle, C.c_void_p(addr), code, len(dims), dims_arg(dims), int(rate),
                                  C.c_void_p(_lib.ptr(out)), int(out.nbytes), C.byref(n)))
    del keep
    return int(n.value)


def _peek(addr: int, size: int) -> tuple:
    dt, rk, rate = C.c_int(), C.c_int(), C.c_uint32()
    dims = (C.c_uint64 * 3)()
    check(lib().hpdr_zfp_peek(C.c_void_p(addr) if addr else None, size, C.byref(dt), C.byref(rk), dims,
                              C.byref(rate)))
    return DTYPE_FROM_CODE[dt.value], tuple(int(dims[i]) for i in range(rk.value)), int(rate.value)


def stream_info(data) -> tuple:
    """(dtype, dims, rate) of a fixed-rate stream, with zfp_decompress's header checks."""
    buf = np.frombuffer(memoryview(data), dtype=np.uint8)
    return _peek(buf.ctypes.data if buf.size else 0, buf.size)


def zfp_decompress(data, adapter=None, *, device: int | None = None, out=None) -> TensorData:
    """zfp_decompress (zfp.py:311-353).  ``data`` may be bytes-like or a CUDA uint8 tensor."""
    if hasattr(data, "data_ptr"):   # torch tensor: CUDA (read in place) or host / pinned
        addr, size = int(data.data_ptr()), int(data.numel() * data.element_size())
        dtype, dims, _ = _peek(addr, size)   # hpdr_zfp_peek copies a device header itself
    else:
        buf = np.frombuffer(memoryview(data), dtype=np.uint8)
        addr, size = (buf.ctypes.data if buf.size else 0), buf.size
        dtype, dims, _ = stream_info(buf)
    ctx = _lib.default_context(device, data if getattr(data, "is_cuda", False) else out)
    res = hostmem.empty(dims, dtype.np_dtype) if out is None else out
    check(lib().hpdr_zfp_decompress(ctx.handle, C.c_void_p(addr), size, C.c_void_p(_lib.ptr(res)), int(res.nbytes)))
    if out is not None:
        return out
    return TensorData(dims, dtype, res)


def compress_pipelined(arr, rate: int, *, chunk_planes: int = 0, chunks=None, device: int | None = None, out=None,
                       trace: bool = False):
    """The streams pipeline with the fixed-rate reducer -> HPDR container (pipeline id 1) of
    per-slab reference-identical streams.  Decompress with ``pipeline.decompress_pipelined``.
    With ``trace`` returns (bytes, (K, 6) array of H2D / compute / D2H start-end times in ms)."""
    addr, dims, code, keep = _as_field(arr)
    dims = tuple(int(d) for d in dims)
    ctx = _lib.default_context(device, arr if getattr(arr, "is_cuda", False) else out)
    lst = None if chunks is None else np.ascontiguousarray(chunks, dtype=np.uint64)
    n = C.c_uint64()

    def run(buf, tr):
        return lib().hpdr_pipeline_zfp_compress(
            ctx.handle, C.c_void_p(addr), code, len(dims), dims_arg(dims), int(rate), int(chunk_planes),
            C.c_void_p(lst.ctypes.data) if lst is not None else None, 0 if lst is None else len(lst),
            C.c_void_p(_lib.ptr(buf)) if buf is not None else None, 0 if buf is None else int(buf.nbytes),
            C.byref(n), C.c_void_p(tr.ctypes.data) if tr is not None else None)

    rc = run(None, None) if out is None else _lib.BUFFER   # size query (fixed-rate: exact)
    if out is None and rc != _lib.BUFFER:
        check(rc)
    buf = _lib.pinned_scratch(n.value) if out is None else out   # pinned: full-speed D2H, then one bytes copy
    from .container import read_container

    tr = None
    if trace:
        if lst is not None:
            k = len(lst)
        else:   # the runner's default: ~64 MB of input per chunk in whole 4-plane rows
            plane = int(np.prod(dims[1:])) * (4 if code == 0 else 8)
            cp = chunk_planes or max(4, (64 << 20) // plane // 4 * 4)
            k = -(-dims[0] // cp)
        tr = np.zeros(6 * k, np.float64)
    check(run(buf, tr))
    del keep
    data = _lib.bytes_from(buf, n.value) if out is None else int(n.value)
    if not trace:
        return data
    h, _ = read_container(buf[: n.value])
    return data, tr[: 6 * len(h.chunks)].reshape(-1, 6)


__all__ = ["BLOCK_SIDE", "MAX_BLOCK_RANK", "compress_pipelined", "compressed_size", "stream_info", "zfp_compress",
           "zfp_decompress"]
