"""Block partitioning along dim 0.

A field is split into contiguous dim-0 slabs; each slab becomes an independent,
reference-identical MGARD blob compressed with the GLOBAL value range, so the error bound of
the whole field holds and every blob decodes with the stock ``mgard_decompress``.

* ``compress_slabs`` / ``decompress_slabs``: one process, chunks in an HPDR container.
* ``distributed_compress`` / ``distributed_decompress``: one rank per GPU, each reducing its
  own block.  The only data that crosses ranks is an all-reduce of (-min, max) (16 bytes)
  and an all-gather of blob sizes (8 bytes per rank); NVLink carries nothing else.

``compressor`` / ``minmax`` are injectable so the partition and metadata logic can be
exercised on CPU (gloo) with the parity oracle; the defaults are the GPU path.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .container import ChunkEntry, ContainerHeader, read_container, slab_bounds, write_container
from .errors import ValidationError
from .tensor import DTYPE_CODES, DTYPE_FROM_CODE, DType


def _default_compressor(arr, eb_rel, dict_size, value_range):
    from .mgard import mgard_compress

    return mgard_compress(arr, eb_rel, dict_size, value_range=value_range)


def _default_decompressor(blob):
    from .mgard import mgard_decompress

    return mgard_decompress(blob).values


def _default_minmax(arr):
    from . import _lib

    ctx = _lib.default_context()
    a = np.ascontiguousarray(arr)
    return _lib.minmax(ctx, a.ctypes.data, 0 if a.dtype == np.float32 else 1, a.size)


def _dtype_code(arr) -> int:
    if arr.dtype == np.float32:
        return DTYPE_CODES[DType.F32]
    if arr.dtype == np.float64:
        return DTYPE_CODES[DType.F64]
    raise ValidationError(f"lossy compression needs F32/F64, got {arr.dtype}")


def compress_slabs(arr: np.ndarray, eb_rel: float, n_slabs: int, dict_size: int = 4096, value_range=None,
                   compressor=None, minmax=None) -> bytes:
    """Split along dim 0 into n_slabs blobs (global range) inside an HPDR container."""
    arr = np.ascontiguousarray(arr)
    code = _dtype_code(arr)
    n_slabs = max(1, min(int(n_slabs), arr.shape[0]))
    compressor = compressor or _default_compressor
    if value_range is None:
        value_range = tuple(float(v) for v in (minmax or _default_minmax)(arr))
    plane = int(np.prod(arr.shape[1:])) if arr.ndim > 1 else 1
    chunks, payloads = [], []
    for k in range(n_slabs):
        a, b = slab_bounds(arr.shape[0], n_slabs, k)
        blob = compressor(arr[a:b], eb_rel, dict_size, value_range)
        chunks.append(ChunkEntry(a * plane, (b - a) * plane, 0, len(blob)))
        payloads.append(blob)
    h = ContainerHeader(code, tuple(arr.shape), float(eb_rel), int(dict_size), value_range[0], value_range[1], chunks)
    return write_container(h, payloads)


def decompress_slabs(data, decompressor=None) -> np.ndarray:
    h, payloads = read_container(data)
    decompressor = decompressor or _default_decompressor
    out = np.empty(h.dims, dtype=DTYPE_FROM_CODE[h.dtype].np_dtype)
    flat = out.reshape(-1)
    for c, p in zip(h.chunks, payloads):
        flat[c.raw_offset:c.raw_offset + c.raw_size] = np.asarray(decompressor(bytes(p))).reshape(-1)
    return out


_HOOK_T = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double))


def _collective_device(group):
    import torch
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def allreduce_range(lo: float, hi: float, group=None) -> tuple:
    """Job-wide (min, max): one all-reduce of (-min, max), 16 bytes."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(lo), float(hi)
    t = torch.tensor([-lo, hi], dtype=torch.float64, device=_collective_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return -float(t[0]), float(t[1])


class RangeExchange:
    """Installs the job-wide min/max all-reduce as a device context's range hook
    (hpdr_ctx_set_range_hook) for the duration of a ``with`` block.

    A relative-mode ``mgard_compress`` of this rank's block then calls the all-reduce from inside
    the library as soon as the block's own min / max are known -- for a streamed host input that
    is after the last chunk has landed and been decomposed -- and quantizes with the job-wide
    range: the blob equals ``mgard_compress(block, eb_rel, value_range=global)`` and the exchange
    costs no extra pass over the field.  ``last`` holds the range of the latest call."""

    def __init__(self, ctx=None, group=None):
        from . import _lib

        self.ctx = ctx if ctx is not None else _lib.default_context()
        self.group = group
        self.last = None
        self.error = None
        self._cb = _HOOK_T(self._hook)

    def _hook(self, _user, pmin, pmax):
        try:
            self.last = allreduce_range(pmin[0], pmax[0], self.group)
            pmin[0], pmax[0] = self.last
            return 0
        except Exception as e:   # noqa: BLE001 - reported as a ValidationError by the library
            self.error = e
            return 1

    def __enter__(self):
        from . import _lib

        _lib.lib().hpdr_ctx_set_range_hook(self.ctx.handle, C.cast(self._cb, C.c_void_p), None)
        return self

    def __exit__(self, *exc):
        from . import _lib

        _lib.lib().hpdr_ctx_set_range_hook(self.ctx.handle, None, None)
        return False


def distributed_compress(block: np.ndarray, eb_rel: float, group=None, dict_size: int = 4096, value_range=None,
                         compressor=None, minmax=None, *, out=None):
    """Compress this rank's dim-0 block with the job-wide range.

    Returns (blob, sizes of every rank's blob, (vmin, vmax)); with ``out`` (a pinned / device
    buffer) the blob is written there and its length stands in for it.  Collectives: one
    all-reduce of two doubles (skipped when value_range is given) and one all-gather of one
    int64.  With the default (GPU) compressor the all-reduce runs inside the compress call
    (RangeExchange), overlapped with the block's transfer and decomposition.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    dev = _collective_device(group)
    if compressor is None and minmax is None and value_range is None:
        from . import _lib
        from .mgard import mgard_compress

        ctx = _lib.default_context(None, block if getattr(block, "is_cuda", False) else out)
        with RangeExchange(ctx, group) as rx:
            try:
                blob = mgard_compress(block, eb_rel, dict_size, out=out)
            except ValidationError:
                if rx.error is not None:
                    raise rx.error
                raise
        value_range = rx.last if rx.last is not None else value_range
        n = blob if out is not None else len(blob)
        sizes = [int(n)]
        if world > 1:
            t = torch.tensor([int(n)], dtype=torch.int64, device=dev)
            g = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(g, t, group=group)
            sizes = [int(x.item()) for x in g]
        return blob, sizes, value_range
    compressor = compressor or _default_compressor
    if value_range is None:
        lo, hi = (minmax or _default_minmax)(block)
        if world > 1:
            t = torch.tensor([-lo, hi], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
            lo, hi = -float(t[0]), float(t[1])
        value_range = (float(lo), float(hi))
    blob = compressor(np.ascontiguousarray(block), eb_rel, dict_size, value_range)
    sizes = [len(blob)]
    if world > 1:
        t = torch.tensor([len(blob)], dtype=torch.int64, device=dev)
        g = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(g, t, group=group)
        sizes = [int(x.item()) for x in g]
    return blob, sizes, value_range


def distributed_decompress(blob, decompressor=None):
    decompressor = decompressor or _default_decompressor
    return decompressor(blob)
