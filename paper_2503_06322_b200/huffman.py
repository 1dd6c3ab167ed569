"""Canonical Huffman codec on the GPU (drop-in for hpdr/huffman.py:361-435).

Stream layout (little-endian): dict_size u16, symbol count u64, lengths dict_size x u8,
decode-unit count u32, unit bit offsets u64 each, total_bits u64, packed bits MSB-first.
Histogram, encode and decode run on the device; the <= 65535-entry codebook is built on
the host with the reference's exact tie-breaking.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib
from .errors import ValidationError

BLOCK_SYMBOLS = 4096
MAX_CODE_LEN = 32
MAX_DICT_SIZE = 65535


@dataclass
class FrequencyTable:
    dict_size: int
    counts: np.ndarray

    def __post_init__(self):
        self.counts = np.asarray(self.counts, dtype=np.int64)
        if self.counts.size != self.dict_size:
            raise ValidationError("counts length must equal dict_size")


@dataclass
class HuffmanCodebook:
    dict_size: int
    lengths: np.ndarray
    codes: np.ndarray

    @property
    def max_length(self) -> int:
        return int(self.lengths.max(initial=0))

    def present_keys(self) -> np.ndarray:
        return np.nonzero(self.lengths)[0]


def _keys(keys):
    if hasattr(keys, "data_ptr"):        # torch tensor (host or CUDA), passed through
        return keys
    arr = np.ascontiguousarray(keys)
    if arr.dtype.kind not in "ui":
        raise ValidationError(f"keys must be unsigned integers, got {arr.dtype}")
    arr = arr.reshape(-1)
    if arr.dtype != np.uint32:
        if arr.size and (int(arr.max()) > 0xFFFFFFFF or int(arr.min()) < 0):
            raise ValidationError("keys exceed uint32")
        arr = arr.astype(np.uint32)
    return arr


def _dict(dict_size):
    d = int(dict_size)
    if d < 1 or d > MAX_DICT_SIZE:
        raise ValidationError(f"dict_size must be in [1, {MAX_DICT_SIZE}]")
    return d


def histogram(keys, dict_size: int, adapter=None, n_threads=None, *, device=None) -> FrequencyTable:
    """huffman.py:74-104 on the GPU."""
    arr = _keys(keys)
    d = _dict(dict_size)
    counts = np.zeros(d, np.int64)
    n = arr.numel() if hasattr(arr, "numel") else arr.size
    ctx = _lib.default_context(device)
    check(lib().hpdr_histogram(ctx.handle, C.c_void_p(_lib.ptr(arr) if n else 0), n, d,
                               C.c_void_p(counts.ctypes.data)))
    return FrequencyTable(d, counts)


def build_codebook(freq: FrequencyTable) -> HuffmanCodebook:
    """huffman.py:160-185 (host; microseconds for 4096 entries)."""
    counts = np.ascontiguousarray(freq.counts, dtype=np.int64)
    lens = np.zeros(freq.dict_size, np.uint8)
    codes = np.zeros(freq.dict_size, np.uint32)
    check(lib().hpdr_build_codebook(C.c_void_p(counts.ctypes.data), freq.dict_size, C.c_void_p(lens.ctypes.data),
                                    C.c_void_p(codes.ctypes.data)))
    return HuffmanCodebook(freq.dict_size, lens, codes)


def huffman_compress(keys, dict_size: int, adapter=None, *, device=None) -> bytes:
    arr = _keys(keys)
    d = _dict(dict_size)
    n = arr.numel() if hasattr(arr, "numel") else arr.size
    ctx = _lib.default_context(device)
    ln = C.c_uint64()
    check(lib().hpdr_huffman_compress(ctx.handle, C.c_void_p(_lib.ptr(arr) if n else 0), n, d, C.byref(ln)))
    b, p = _lib.new_bytes(ln.value)
    check(lib().hpdr_huffman_fetch(ctx.handle, C.c_void_p(p), ln.value))
    return b


def huffman_decompress(data, adapter=None, *, device=None) -> np.ndarray:
    buf = np.frombuffer(memoryview(data), dtype=np.uint8)
    ctx = _lib.default_context(device)
    n = C.c_uint64()
    addr = C.c_void_p(buf.ctypes.data if buf.size else 0)
    n_hint = int.from_bytes(bytes(buf[2:10]), "little") if buf.size >= 10 else 0
    out = np.empty(max(1, min(n_hint, 8 * buf.size * 8 + 1)), np.uint32)
    rc = lib().hpdr_huffman_decompress(ctx.handle, addr, buf.size, C.c_void_p(out.ctypes.data), out.size,
                                       C.byref(n))
    if rc == _lib.BUFFER and n.value > out.size:
        out = np.empty(n.value, np.uint32)
        rc = lib().hpdr_huffman_decompress(ctx.handle, addr, buf.size, C.c_void_p(out.ctypes.data), out.size,
                                           C.byref(n))
    check(rc)
    return out[: n.value]


__all__ = ["BLOCK_SYMBOLS", "MAX_CODE_LEN", "MAX_DICT_SIZE", "FrequencyTable", "HuffmanCodebook", "histogram",
           "build_codebook", "huffman_compress", "huffman_decompress"]
