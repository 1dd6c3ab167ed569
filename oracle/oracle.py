"""ctypes wrapper of the CPU parity oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.  It restates the reference hpdr MGARD path
(/root/reference/pkg/src/hpdr/mgard/codec.py:25-113) in C; see mgard_oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")

OK, VALIDATION, CORRUPT, ALLOC, INDEX, OVERFLOW = 0, 1, 2, 3, 5, 6


class OracleError(Exception):
    def __init__(self, code, bit_offset=-1):
        super().__init__(f"oracle error code {code} (bit_offset {bit_offset})")
        self.code = code
        self.bit_offset = bit_offset


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        _lib = C.CDLL(_LIB)
        _lib.orc_huffman_bound.restype = C.c_uint64
    return _lib


def set_threads(n: int):
    lib().orc_set_threads(int(n))


def _dims(dims):
    arr = (C.c_uint64 * len(dims))(*[int(d) for d in dims])
    return arr


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _chk(rc, bit=-1):
    if rc:
        raise OracleError(rc, bit)


def hierarchy(dims):
    L = C.c_int()
    counts = np.zeros(len(dims) * 64, dtype=np.uint64)
    _chk(lib().orc_hierarchy(len(dims), _dims(dims), C.byref(L), _p(counts)))
    return L.value, counts[: len(dims) * L.value].reshape(len(dims), L.value)


def decompose(arr: np.ndarray):
    arr = np.ascontiguousarray(arr)
    dt = {np.dtype("<f4"): 0, np.dtype("<f8"): 1}[arr.dtype]
    coef = np.empty(arr.shape, dtype=np.float64)
    vmin, vmax = C.c_double(), C.c_double()
    _chk(lib().orc_decompose(_p(arr), dt, arr.ndim, _dims(arr.shape), _p(coef), C.byref(vmin), C.byref(vmax)))
    return coef, vmin.value, vmax.value


def recompose(coef: np.ndarray):
    coef = np.ascontiguousarray(coef, dtype=np.float64)
    out = np.empty_like(coef)
    _chk(lib().orc_recompose(_p(coef), coef.ndim, _dims(coef.shape), _p(out)))
    return out


def coarsest_indices(dims):
    n = C.c_uint64()
    out = np.zeros(int(np.prod(dims)), dtype=np.uint64)
    _chk(lib().orc_coarsest_indices(len(dims), _dims(dims), _p(out), C.byref(n)))
    return out[: n.value]


def quantize(coef, u_min, u_max, eb_rel, dict_size=4096, value_range=None):
    coef = np.ascontiguousarray(coef, dtype=np.float64)
    N = coef.size
    keys = np.empty(N, np.uint32)
    oidx = np.empty(N, np.uint64)
    obins = np.empty(N, np.int64)
    cv = np.empty(max(1, N), np.float64)
    no, nco = C.c_uint64(), C.c_uint64()
    eb_abs, binw = C.c_double(), C.c_double()
    L = C.c_int()
    has = value_range is not None
    r0, r1 = (float(value_range[0]), float(value_range[1])) if has else (0.0, 0.0)
    _chk(lib().orc_quantize(_p(coef), coef.ndim, _dims(coef.shape), C.c_double(u_min), C.c_double(u_max),
                            C.c_double(eb_rel), C.c_uint32(dict_size), int(has), C.c_double(r0), C.c_double(r1),
                            _p(keys), _p(oidx), _p(obins), C.byref(no), _p(cv), C.byref(nco),
                            C.byref(eb_abs), C.byref(binw), C.byref(L)))
    return dict(keys=keys, outlier_idx=oidx[: no.value].copy(), outlier_bins=obins[: no.value].copy(),
                coarse_values=cv[: nco.value].copy(), eb_abs=eb_abs.value, bin_width=binw.value,
                total_levels=L.value)


def build_codebook(counts, dict_size):
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    lens = np.zeros(dict_size, np.uint8)
    codes = np.zeros(dict_size, np.uint32)
    _chk(lib().orc_build_codebook(_p(counts), C.c_uint32(dict_size), _p(lens), _p(codes)))
    return lens, codes


def huffman_compress(keys, dict_size):
    keys = np.ascontiguousarray(keys, dtype=np.uint32).reshape(-1)
    cap = lib().orc_huffman_bound(C.c_uint64(keys.size), C.c_uint32(dict_size))
    out = np.empty(cap, np.uint8)
    ln = C.c_uint64()
    _chk(lib().orc_huffman_compress(_p(keys), C.c_uint64(keys.size), C.c_uint32(dict_size), _p(out),
                                    C.c_uint64(cap), C.byref(ln)))
    return out[: ln.value].tobytes()


def huffman_decompress(data: bytes):
    buf = np.frombuffer(data, dtype=np.uint8)
    n = int.from_bytes(data[2:10], "little") if len(data) >= 10 else 0
    keys = np.empty(max(1, n), np.uint32)
    nout, bit = C.c_uint64(), C.c_int64()
    rc = lib().orc_huffman_decompress(_p(buf), C.c_uint64(len(data)), _p(keys), C.c_uint64(n),
                                      C.byref(nout), C.byref(bit))
    _chk(rc, bit.value)
    return keys[: nout.value].copy()


def mgard_compress(arr: np.ndarray, eb_rel: float, dict_size: int = 4096, value_range=None) -> bytes:
    arr = np.ascontiguousarray(arr)
    dt = {np.dtype("<f4"): 0, np.dtype("<f8"): 1}[arr.dtype]
    blob = C.POINTER(C.c_uint8)()
    ln = C.c_uint64()
    has = value_range is not None
    r0, r1 = (float(value_range[0]), float(value_range[1])) if has else (0.0, 0.0)
    _chk(lib().orc_mgard_compress(_p(arr), dt, arr.ndim, _dims(arr.shape), C.c_double(eb_rel),
                                  C.c_uint32(dict_size), int(has), C.c_double(r0), C.c_double(r1),
                                  C.byref(blob), C.byref(ln)))
    try:
        return C.string_at(blob, ln.value)
    finally:
        lib().orc_free(blob)


def mgard_decompress(data: bytes) -> np.ndarray:
    buf = np.frombuffer(data, dtype=np.uint8)
    rank = data[0]
    dims = [int.from_bytes(data[1 + 8 * i: 9 + 8 * i], "little") for i in range(min(rank, 4))]
    dtype = data[1 + 8 * rank] if len(data) > 1 + 8 * rank else 0
    npdt = np.float32 if dtype == 0 else np.float64
    out = np.empty(int(np.prod(dims)) if dims else 1, dtype=npdt)
    dto, rko, bit = C.c_int(), C.c_int(), C.c_int64()
    dout = (C.c_uint64 * 4)()
    rc = lib().orc_mgard_decompress(_p(buf), C.c_uint64(len(data)), _p(out), C.c_uint64(out.nbytes),
                                    C.byref(dto), C.byref(rko), dout, C.byref(bit))
    _chk(rc, bit.value)
    return out.reshape(dims)


# ---- fixed-rate block coder (zfp_oracle.c restates hpdr/zfp.py) ----

def zfp_compressed_size(dims, dtype_code: int, rate: int) -> int:
    size = C.c_uint64()
    _chk(lib().orz_compressed_size(int(dtype_code), len(dims), _dims(dims), int(rate), C.byref(size)))
    return size.value


def zfp_compress(arr: np.ndarray, rate: int) -> bytes:
    arr = np.ascontiguousarray(arr)
    dt = {np.dtype("<f4"): 0, np.dtype("<f8"): 1}[arr.dtype]
    size = zfp_compressed_size(arr.shape, dt, rate)
    out = np.empty(size, np.uint8)
    ln = C.c_uint64()
    _chk(lib().orz_compress(_p(arr), dt, arr.ndim, _dims(arr.shape), int(rate), _p(out), C.c_uint64(size),
                            C.byref(ln)))
    return out.tobytes()


def zfp_decompress(data: bytes) -> np.ndarray:
    buf = np.frombuffer(data, dtype=np.uint8)
    dt, rk, rate = C.c_int(), C.c_int(), C.c_int()
    dims = (C.c_uint64 * 3)()
    _chk(lib().orz_peek(_p(buf), C.c_uint64(buf.size), C.byref(dt), C.byref(rk), dims, C.byref(rate)))
    shape = [int(dims[i]) for i in range(rk.value)]
    out = np.empty(shape, np.float32 if dt.value == 0 else np.float64)
    _chk(lib().orz_decompress(_p(buf), C.c_uint64(buf.size), _p(out), C.c_uint64(out.nbytes)))
    return out
