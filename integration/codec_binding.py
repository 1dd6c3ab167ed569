"""The reference-side binding of INTEGRATION.md §2, as an installable module.

A maintainer of the reference would paste these two functions into ``hpdr/mgard/codec.py``
(codec.py:25 ``mgard_compress``, :59 ``mgard_decompress``).  ``install(codec)`` does exactly that
at run time: it defines them against the given codec module's own names (TensorData, DType,
DTYPE_CODES, DTYPE_FROM_CODE and the hpdr error classes) and rebinds ``codec.mgard_compress`` /
``codec.mgard_decompress`` and the ``hpdr.mgard`` package re-exports, so the reference's public
API runs on the B200 library through its C ABI (include/hpdr_b200.h) and nothing else.

tests/test_reference_binding.py installs it into the unmodified reference (baseline/_ref) and
checks the reference's own calls against the golden blobs the reference produced.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2503_06322_b200",
                    "libhpdr_b200.so")


def install(codec, lib_path: str = _LIB, device: int = 0):
    """Rebind codec.mgard_compress / codec.mgard_decompress (and hpdr.mgard's re-exports) to
    the B200 library.  Returns the previous functions so a caller can restore them."""
    errors = sys.modules[codec.__name__.rsplit(".", 2)[0] + ".errors"]
    TensorData, DType = codec.TensorData, codec.DType
    DTYPE_CODES, DTYPE_FROM_CODE = codec.DTYPE_CODES, codec.DTYPE_FROM_CODE

    L = C.CDLL(lib_path)
    L.hpdr_last_error.restype = C.c_char_p
    L.hpdr_last_error.argtypes = [C.POINTER(C.c_int64)]
    ALLOC = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_uint64)   # hpdr_alloc_fn
    L.hpdr_mgard_compress_alloc.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_uint64),
                                            C.c_double, C.c_uint32, C.c_int, C.c_double, C.c_double, ALLOC,
                                            C.c_void_p, C.POINTER(C.c_uint64)]
    pybytes_new = C.pythonapi.PyBytes_FromStringAndSize
    pybytes_new.restype, pybytes_new.argtypes = C.py_object, [C.c_void_p, C.c_ssize_t]
    pybytes_ptr = C.pythonapi.PyBytes_AsString
    pybytes_ptr.restype, pybytes_ptr.argtypes = C.c_void_p, [C.py_object]
    ctx = C.c_void_p()
    if L.hpdr_ctx_create(int(device), C.byref(ctx)) != 0:
        raise RuntimeError("hpdr_ctx_create failed: " + L.hpdr_last_error(None).decode())

    def _raise(rc):
        bit = C.c_int64(-1)
        msg = L.hpdr_last_error(C.byref(bit)).decode()
        if rc == 2:
            raise errors.CorruptStreamError(msg, bit.value)
        raise {1: errors.ValidationError, 3: errors.AllocationError, 5: IndexError, 6: OverflowError,
               7: ValueError}.get(rc, RuntimeError)(msg)

    def mgard_compress(u, eb_rel, dict_size=4096, adapter=None, cache=None, value_range=None):
        if u.dtype not in (DType.F32, DType.F64):
            raise errors.ValidationError(f"lossy compression needs F32/F64, got {u.dtype}")
        arr = np.ascontiguousarray(u.values)
        dims = (C.c_uint64 * len(u.dims))(*u.dims)
        n = C.c_uint64()
        has = value_range is not None
        lo, hi = value_range if has else (0.0, 0.0)
        # the result bytes object is created by the library's allocator callback once the blob size is
        # known, and the blob streams into it behind the payload encode (no second copy)
        res = {}

        def alloc(_user, size):
            res["b"] = pybytes_new(None, size)
            return pybytes_ptr(res["b"])

        cb = ALLOC(alloc)
        rc = L.hpdr_mgard_compress_alloc(ctx, C.c_void_p(arr.ctypes.data), DTYPE_CODES[u.dtype], len(u.dims),
                                         dims, C.c_double(eb_rel), C.c_uint32(dict_size), int(has), C.c_double(lo),
                                         C.c_double(hi), cb, None, C.byref(n))
        if rc:
            _raise(rc)
        return res["b"]

    def mgard_decompress(data, adapter=None, cache=None):
        buf = np.frombuffer(memoryview(data), np.uint8)
        addr = C.c_void_p(buf.ctypes.data if buf.size else 0)
        dt, rk, dims = C.c_int(), C.c_int(), (C.c_uint64 * 4)()
        rc = L.hpdr_mgard_peek(addr, C.c_uint64(buf.size), C.byref(dt), C.byref(rk), dims)
        if rc:
            _raise(rc)
        # an unknown dtype code or rank is reported by the decoder with the reference's exception
        dtype = DTYPE_FROM_CODE.get(dt.value, DType.F64)
        shape = tuple(int(dims[i]) for i in range(rk.value)) if 1 <= rk.value <= 4 else (1,)
        out = np.empty(shape, dtype.np_dtype)
        rc = L.hpdr_mgard_decompress(ctx, addr, C.c_uint64(buf.size), C.c_void_p(out.ctypes.data),
                                     C.c_uint64(out.nbytes))
        if rc:
            _raise(rc)
        return TensorData(shape, dtype, out)

    prev = (codec.mgard_compress, codec.mgard_decompress)
    pkg = sys.modules[codec.__name__.rsplit(".", 1)[0]]
    for mod in (codec, pkg):
        mod.mgard_compress, mod.mgard_decompress = mgard_compress, mgard_decompress
    return prev
