"""ctypes binding of libhpdr_b200.so (include/hpdr_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device is
visible, every entry point raises ``DeviceError``.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import threading

import numpy as np

from .errors import AllocationError, CorruptStreamError, DeviceError, FormatError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libhpdr_b200.so")

OK, VALIDATION, CORRUPT, ALLOCATION, CUDA, INDEX, OVERFLOW, VALUE, BUFFER, FORMAT = range(10)

_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)

_SIGS = {
    "hpdr_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "hpdr_ctx_destroy": (None, [C.c_void_p]),
    "hpdr_ctx_alloc_events": (C.c_uint64, [C.c_void_p]),
    "hpdr_ctx_device": (C.c_int, [C.c_void_p]),
    "hpdr_ctx_trim": (None, [C.c_void_p]),
    "hpdr_ctx_set_range_hook": (None, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "hpdr_last_error": (C.c_char_p, [_i64p]),
    "hpdr_host_alloc": (C.c_void_p, [C.c_uint64]),
    "hpdr_host_copy": (None, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "hpdr_host_free": (None, [C.c_void_p]),
    "hpdr_host_prefault_begin": (C.c_void_p, [C.c_void_p, C.c_uint64]),
    "hpdr_host_prefault_wait": (None, [C.c_void_p]),
    "hpdr_host_register": (C.c_int, [C.c_void_p, C.c_uint64]),
    "hpdr_host_unregister": (None, [C.c_void_p]),
    "hpdr_mgard_compress": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, _u64p, C.c_double, C.c_uint32,
                                      C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_uint64, _u64p]),
    "hpdr_mgard_fetch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "hpdr_mgard_compress_alloc": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, _u64p, C.c_double, C.c_uint32,
                                            C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_void_p, _u64p]),
    "hpdr_mgard_peek": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_int), C.POINTER(C.c_int), _u64p]),
    "hpdr_mgard_decompress": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    "hpdr_decompose": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, _u64p, C.c_void_p, _dp, _dp]),
    "hpdr_recompose": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, _u64p, C.c_void_p]),
    "hpdr_quantize": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, _u64p, C.c_double, C.c_double, C.c_double,
                                C.c_uint32, C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                _u64p, C.c_void_p, _u64p, _dp, _dp, C.POINTER(C.c_uint32)]),
    "hpdr_dequantize": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, _u64p, C.c_uint32, C.c_double,
                                  C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p]),
    "hpdr_histogram": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p]),
    "hpdr_build_codebook": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]),
    "hpdr_huffman_compress": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, _u64p]),
    "hpdr_huffman_fetch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "hpdr_huffman_decompress": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, _u64p]),
    "hpdr_launch_count": (C.c_uint64, [C.c_int]),
    "hpdr_prof_enable": (None, [C.c_int]),
    "hpdr_prof_read": (C.c_int, [C.c_char_p, C.c_uint64]),
    "hpdr_ctx_stream": (C.c_void_p, [C.c_void_p]),
    "hpdr_selftest_div": (C.c_int, [C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "hpdr_minmax": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, _dp, _dp]),
    "hpdr_pipeline_compress": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, _u64p, C.c_double, C.c_uint32,
                                         C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_void_p, C.c_uint64,
                                         C.c_void_p, C.c_uint64, _u64p, C.c_void_p]),
    "hpdr_zfp_compressed_size": (C.c_int, [C.c_int, C.c_int, _u64p, C.c_uint32, _u64p]),
    "hpdr_zfp_compress": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, _u64p, C.c_uint32, C.c_void_p,
                                    C.c_uint64, _u64p]),
    "hpdr_zfp_peek": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_int), C.POINTER(C.c_int), _u64p,
                                C.POINTER(C.c_uint32)]),
    "hpdr_zfp_decompress": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    "hpdr_pipeline_zfp_compress": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, _u64p, C.c_uint32, C.c_uint64,
                                             C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, _u64p, C.c_void_p]),
    "hpdr_pipeline_decompress": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load the native library (raises DeviceError when it is absent)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(SO_PATH):
                    raise DeviceError(f"native library {SO_PATH} not built; run __graft_entry__.build()")
                L = C.CDLL(SO_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def check(rc: int):
    if rc == OK:
        return
    bit = C.c_int64(-1)
    msg = lib().hpdr_last_error(C.byref(bit)).decode("utf-8", "replace")
    if rc == VALIDATION:
        raise ValidationError(msg)
    if rc == CORRUPT:
        raise CorruptStreamError(msg, bit_offset=int(bit.value))
    if rc == ALLOCATION:
        raise AllocationError(msg)
    if rc == INDEX:
        raise IndexError(msg)
    if rc == OVERFLOW:
        raise OverflowError(msg)
    if rc == VALUE:
        raise ValueError(msg)
    if rc == BUFFER:
        raise ValueError(msg)
    if rc == FORMAT:
        raise FormatError(msg)
    raise DeviceError(msg)


def dims_arg(dims):
    return (C.c_uint64 * max(1, len(dims)))(*[int(d) for d in dims])


def ptr(a) -> int:
    """Address of a numpy array, bytes-like object or torch tensor."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return int(a.data_ptr())
    if isinstance(a, (bytes, bytearray, memoryview)):
        return np.frombuffer(a, dtype=np.uint8).ctypes.data if len(a) else 0
    raise TypeError(f"unsupported buffer type {type(a)}")


class DeviceContext:
    """One hpdr_ctx: persistent device buffers, streams and operator tables on one GPU."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().hpdr_ctx_create(int(device), C.byref(h)))
        self._h = h
        self.device = int(device)

    @property
    def handle(self):
        if self._h is None:
            raise DeviceError("context closed")
        return self._h

    @property
    def alloc_events(self) -> int:
        return int(lib().hpdr_ctx_alloc_events(self.handle))

    def trim(self):
        lib().hpdr_ctx_trim(self.handle)

    @property
    def stream(self) -> int:
        """cudaStream_t of the context's compute stream (for external event timing)."""
        return int(lib().hpdr_ctx_stream(self.handle) or 0)

    def close(self):
        if self._h is not None and _lib is not None:
            _lib.hpdr_ctx_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def default_device(obj=None) -> int:
    """The GPU a call runs on: a CUDA tensor argument's own device, else HPDR_DEVICE, else torch's
    current device (torch.cuda.set_device, one process per GPU), else LOCAL_RANK, else 0."""
    dev = getattr(obj, "device", None)
    if getattr(dev, "type", None) == "cuda" and dev.index is not None:
        return int(dev.index)
    env = os.environ.get("HPDR_DEVICE")
    if env:
        return int(env)
    t = sys.modules.get("torch")
    if t is not None:
        try:
            if t.cuda.is_initialized():
                return int(t.cuda.current_device())
        except Exception:   # noqa: BLE001 - torch without CUDA
            pass
    lr = os.environ.get("LOCAL_RANK")
    return int(lr) if lr else 0


def default_context(device: int | None = None, obj=None) -> DeviceContext:
    """Per-thread, per-device persistent context (a context is never shared across threads).
    device None: default_device(obj) (obj: the call's tensor argument, if any)."""
    device = default_device(obj) if device is None else int(device)
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    c = ctxs.get(device)
    if c is None:
        c = ctxs[device] = DeviceContext(device)
    return c


_pybytes_new = C.pythonapi.PyBytes_FromStringAndSize
_pybytes_new.restype = C.py_object
_pybytes_new.argtypes = [C.c_void_p, C.c_ssize_t]
_pybytes_ptr = C.pythonapi.PyBytes_AsString
_pybytes_ptr.restype = C.c_void_p
_pybytes_ptr.argtypes = [C.py_object]


_scratch = threading.local()


def pinned_scratch(nbytes: int) -> np.ndarray:
    """A per-thread, grow-only pinned host buffer (uint8) of at least nbytes, owned by the library
    (for results whose size is only known after the call, e.g. a pipeline container)."""
    cur = getattr(_scratch, "buf", None)
    if cur is None or cur[1] < nbytes:
        if cur is not None:
            lib().hpdr_host_free(C.c_void_p(cur[0]))
        p = lib().hpdr_host_alloc(int(nbytes))
        if not p:
            raise AllocationError(f"cudaHostAlloc of {nbytes} bytes failed")
        cur = (p, int(nbytes))
        _scratch.buf = cur
    return np.ctypeslib.as_array((C.c_uint8 * cur[1]).from_address(cur[0]))


def bytes_from(buf: np.ndarray, n: int) -> bytes:
    """bytes(buf[:n]) with the copy split across the library's threads."""
    b, p = new_bytes(n)
    if n:
        lib().hpdr_host_copy(C.c_void_p(p), C.c_void_p(buf.ctypes.data), int(n))
    return b


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_uint64)   # hpdr_alloc_fn


_pybytes_resize = C.pythonapi._PyBytes_Resize
_pybytes_resize.argtypes = [C.POINTER(C.py_object), C.c_ssize_t]
_pybytes_resize.restype = C.c_int


class BytesSink:
    """hpdr_alloc_fn that hands the library the result ``bytes`` once the blob size is known.

    With ``hint`` (the size of a previous blob of the same shape) a slightly larger bytes object is
    created up front and first-touched on background threads while the GPU works (a fresh
    destination otherwise pays its page faults inside the staged copy); ``take`` then trims it to
    the exact size in place (``_PyBytes_Resize``: a shrinking realloc, no copy)."""

    MIN_HINT = 64 << 20

    def __init__(self, hint: int = 0):
        self.obj = None
        self.n = 0
        self.fn = ALLOC_FN(self._alloc)
        self._pre = None   # (bytes, address, capacity, prefault handle)
        if hint >= self.MIN_HINT:
            cap = int(hint * 1.02) + (1 << 20)
            try:
                b, p = new_bytes(cap)
            except MemoryError:
                return
            self._pre = (b, p, cap, lib().hpdr_host_prefault_begin(C.c_void_p(p), cap))

    def _join(self):
        if self._pre is not None and self._pre[3]:
            lib().hpdr_host_prefault_wait(C.c_void_p(self._pre[3]))
            self._pre = self._pre[:3] + (None,)

    def _alloc(self, _user, n):
        self.n = int(n)
        try:
            self._join()
            if self._pre is not None and n <= self._pre[2]:
                self.obj, p = self._pre[0], self._pre[1]
                self._pre = None
                return p
            self._pre = None
            self.obj, p = new_bytes(n)
            return p
        except MemoryError:
            return None

    def take(self):
        """The result: exactly ``n`` bytes."""
        self._join()
        self._pre = None
        obj, self.obj = self.obj, None
        if obj is None or len(obj) == self.n:
            return obj
        box = C.py_object(obj)
        del obj
        # the box must hold the only reference (getrefcount adds the temporary of box.value)
        if sys.getrefcount(box.value) == 2 and _pybytes_resize(C.byref(box), self.n) == 0:
            return box.value
        return bytes(memoryview(box.value)[: self.n])


def new_bytes(n: int):
    """A fresh, writable-until-returned bytes object of length n and its address."""
    b = _pybytes_new(None, int(n))
    return b, _pybytes_ptr(b)


def launch_count(reset: bool = False) -> int:
    return int(lib().hpdr_launch_count(1 if reset else 0))


def prof_enable(on=True):
    """on: False / True (live events) / "serial" (device synchronized around every launch)."""
    lib().hpdr_prof_enable(2 if on == "serial" else (1 if on else 0))


def prof_read() -> dict:
    """{kernel: (launches, total_ms, total_algorithmic_bytes, max_ms)} since prof_enable."""
    import json

    buf = C.create_string_buffer(1 << 16)
    check(lib().hpdr_prof_read(buf, len(buf)))
    return {k: tuple(v) for k, v in json.loads(buf.value.decode()).items()}


def minmax(ctx: "DeviceContext", addr: int, dtype_code: int, n: int):
    lo, hi = C.c_double(), C.c_double()
    check(lib().hpdr_minmax(ctx.handle, C.c_void_p(addr), int(dtype_code), int(n), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value
