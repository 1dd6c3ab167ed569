"""Cost of filling a fresh pageable 857 MB buffer (a Python bytes result) on this host:
first-touch faults with and without MADV_HUGEPAGE, the library's parallel memcpy from pinned
memory, and cudaHostRegister of the fresh buffer.   python tools/fault_probe.py [MB]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_06322_b200 import _lib  # noqa: E402
from paper_2503_06322_b200._lib import lib  # noqa: E402

n = int(sys.argv[1]) << 20 if len(sys.argv) > 1 else 857 << 20
libc = C.CDLL(None)
libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
src = torch.empty(n, dtype=torch.uint8).pin_memory()
src.fill_(7)


def fresh(huge):
    b, p = _lib.new_bytes(n)
    if huge:
        a = (p + (2 << 20) - 1) & ~((2 << 20) - 1)
        e = (p + n) & ~((2 << 20) - 1)
        libc.madvise(a, e - a, 14)   # MADV_HUGEPAGE
    return b, p


for huge in (False, True):
    b, p = fresh(huge)
    t = time.perf_counter()
    C.memset(p, 0, n)
    t1 = time.perf_counter() - t
    del b
    b, p = fresh(huge)
    t = time.perf_counter()
    lib().hpdr_host_copy(C.c_void_p(p), C.c_void_p(src.data_ptr()), C.c_uint64(n))
    t2 = time.perf_counter() - t
    t = time.perf_counter()
    lib().hpdr_host_copy(C.c_void_p(p), C.c_void_p(src.data_ptr()), C.c_uint64(n))
    t3 = time.perf_counter() - t
    del b
    b, p = fresh(huge)
    t = time.perf_counter()
    lib().hpdr_host_register(C.c_void_p(p), C.c_uint64(n))
    t4 = time.perf_counter() - t
    t = time.perf_counter()
    lib().hpdr_host_unregister(C.c_void_p(p))
    t5 = time.perf_counter() - t
    del b
    print(f"huge={huge}: memset-fresh {n / t1 / 1e9:.1f} GB/s, pool-copy-fresh {n / t2 / 1e9:.1f} GB/s, "
          f"pool-copy-warm {n / t3 / 1e9:.1f} GB/s, register-fresh {t4 * 1e3:.1f} ms, unregister {t5 * 1e3:.1f} ms",
          flush=True)
