"""Host codebook build time (hpdr_build_codebook) on a C1-like key histogram.
    python tools/codebook_probe.py"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2503_06322_b200._lib import lib  # noqa: E402

rng = np.random.default_rng(0)
k = np.rint(rng.normal(0, 200, 2_000_000)).astype(np.int64)
z = np.where(k >= 0, 2 * k, -2 * k - 1)
counts = np.bincount(z[z < 4096], minlength=4096).astype(np.int64)
lens = np.zeros(4096, np.uint8)
codes = np.zeros(4096, np.uint32)
f = lib().hpdr_build_codebook
args = (counts.ctypes.data_as(C.c_void_p), C.c_uint32(4096), lens.ctypes.data_as(C.c_void_p),
        codes.ctypes.data_as(C.c_void_p))
for _ in range(10):
    f(*args)
t = time.perf_counter()
for _ in range(1000):
    f(*args)
print(f"present {int((counts > 0).sum())}: {(time.perf_counter() - t) * 1e3:.1f} us per build (1000 reps)")
