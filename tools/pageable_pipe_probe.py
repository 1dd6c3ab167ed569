"""Streams pipeline with pageable numpy in/out (513^3 fp32 rel 1e-4)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_06322_b200 import pipeline as PL  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

a = S.smooth_noise((513,) * 3, seed=0)
for vr in (None, (float(a.min()), float(a.max()))):
    c = PL.compress_pipelined(a, 1e-4, value_range=vr)
    t = time.perf_counter()
    for _ in range(3):
        c = PL.compress_pipelined(a, 1e-4, value_range=vr)
    dt = (time.perf_counter() - t) / 3
    y = PL.decompress_pipelined(c)
    t = time.perf_counter()
    for _ in range(3):
        y = PL.decompress_pipelined(c)
    dd = (time.perf_counter() - t) / 3
    print(f"{'rel' if vr is None else 'abs'}: compress {a.nbytes / dt / 1e9:.1f} GB/s, decompress {a.nbytes / dd / 1e9:.1f} GB/s")
