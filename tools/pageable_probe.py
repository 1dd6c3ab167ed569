"""Drop-in API with plain numpy / bytes (pageable host memory), C2 513^3 fp32 rel 1e-4:
mgard_compress(ndarray) -> bytes and mgard_decompress(bytes) -> TensorData, wall time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2503_06322_b200 as P  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402
from paper_2503_06322_b200 import zfp as Z  # noqa: E402

a = S.smooth_noise((513,) * 3, seed=0)
for name, fn in (("mgard_compress(ndarray)->bytes", lambda: P.mgard_compress(a, 1e-4)),
                 ("zfp_compress(ndarray)->bytes", lambda: Z.zfp_compress(a, 16))):
    b = fn()
    t = time.perf_counter()
    for _ in range(3):
        b = fn()
    dt = (time.perf_counter() - t) / 3
    print(f"{name}: {dt * 1e3:.1f} ms, {a.nbytes / dt / 1e9:.1f} GB/s")
    dec = (lambda: P.mgard_decompress(b)) if name.startswith("mgard") else (lambda: Z.zfp_decompress(b))
    dec()
    t = time.perf_counter()
    for _ in range(3):
        y = dec()
    dt = (time.perf_counter() - t) / 3
    print(f"  decompress(bytes)->array: {dt * 1e3:.1f} ms, {a.nbytes / dt / 1e9:.1f} GB/s")
