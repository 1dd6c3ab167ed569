"""Pipelined compress/decompress wall time (CUDA events) vs chunk size at 513^3 (queues: env)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_06322_b200 import pipeline as PL  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
a = S.smooth_noise((n, n, n), seed=0)
vr = (float(a.min()), float(a.max()))
h_in = torch.from_numpy(a).pin_memory()
out = torch.empty(a.nbytes + (64 << 20), dtype=torch.uint8).pin_memory().numpy()
y = torch.empty(a.shape, dtype=torch.float32).pin_memory().numpy()
plane = a[0].nbytes
res = []
for mb in (16, 32, 64, 128):
    cp = max(1, (mb << 20) // plane)
    m = PL.compress_pipelined(h_in, 1e-4, value_range=vr, out=out, chunk_planes=cp)
    blob = torch.from_numpy(out[:m].copy()).pin_memory().numpy()
    times = {}
    for name, fn in (("c", lambda: PL.compress_pipelined(h_in, 1e-4, value_range=vr, out=out, chunk_planes=cp)),
                     ("d", lambda: PL.decompress_pipelined(blob, out=y))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        e1.synchronize()
        times[name] = e0.elapsed_time(e1) / 5
    res.append(f"{mb:4d}MB c {times['c']:6.2f} ms ({a.nbytes / times['c'] / 1e6:5.1f} GB/s)  "
               f"d {times['d']:6.2f} ms ({a.nbytes / times['d'] / 1e6:5.1f} GB/s) cr {a.nbytes / m:.3f}")
print(f"queues={os.environ.get('HPDR_PIPE_QUEUES', '3')}")
print("\n".join(res))
