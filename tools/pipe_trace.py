"""Print the streams-pipeline trace (per chunk: H2D, compute, D2H start/end in ms) at a size.

    python tools/pipe_trace.py [n] [chunk_planes]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_06322_b200 import pipeline as PL  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
cp = int(sys.argv[2]) if len(sys.argv) > 2 else 0
a = S.smooth_noise((n, n, n), seed=0)
vr = None if (len(sys.argv) > 3 and sys.argv[3] == "rel") else (float(a.min()), float(a.max()))
h_in = torch.from_numpy(a).pin_memory()
out = torch.empty(a.nbytes + (64 << 20), dtype=torch.uint8).pin_memory().numpy()
m = PL.compress_pipelined(h_in, 1e-4, value_range=vr, out=out, chunk_planes=cp)
blob = torch.from_numpy(out[:m].copy()).pin_memory().numpy()
y = torch.empty(a.shape, dtype=torch.float32).pin_memory().numpy()
for _ in range(3):
    PL.compress_pipelined(h_in, 1e-4, value_range=vr, out=out, chunk_planes=cp)
    PL.decompress_pipelined(blob, out=y)
for name, fn in (("compress", lambda: PL.compress_pipelined(h_in, 1e-4, value_range=vr, out=out, chunk_planes=cp,
                                                            trace=True)[1]),
                 ("decompress", lambda: PL.decompress_pipelined(blob, out=y, trace=True)[1])):
    tr = fn()
    print(f"== {name}: total {tr.max():.2f} ms, overlap {PL.overlap_ratio(tr):.3f}")
    print("  k   h2d_s   h2d_e   cmp_s   cmp_e   d2h_s   d2h_e")
    for k, r in enumerate(tr):
        print(f"{k:3d} " + " ".join(f"{v:7.2f}" for v in r))

# per-kernel device time inside one pipelined call (library's live CUDA-event profiler)
from paper_2503_06322_b200 import _lib  # noqa: E402
import time  # noqa: E402

for name, fn in (("compress", lambda: PL.compress_pipelined(h_in, 1e-4, value_range=vr, out=out, chunk_planes=cp)),
                 ("decompress", lambda: PL.decompress_pipelined(blob, out=y))):
    torch.cuda.synchronize()
    _lib.prof_enable(True)
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) * 1e3
    k = _lib.prof_read()
    _lib.prof_enable(False)
    tot = sum(v[1] for v in k.values())
    print(f"== {name} kernels: wall {wall:.2f} ms, kernel sum {tot:.2f} ms")
    for kk, v in sorted(k.items(), key=lambda kv: -kv[1][1])[:12]:
        print(f"   {kk:24s} n={v[0]:5.0f} {v[1]:8.3f} ms")
