"""M2 compress/decompress time for a few chunk schedules (513^3 fp32, abs bound, pinned buffers)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_06322_b200 import pipeline as PL  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

a = S.smooth_noise((513,) * 3, seed=0)
vr = (float(a.min()), float(a.max()))
h = torch.from_numpy(a).pin_memory()
out = torch.empty(a.nbytes + (64 << 20), dtype=torch.uint8).pin_memory().numpy()
y = torch.empty(a.shape, dtype=torch.float32).pin_memory().numpy()
scheds = {
    "fixed57": [57] * 9,
    "taper1": [57] * 7 + [40, 30, 20, 14, 10],
    "taper2": [29, 57, 57, 57, 57, 57, 57, 57, 29, 29, 15, 12],
    "taper3": [20, 40] + [57] * 6 + [40, 30, 20, 15, 6],
    "fixed43": [43] * 11 + [40],
}
for name, sc in scheds.items():
    assert sum(sc) == 513, name
    res = {}
    for mode in ("c", "d"):
        if mode == "c":
            fn = lambda: PL.compress_pipelined(h, 1e-4, value_range=vr, chunks=sc, out=out)  # noqa: E731
        else:
            m = PL.compress_pipelined(h, 1e-4, value_range=vr, chunks=sc, out=out)
            blob = torch.from_numpy(out[:m].copy()).pin_memory().numpy()
            fn = lambda: PL.decompress_pipelined(blob, out=y)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        e1.synchronize()
        res[mode] = e0.elapsed_time(e1) / 5
    print(f"{name:8s} c {res['c']:6.2f} ms ({a.nbytes / res['c'] / 1e6:5.1f} GB/s)  d {res['d']:6.2f} ms ({a.nbytes / res['d'] / 1e6:5.1f} GB/s)")
