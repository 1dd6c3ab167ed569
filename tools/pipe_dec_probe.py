import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2503_06322_b200 import pipeline as PL
from paper_2503_06322_b200 import synthetic as S
a = S.smooth_noise((513,) * 3, seed=0)
vr = (float(a.min()), float(a.max()))
h_in = torch.from_numpy(a).pin_memory()
out = torch.empty(a.nbytes + (64 << 20), dtype=torch.uint8).pin_memory().numpy()
m = PL.compress_pipelined(h_in, 1e-4, value_range=vr, out=out)
blob = torch.from_numpy(out[:m].copy()).pin_memory().numpy()
yd = torch.empty(a.shape, dtype=torch.float32, device="cuda")
yh = torch.empty(a.shape, dtype=torch.float32).pin_memory().numpy()
for name, y in (("device out", yd), ("host out", yh)):
    for _ in range(3):
        PL.decompress_pipelined(blob, out=y)
    _, tr = PL.decompress_pipelined(blob, out=y, trace=True)
    print(name, "total %.2f" % tr.max(), "compute per chunk", " ".join("%.2f" % (r[3] - r[2]) for r in tr))
