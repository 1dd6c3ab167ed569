"""ncu driver: one warm + one measured pipelined compress / decompress at 513^3 (64 MB chunks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_06322_b200 import pipeline as PL  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "decompress"
a = S.smooth_noise((513, 513, 513), seed=0)
vr = (float(a.min()), float(a.max()))
h = torch.from_numpy(a).pin_memory()
out = torch.empty(a.nbytes + (64 << 20), dtype=torch.uint8).pin_memory().numpy()
m = PL.compress_pipelined(h, 1e-4, value_range=vr, out=out)
blob = torch.from_numpy(out[:m].copy()).pin_memory().numpy()
y = torch.empty(a.shape, dtype=torch.float32).pin_memory().numpy()
for _ in range(2):
    if what == "decompress":
        PL.decompress_pipelined(blob, out=y)
    else:
        PL.compress_pipelined(h, 1e-4, value_range=vr, out=out)
torch.cuda.synchronize()
print("ok")
