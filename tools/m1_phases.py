"""Phase timeline (HPDR_PHASES=1) of the whole-field M1 compress / decompress with pinned host buffers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_06322_b200 as P  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
a = S.smooth_noise((n, n, n), seed=0)
vr = (float(a.min()), float(a.max())) if (len(sys.argv) > 2 and sys.argv[2] == "abs") else None
h_in = torch.from_numpy(a).pin_memory()
blob = P.mgard_compress(h_in, 1e-4, value_range=vr)
h_blob = torch.empty(len(blob) + (1 << 20), dtype=torch.uint8).pin_memory()
pin = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).pin_memory().numpy()
h_out = torch.empty(a.shape, dtype=torch.float32).pin_memory()
for _ in range(3):
    P.mgard_compress(h_in, 1e-4, value_range=vr, out=h_blob)
    P.mgard_decompress(pin, out=h_out)
print("ok", len(blob))
