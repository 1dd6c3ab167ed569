"""ncu driver: device-resident compress (bench kernel-only leg) and decompress into device memory.
Launch order per call is fixed, so ncu -s/-c select the finest-level launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_06322_b200 as P  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
a = S.smooth_noise((n, n, n), seed=0)
d = torch.from_numpy(a).cuda()
out = torch.empty(a.shape, dtype=torch.float32, device="cuda")
blob = P.mgard_compress(d, 1e-4)
pin = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).pin_memory().numpy()
for _ in range(2):
    P.mgard_compress(d, 1e-4)
    P.mgard_decompress(pin, out=out)
torch.cuda.synchronize()
print("ok", len(blob))
