"""M1 phase timeline (HPDR_PHASES=1 marks, ms since the first mark) for the bench Target's
end-to-end calls: pinned host field -> blob in pinned memory, and back.
    HPDR_PHASES=1 python tools/m1_phases.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_06322_b200 as P  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
a = S.smooth_noise((n, n, n), seed=0)
h = torch.from_numpy(a).pin_memory()
blob = torch.empty(int(a.nbytes * 1.3) + (16 << 20), dtype=torch.uint8).pin_memory()
out = torch.empty(a.shape, dtype=torch.float32).pin_memory()
for _ in range(3):
    m = P.mgard_compress(h, 1e-4, out=blob)
    P.mgard_decompress(blob[:m], out=out)
torch.cuda.synchronize()
print("blob", m, flush=True)
