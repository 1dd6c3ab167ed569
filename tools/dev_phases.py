"""Phase timeline (HPDR_PHASES=1) of the kernel-only compress: device input, device output."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_06322_b200 as P  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
a = S.smooth_noise((n, n, n), seed=0)
d = torch.from_numpy(a).cuda()
o = torch.empty(a.nbytes, dtype=torch.uint8, device="cuda")
for _ in range(4):
    P.mgard_compress(d, 1e-4, out=o)
torch.cuda.synchronize()
print("ok")
