import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2503_06322_b200 as P
from paper_2503_06322_b200 import synthetic as S
a = S.smooth_noise((513,) * 3, seed=0)
d = torch.from_numpy(a).cuda()
blob = P.mgard_compress(d, 1e-4)
o = torch.empty(len(blob) + (1 << 20), dtype=torch.uint8, device="cuda")
for _ in range(4):
    P.mgard_compress(d, 1e-4, out=o)
