"""Debug driver: streams-pipeline compress at a given size / chunking (env-free)."""
import sys, os, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2503_06322_b200 as P
from paper_2503_06322_b200 import pipeline as PL
from paper_2503_06322_b200 import synthetic as S

n = int(sys.argv[1]); planes = int(sys.argv[2]); mode = sys.argv[3]
a = S.smooth_noise((n, n, n), seed=0)
vr = (float(a.min()), float(a.max()))
if mode == "direct":
    for p0 in (planes, n % planes or planes):
        d = torch.from_numpy(np.ascontiguousarray(a[:p0])).cuda()
        b = P.mgard_compress(d, 1e-4, value_range=vr)
        print("direct", p0, len(b), flush=True)
    sys.exit(0)
if mode == "pinned":
    src = torch.from_numpy(a).pin_memory()
elif mode == "m1first":
    d = torch.from_numpy(a).cuda()
    P.mgard_compress(d, 1e-4)
    src = torch.from_numpy(a).pin_memory()
else:
    src = a
out = torch.empty(a.nbytes + (64 << 20), dtype=torch.uint8).pin_memory().numpy()
m = PL.compress_pipelined(src, 1e-4, value_range=vr, chunk_planes=planes, out=out)
print(mode, n, planes, "ok", m, flush=True)
y = PL.decompress_pipelined(out[:m].copy())
print("err/eb", float(np.max(np.abs(y.astype(np.float64) - a))) / (1e-4 * (vr[1] - vr[0])))
