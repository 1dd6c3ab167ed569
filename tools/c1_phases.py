"""C1 (129^3 fp32 GRF, abs 1e-3) end-to-end calls with pinned host buffers: wall time per call and,
with HPDR_PHASES=1, the library's phase marks.   python tools/c1_phases.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_06322_b200 as P  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
a = S.grf((129, 129, 129), m=8, seed=0)
h = torch.from_numpy(a).pin_memory()
blob = torch.empty(a.nbytes * 2, dtype=torch.uint8).pin_memory()
out = torch.empty(a.shape, dtype=torch.float32).pin_memory()
for _ in range(3):
    m = P.mgard_compress(h, 1e-3, value_range=(0.0, 1.0), out=blob)
    P.mgard_decompress(blob[:m], out=out)
torch.cuda.synchronize()
d = h.cuda()
dblob = torch.empty(a.nbytes * 2, dtype=torch.uint8, device="cuda")
dout = torch.empty(a.shape, dtype=torch.float32, device="cuda")
md = P.mgard_compress(d, 1e-3, value_range=(0.0, 1.0), out=dblob)
for name, fn in (("compress", lambda: P.mgard_compress(h, 1e-3, value_range=(0.0, 1.0), out=blob)),
                 ("decompress", lambda: P.mgard_decompress(blob[:m], out=out)),
                 ("compress device in/out", lambda: P.mgard_compress(d, 1e-3, value_range=(0.0, 1.0), out=dblob)),
                 ("decompress device in/out", lambda: P.mgard_decompress(dblob[:md], out=dout))):
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    print(f"{name}: {(time.perf_counter() - t) / reps * 1e3:.3f} ms/call (wall)", flush=True)
