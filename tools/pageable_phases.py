"""Drop-in numpy -> bytes compress at the 1024^3 Target: wall time of the call and of freeing the
previous result, with HPDR_PHASES=1 marks.   HPDR_PHASES=1 python tools/pageable_phases.py [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2503_06322_b200 as P  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
a = S.smooth_noise((n, n, n), seed=0)
vr = (float(a.min()), float(a.max()))
b = P.mgard_compress(a, 1e-4, value_range=vr)
b = P.mgard_compress(a, 1e-4, value_range=vr)
for _ in range(3):
    t0 = time.perf_counter()
    del b
    t1 = time.perf_counter()
    b = P.mgard_compress(a, 1e-4, value_range=vr)
    t2 = time.perf_counter()
    print(f"free previous {1e3 * (t1 - t0):.1f} ms, compress -> bytes {1e3 * (t2 - t1):.1f} ms", flush=True)
