"""Fixed vs adaptive (Algorithm 4) chunking of the streams pipeline, end to end (pinned host).

    python tools/adaptive_sweep.py [n] [eb]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_06322_b200 import pipeline as PL  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
eb = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
a = S.smooth_noise((n, n, n), seed=0)
h = torch.from_numpy(a).pin_memory()
out = torch.empty(a.nbytes + (256 << 20), dtype=torch.uint8).pin_memory().numpy()
vr = (float(a.min()), float(a.max()))
phi, theta, samples = PL.profile_models(h, eb)
sched = PL.adaptive_schedule(a.shape[0], a[0].nbytes, phi, theta, c_init=16 << 20, c_limit=1 << 30)
res = {"n": n, "phi_samples_gbs": [(c / 2**20, p / 1e9) for c, p in samples],
       "phi": {"alpha": phi.alpha, "beta": phi.beta_slope, "gamma_gbs": phi.gamma / 1e9, "c_thr_mb": phi.c_threshold / 2**20},
       "theta_gbs": 1.0 / theta.beta_copy / 1e9, "adaptive_chunks_planes": sched}


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3, r


for mb in (16, 64, 256):
    cp = max(1, (mb << 20) // a[0].nbytes)
    ms, m = timed(lambda: PL.compress_pipelined(h, eb, value_range=vr, chunk_planes=cp, out=out))
    res[f"fixed_{mb}MB"] = {"ms": ms, "gbs": a.nbytes / ms / 1e6, "cr": a.nbytes / m}
ms, m = timed(lambda: PL.compress_pipelined(h, eb, value_range=vr, chunks=sched, out=out))
res["adaptive"] = {"ms": ms, "gbs": a.nbytes / ms / 1e6, "cr": a.nbytes / m}
print(json.dumps(res))
