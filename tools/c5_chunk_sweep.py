"""BASELINE configs[4]: streaming host-to-host pipeline over 1024^3 fp32 timesteps, chunk-size
sweep 16 MB - 1 GB (plus the Algorithm-4 adaptive schedule).  Each timestep is a fresh field
(seed t) compressed through the same persistent context; times are per timestep.

    python tools/c5_chunk_sweep.py [timesteps] [eb] > c5.json
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

T = int(sys.argv[1]) if len(sys.argv) > 1 else 2
eb = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2
n = 1024
steps = [torch.from_numpy(S.smooth_noise((n, n, n), seed=t)).pin_memory() for t in range(T)]
nbytes = steps[0].numel() * 4
out = torch.empty(nbytes + (512 << 20), dtype=torch.uint8).pin_memory().numpy()
y = torch.empty((n, n, n), dtype=torch.float32).pin_memory().numpy()
plane = n * n * 4
res = {"config": f"configs[4]: 1024^3 fp32 timesteps x{T}, rel {eb} (range known per timestep: absolute bound)",
       "rows": []}
models = PL.profile_models(steps[0], eb)[:2]
sched = PL.adaptive_schedule(n, plane, *models, c_init=16 << 20, c_limit=1 << 30)
for label, kw in [(f"fixed {mb} MB", {"chunk_planes": max(1, (mb << 20) // plane)}) for mb in (16, 32, 64, 128, 256, 512, 1024)] + \
        [("adaptive (Algorithm 4)", {"chunks": sched})]:
    vrs = [(float(s.min()), float(s.max())) for s in steps]
    PL.compress_pipelined(steps[0], eb, value_range=vrs[0], out=out, **kw)   # warm buffers
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lens = [PL.compress_pipelined(s, eb, value_range=vr, out=out, **kw) for s, vr in zip(steps, vrs)]
    torch.cuda.synchronize()
    tc = (time.perf_counter() - t0) / T
    blob = torch.from_numpy(out[: lens[-1]].copy()).pin_memory().numpy()
    PL.decompress_pipelined(blob, out=y)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(T):
        PL.decompress_pipelined(blob, out=y)
    torch.cuda.synchronize()
    td = (time.perf_counter() - t0) / T
    res["rows"].append({"chunks": label, "compress_gbs": nbytes / tc / 1e9, "decompress_gbs": nbytes / td / 1e9,
                        "cr": nbytes / lens[-1]})
    print(json.dumps(res["rows"][-1]), file=sys.stderr, flush=True)
res["adaptive_schedule_planes"] = [int(x) for x in sched]
print(json.dumps(res))
