"""Per-kernel timing of one configuration (library's live CUDA-event profiler).

    python tools/kbench.py [n] [reps]      # env vars select kernel variants (HPDR_*)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_06322_b200 as P  # noqa: E402
from paper_2503_06322_b200 import _lib  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
a = S.smooth_noise((n, n, n), seed=0)
d = torch.from_numpy(a).cuda()
blob = P.mgard_compress(d, 1e-4)
pin = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).pin_memory().numpy()
out = torch.empty(a.shape, dtype=torch.float32, device="cuda")
for _ in range(2):
    P.mgard_compress(d, 1e-4)
    P.mgard_decompress(pin, out=out)
res = {}
for name, fn in (("compress", lambda: P.mgard_compress(d, 1e-4)),
                 ("decompress", lambda: P.mgard_decompress(pin, out=out))):
    torch.cuda.synchronize()
    _lib.prof_enable("serial" if os.environ.get("KB_SERIAL") else True)
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) / reps * 1e3
    k = _lib.prof_read()
    _lib.prof_enable(False)
    res[name] = {"wall_ms": round(wall, 3),
                 "kernels": {kk: [round(v[1] / reps, 4), round(v[2] / max(v[1], 1e-9) / 1e6, 1)]
                             for kk, v in sorted(k.items(), key=lambda kv: -kv[1][1])}}
env = {k: v for k, v in os.environ.items() if k.startswith("HPDR_")}
print(json.dumps({"env": env, "n": n, **res}))
assert P.mgard_compress(d, 1e-4) == blob
