"""Per-kernel device time of one C3 field / bound (kernel-only compress + decompress, device buffers).

    python tools/c3_probe.py [field] [eb_rel] [n]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_06322_b200 as P  # noqa: E402
from paper_2503_06322_b200 import _lib  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

field = sys.argv[1] if len(sys.argv) > 1 else "velocity_x"
eb = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
n = int(sys.argv[3]) if len(sys.argv) > 3 else 512
a = S.nyx_like((n, n, n), field, seed=0)
d = torch.from_numpy(a).cuda()
blob = P.mgard_compress(d, eb)
db = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).cuda()
out = torch.empty(a.shape, dtype=torch.float32, device="cuda")
print(f"{field} eb {eb}: CR {a.nbytes / len(blob):.3f}")
for name, fn in (("compress", lambda: P.mgard_compress(d, eb)), ("decompress", lambda: P.mgard_decompress(db, out=out))):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    e1.synchronize()
    _lib.prof_enable(True)
    fn()
    torch.cuda.synchronize()
    k = _lib.prof_read()
    _lib.prof_enable(False)
    print(f"== {name}: {e0.elapsed_time(e1):.3f} ms")
    for kk, v in sorted(k.items(), key=lambda kv: -kv[1][1])[:8]:
        print(f"   {kk:24s} n={v[0]:4.0f} {v[1]:8.3f} ms")
