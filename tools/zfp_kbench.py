"""Device-resident fixed-rate coder timing (kernel-only) for quick iteration and ncu captures:
    python tools/zfp_kbench.py [rate] [f32|f64] [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2503_06322_b200 import synthetic as S
from paper_2503_06322_b200 import zfp as Z
from paper_2503_06322_b200.tensor import DType

rate = int(sys.argv[1]) if len(sys.argv) > 1 else 16
dt = np.float64 if len(sys.argv) > 2 and sys.argv[2] == "f64" else np.float32
n = int(sys.argv[3]) if len(sys.argv) > 3 else 513
a = S.smooth_noise((n, n, n), seed=0, dtype=dt)
d_in = torch.from_numpy(a).cuda()
ln = Z.compressed_size(a.shape, DType.F32 if dt == np.float32 else DType.F64, rate)
d_z = torch.empty(ln, dtype=torch.uint8, device="cuda")
d_out = torch.empty_like(d_in)
for name, fn in (("compress", lambda: Z.zfp_compress(d_in, rate, out=d_z)),
                 ("decompress", lambda: Z.zfp_decompress(d_z, out=d_out))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {ms:.3f} ms  {a.nbytes / ms / 1e6:.1f} GB/s (field)  {(a.nbytes + ln) / ms / 1e6:.1f} GB/s (field+stream)")
