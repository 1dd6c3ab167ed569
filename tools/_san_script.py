
import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2503_06322_b200 as P
from paper_2503_06322_b200 import synthetic as S
# quad pass 1 with TMA (rows of 64 fp32) and with cp.async (odd rows), fused levels, Thomas,
# Huffman, the streamed decompress, the fixed-rate coder, the per-axis rank-4 path and the
# one-block small end of the hierarchy
for shape, dt in (((34, 36, 64), np.float32), ((21, 19, 23), np.float64), ((9, 10, 11, 6), np.float32),
                  ((5,), np.float64)):   # (5,): a payload of a few bits
    a = S.smooth_noise(shape, seed=1, dtype=dt)
    for vr in (None, (-1.0, 2.0)):
        b = P.mgard_compress(a, 1e-3, value_range=vr)
        y = P.mgard_decompress(b).values
        assert np.max(np.abs(y.astype(np.float64) - a)) <= 1e-3 * (3.0 if vr else float(a.max() - a.min()))
    if len(shape) <= 3:
        z = P.zfp_compress(a, 12)
        P.zfp_decompress(z)
print("sanitized run ok")
