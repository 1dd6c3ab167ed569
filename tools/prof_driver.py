"""Small driver for ncu captures: one warm compress+decompress, then one measured pair."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2503_06322_b200 as P
from paper_2503_06322_b200 import synthetic as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
a = S.smooth_noise((n, n, n), seed=0)
for _ in range(2):
    b = P.mgard_compress(a, 1e-4)
    y = P.mgard_decompress(b)
print("ok", len(b))
