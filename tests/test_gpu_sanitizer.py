"""compute-sanitizer over a small compress / decompress round trip on every kernel family:
memcheck (out-of-bounds / misaligned device accesses, leaks), racecheck (shared-memory
hazards, including the mbarrier-ordered TMA ring of k_pass1_quad) and initcheck (device memory
read before it is written, including the payload copies of the streamed drop-in paths)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SANITIZER = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r)
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
"""


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "initcheck"])
def test_compute_sanitizer_clean(tool):
    if not os.path.exists(SANITIZER):
        pytest.skip("compute-sanitizer not found")
    cmd = [SANITIZER, "--tool", tool, "--error-exitcode", "99"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    r = subprocess.run(cmd + [sys.executable, "-c", _SCRIPT % ROOT], capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "sanitized run ok" in out, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-4000:]
