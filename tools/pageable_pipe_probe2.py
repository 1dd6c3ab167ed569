import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2503_06322_b200 import pipeline as PL, synthetic as S
a = S.smooth_noise((513,) * 3, seed=0)
vr = (float(a.min()), float(a.max()))
out = np.empty(a.nbytes + (1 << 20), np.uint8)
for _ in range(2): n = PL.compress_pipelined(a, 1e-4, value_range=vr, out=out)
t = time.perf_counter(); n = PL.compress_pipelined(a, 1e-4, value_range=vr, out=out); print("pageable in, preallocated pageable out: %.1f ms" % ((time.perf_counter() - t) * 1e3))
import torch
pin = torch.empty(a.nbytes + (1 << 20), dtype=torch.uint8).pin_memory().numpy()
for _ in range(2): n = PL.compress_pipelined(a, 1e-4, value_range=vr, out=pin)
t = time.perf_counter(); n = PL.compress_pipelined(a, 1e-4, value_range=vr, out=pin); print("pageable in, pinned out: %.1f ms" % ((time.perf_counter() - t) * 1e3))
t = time.perf_counter(); c = PL.compress_pipelined(a, 1e-4, value_range=vr); print("pageable in, bytes out: %.1f ms" % ((time.perf_counter() - t) * 1e3))
