import sys, time, os, torch, numpy as np
sys.path.insert(0, ".")
from paper_2503_06322_b200 import pipeline as PL, synthetic as S
a = S.smooth_noise((513,)*3, seed=0); h = torch.from_numpy(a).pin_memory()
out = torch.empty(a.nbytes + (64<<20), dtype=torch.uint8).pin_memory().numpy()
for vr in (None, (float(a.min()), float(a.max()))):
    for _ in range(3): m = PL.compress_pipelined(h, 1e-4, value_range=vr, out=out)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5): m = PL.compress_pipelined(h, 1e-4, value_range=vr, out=out)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
    print(os.environ.get("HPDR_PIPE_QUEUES_B"), "rel" if vr is None else "abs", round(dt * 1e3, 2), "ms", round(a.nbytes / dt / 1e9, 1), "GB/s", m)
