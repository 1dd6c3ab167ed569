import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2503_06322_b200 as P
from paper_2503_06322_b200 import synthetic as S
a = S.nyx_like((512,)*3, "velocity_x", seed=3)
y = torch.empty(a.shape, dtype=torch.float32, device="cuda")
for eb in (1e-3, 1e-4, 1e-5):
    blob = P.mgard_compress(torch.from_numpy(a).cuda(), eb)
    pin = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).pin_memory().numpy()
    P.mgard_decompress(pin, out=y); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): P.mgard_decompress(pin, out=y)
    e1.record(); e1.synchronize()
    print(eb, len(blob), round(e0.elapsed_time(e1) / 3, 2), "ms")
