"""BASELINE configs[2]: NYX-like 6-field fp32 512^3 set, relative bounds 1e-2..1e-5 -- compression
ratio, error and throughput per field and bound (M1 drop-in path; kernel-only and end to end).

    python tools/sweep_c3.py [n] > c3.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_06322_b200 as P  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512


def ev_ms(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


rows = []
for fi, field in enumerate(S.NYX_FIELDS):
    a = S.nyx_like((n, n, n), field, seed=fi)
    d = torch.from_numpy(a).cuda()
    h = torch.from_numpy(a).pin_memory()
    rng = float(a.max()) - float(a.min())
    for eb in (1e-2, 1e-3, 1e-4, 1e-5):
        blob = P.mgard_compress(d, eb)
        nb = len(blob)
        dev_out = torch.empty(nb + (1 << 20), dtype=torch.uint8, device="cuda")
        h_blob = torch.empty(nb + (1 << 20), dtype=torch.uint8).pin_memory()
        pin = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).pin_memory().numpy()
        y_dev = torch.empty(a.shape, dtype=torch.float32, device="cuda")
        y_h = torch.empty(a.shape, dtype=torch.float32).pin_memory()
        c_ms = ev_ms(lambda: P.mgard_compress(d, eb, out=dev_out))
        ce_ms = ev_ms(lambda: P.mgard_compress(h, eb, out=h_blob))
        d_ms = ev_ms(lambda: P.mgard_decompress(pin, out=y_dev))
        de_ms = ev_ms(lambda: P.mgard_decompress(pin, out=y_h))
        err = float(np.max(np.abs(y_h.numpy().astype(np.float64) - a)))
        gb = a.nbytes / 1e6
        rows.append({"field": field, "eb_rel": eb, "cr": a.nbytes / nb, "max_err_over_eb": err / (eb * rng),
                     "compress_gbs": gb / c_ms, "compress_e2e_gbs": gb / ce_ms,
                     "decompress_gbs": gb / d_ms, "decompress_e2e_gbs": gb / de_ms})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
print(json.dumps({"config": f"configs[2]: NYX-like 6-field fp32 {n}^3, rel 1e-2..1e-5", "rows": rows}))
