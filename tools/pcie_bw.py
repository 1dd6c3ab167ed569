"""Pinned host<->device copy bandwidth on this box (the end-to-end roofline denominators).

    python tools/pcie_bw.py [MiB]   -> one JSON line: h2d / d2h / bidirectional GB/s
"""
import json
import sys

import torch


def measure(mib=1024, reps=5):
    n = mib << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        for s in (s1, s2):
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3

    def h2d():
        d.copy_(h, non_blocking=True)

    def d2h():
        h.copy_(d, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    t_h2d, t_d2h, t_bi = timed(h2d), timed(d2h), timed(both)
    return {"bytes": n, "h2d_gbs": n / t_h2d / 1e9, "d2h_gbs": n / t_d2h / 1e9,
            "bidir_each_gbs": n / t_bi / 1e9, "memory": "pinned (cudaHostAlloc via torch pin_memory)"}


if __name__ == "__main__":
    print(json.dumps(measure(int(sys.argv[1]) if len(sys.argv) > 1 else 1024)))
