"""Cost of cudaHostRegister / first-touch / pinned copies on this box (pageable-path design probe)."""
import ctypes, time, os, sys
import numpy as np, torch
cr = ctypes.CDLL("libcudart.so.12") if False else None
rt = torch.cuda.cudart()
torch.cuda.init()
def t(f):
    t0 = time.perf_counter(); r = f(); return time.perf_counter() - t0, r
for gb in (0.86, 4.29):
    n = int(gb * 1e9)
    a = np.ones(n, np.uint8)               # touched
    dt, _ = t(lambda: rt.cudaHostRegister(a.ctypes.data, n, 0))
    du, _ = t(lambda: rt.cudaHostUnregister(a.ctypes.data))
    b = np.empty(n, np.uint8)              # untouched
    dtu, _ = t(lambda: rt.cudaHostRegister(b.ctypes.data, n, 0))
    rt.cudaHostUnregister(b.ctypes.data)
    df, _ = t(lambda: np.empty(n, np.uint8).fill(0))
    dp, p = t(lambda: torch.empty(n, dtype=torch.uint8).pin_memory())
    print(f"{gb} GB: register touched {dt*1e3:.1f} ms, unregister {du*1e3:.1f} ms, register untouched {dtu*1e3:.1f} ms, "
          f"first-touch fill {df*1e3:.1f} ms, torch pin_memory {dp*1e3:.1f} ms", flush=True)
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
