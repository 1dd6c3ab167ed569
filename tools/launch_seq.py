"""Per-launch durations (us) of the last call pair in an ncu launch list, in launch order.
    python tools/launch_seq.py launches.csv [calls]"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 4
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h, st = r, i + 1
        break
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
gi = h.index("Grid Size") if "Grid Size" in h else None
seq = []
for r in rows[st:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    m = re.search(r"\b(k_[a-z0-9_]+)", r[ki]) or re.search(r"(cub[^ (<]*)", r[ki])
    v = float(r[vi].replace(",", ""))
    v = v * 1000 if r[ui] == "ms" else v / 1000 if r[ui] == "ns" else v
    seq.append((m.group(1) if m else r[ki][:30], v, r[gi] if gi is not None else ""))
n = len(seq) // calls
tot = 0.0
for name, v, g in seq[-n:]:
    tot += v
    print(f"{name:28s} {v:8.1f}  {g}")
print(f"{n} launches, {tot:.1f} us")
