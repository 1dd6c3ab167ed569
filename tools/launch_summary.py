"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel launches,
total time and share.   python tools/launch_summary.py launches.csv"""
import collections, csv, re, sys

rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h = r
        start = i + 1
        break
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[start:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    m = re.search(r"\b(k_[a-z0-9_]+)", r[ki]) or re.search(r"(cub[^ (<]*|at::[^ (<]*)", r[ki])
    name = m.group(1) if m else r[ki][:40]
    v = float(r[vi].replace(",", ""))
    v = v * 1000 if r[ui] == "ms" else v / 1000 if r[ui] == "ns" else v
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"# {sum(cnt.values())} launches, {T / 1000:.2f} ms device time (ncu-serialised, cold cache: compare shares)")
print(f"{'kernel':34s} {'launches':>8s} {'total_ms':>9s} {'share':>6s}")
for k, v in tot.most_common():
    print(f"{k:34s} {cnt[k]:8d} {v / 1000:9.2f} {100 * v / T:5.1f}%")
