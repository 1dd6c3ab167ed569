"""Per-CUDA-source-line stall samples from an ncu report (needs -lineinfo + --import-source).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
data, fname = [], ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > 6 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            data.append((float(r[4] or 0), float(r[7] or 0), f"{fname}:{r[0]}", r[1].strip()[:100]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
for s, inst, loc, src in sorted(data, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  inst={inst:12.0f}  {loc:16s} {src}")
