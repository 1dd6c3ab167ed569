"""Per-CUDA-source-line executed warp instructions from an ncu report (-lineinfo + --import-source).

    python tools/ncu_inst.py report.ncu-rep [top]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
data, fname = [], ""
for r in csv.reader(io.StringIO(raw)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > 7 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            data.append((float(r[7] or 0), float(r[4] or 0), f"{fname}:{r[0]}", r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
stot = sum(d[1] for d in data) or 1
print(f"total warp instructions {tot:.0f}")
for inst, smp, loc, src in sorted(data, reverse=True)[:top]:
    print(f"{100 * inst / tot:5.1f}% inst  {100 * smp / stot:5.1f}% stall  {loc:16s} {src}")
