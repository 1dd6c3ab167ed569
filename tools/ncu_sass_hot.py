"""Hot SASS of one kernel from an ncu report: instructions executed and stall samples per opcode
and the top individual instructions.   python tools/ncu_sass_hot.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iA, iS, iE, iW = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), \
    hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) <= iE:
        continue
    try:
        e, w = int(r[iE]), int(r[iW])
    except ValueError:
        continue
    data.append((r[iA], r[iS].strip(), e, w))
tot_e = sum(d[2] for d in data) or 1
tot_w = sum(d[3] for d in data) or 1
by_op = collections.Counter()
st_op = collections.Counter()
for a, s, e, w in data:
    op = s.split()[0] if not s.startswith("@") else s.split()[1]
    op = op.split(".")[0]
    by_op[op] += e
    st_op[op] += w
print(f"total warp instructions {tot_e}, stall samples {tot_w}")
for op, e in by_op.most_common(30):
    print(f"  {op:10s} {100 * e / tot_e:5.1f}% inst  {100 * st_op[op] / tot_w:5.1f}% stall")
print("top instructions by stall samples:")
for a, s, e, w in sorted(data, key=lambda d: -d[3])[:top]:
    print(f"  {a[-5:]} {100 * w / tot_w:5.2f}% stall {100 * e / tot_e:5.2f}% inst  {s[:90]}")
