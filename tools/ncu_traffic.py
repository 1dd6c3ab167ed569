"""Write profiles/ncu_traffic.json: DRAM bytes (read + write) per launch from ncu --set full reports.

    python tools/ncu_traffic.py <dir with LABEL.ncu-rep files> <bench config, e.g. target> [out.json]
The report file name is the bench's kernel label (pass1q.ncu-rep -> k_level_pass1q, ...); results are
stored under the bench config they were captured on (bench.py reads profiles/ncu_traffic.json[config]).
"""
import csv, io, json, os, subprocess, sys

LABELS = {"pass1q": "k_level_pass1q", "pass1r": "k_level_pass1r", "pass2": "k_level_pass2", "minmax": "k_minmax",
          "final": "k_level_final", "decode": "k_decode", "encode": "k_encode", "thomas": "k_thomas"}
d = sys.argv[1]
config = sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                         "profiles", "ncu_traffic.json")
allres = json.load(open(out)) if os.path.exists(out) else {}
res = allres.setdefault(config, {})   # merge: other kernels keep their captures
for f in sorted(os.listdir(d)):
    if not f.endswith(".ncu-rep"):
        continue
    lab = LABELS.get(f[:-8], f[:-8])
    raw = subprocess.run(["ncu", "-i", os.path.join(d, f), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    for r in rows[2:3]:   # first captured launch
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(m)
            v = float(r[i].replace(",", ""))
            u = units[i]
            tot += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        t = h.index("gpu__time_duration.sum")
        res[lab] = tot
        res[lab + ".ncu_us"] = float(r[t].replace(",", "")) * (1000 if units[t] == "ms" else 1)
json.dump(allres, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
