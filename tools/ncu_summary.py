"""Summarise ncu --set full reports: time, DRAM bytes/throughput, occupancy, top stalls."""
import csv, io, re, subprocess, sys

KEYS = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rd"), ("dram__bytes_write.sum", "wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("launch__registers_per_thread", "regs"), ("sm__inst_executed.avg.per_cycle_active", "ipc"),
        ("launch__grid_size", "grid")]
STALLS = "smsp__average_warps_issue_stalled_"

def scale(v, unit):
    return v

for path in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    for row in rows[2:]:
        name = re.search(r"k_[a-z0-9_]+", row[h.index("Kernel Name")]).group(0)
        out = [name]
        for k, lab in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"{lab}={row[i]}{'' if units[i] in ('', 'register/thread') else units[i]}")
        st = []
        for i, c in enumerate(h):
            if c.startswith(STALLS) and c.endswith("_per_issue_active.ratio"):
                try:
                    v = float(row[i])
                except ValueError:
                    continue
                if v > 0.3:
                    st.append((v, c[len(STALLS):-len("_per_issue_active.ratio")]))
        st.sort(reverse=True)
        out.append("stalls: " + ", ".join(f"{n}={v:.1f}" for v, n in st[:5]))
        print(" | ".join(out))
