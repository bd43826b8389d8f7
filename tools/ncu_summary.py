"""Summarise an ncu report (raw page) into a small text table.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN/ncu_<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__bytes.sum.per_second", "dram_bw"),
    ("dram__cycles_active.avg.pct_of_peak_sustained_elapsed", "dram_active_%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_registers", "ctas/sm(regs)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("launch__grid_size", "grid"),
]

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
idx = {k: hdr.index(k) for k, _ in KEYS if k in hdr}
kn = hdr.index("Kernel Name")
print("# " + rep)
for r in rows[2:]:
    name = r[kn].split("(")[0]
    vals = [f"{lab}={r[idx[k]]}{units[idx[k]]}" for k, lab in KEYS if k in idx]
    print(name, " ".join(vals))
