"""Record the measured DRAM traffic of one kernel instance for bench.py's roofline.

    ncu --nvtx --nvtx-include "regex:cf:jacobi_merged@L1/" --set full -c 1 \
        -o gpurun_out/full_c2 python tools/profile_step.py --config c2 --profile
    python tools/traffic.py c2 jacobi_merged@L1 gpurun_out/full_c2.ncu-rep

Writes profiles/traffic_<cfg>.json: {"<kind>@L<level>": dram bytes (read + write) per
launch, averaged over the captured launches, "_meta": {...}}.  bench.py reports it
as roofline.traffic for the dominant instance.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg, inst, rep = sys.argv[1:4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9}
tscale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}


def col(r, key, table):
    i = hdr.index(key)
    return float(r[i].replace(",", "")) * table[units[i]]


launches = []
for r in rows[2:]:
    b = col(r, "dram__bytes_read.sum", scale) + col(r, "dram__bytes_write.sum", scale)
    launches.append((r[hdr.index("Kernel Name")].split("(")[0], b,
                     col(r, "gpu__time_duration.sum", tscale)))
if not launches:
    sys.exit("no launches in " + rep)
path = os.path.join(ROOT, "profiles", f"traffic_{cfg}.json")
data = json.load(open(path)) if os.path.exists(path) else {}
per = sum(b for _, b, _ in launches) / len(launches)
data[inst] = per
meta = data.setdefault("_meta", {})
meta[inst] = {"kernels": sorted({k for k, _, _ in launches}), "launches": len(launches),
              "ms_per_launch_under_ncu": sum(t for _, _, t in launches) / len(launches),
              "dram_gbs_under_ncu": per / (sum(t for _, _, t in launches) / len(launches)) / 1e6,
              "source": os.path.basename(rep) + " (ncu --set full, dram__bytes_read.sum + "
                        "dram__bytes_write.sum)"}
with open(path, "w") as f:
    json.dump(data, f, indent=1, sort_keys=True)
print(inst, f"{per / 1e9:.4f} GB per launch", meta[inst])
