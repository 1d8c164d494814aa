"""Measured DRAM traffic of one solve-2 SA-PCG iteration from an ncu launch list with
dram__bytes_read.sum / dram__bytes_write.sum (tools/profile_step.py under ncu, IBMGPU_EAGER=1).
Iterations are delimited by the B1 kernel (k_spmv_*<XPlain, EpiSpmvPAp>) on lhs2 (grid = the
given block count); only complete iterations are counted.

  python tools/traffic_per_iteration.py launches.csv --b1-grid 16281
"""
import argparse
import csv
import json
from collections import defaultdict

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--b1-grid", required=True)
a = ap.parse_args()
rows = [r for r in csv.reader(open(a.csv)) if len(r) > 14 and r[0].isdigit()]
k = defaultdict(dict)
name, grid = {}, {}
for r in rows:
    i = int(r[0])
    name[i], grid[i] = r[4], r[8]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
             "msecond": 1e3}.get(r[13])
    try:
        k[i][r[12]] = float(r[14].replace(",", "")) * scale
    except (ValueError, TypeError):
        pass
ids = sorted(k)
starts = [i for i in ids if "EpiSpmvPAp" in name[i] and grid[i].startswith("(" + a.b1_grid + ",")]
it_bytes, it_ms = [], []
for s, e in zip(starts, starts[1:]):
    seg = [i for i in ids if s <= i < e]
    if not all(len(k[i]) == 3 for i in seg):
        continue
    it_bytes.append(sum(k[i]["dram__bytes_read.sum"] + k[i]["dram__bytes_write.sum"] for i in seg))
    it_ms.append(sum(k[i]["gpu__time_duration.sum"] for i in seg))
print(json.dumps({"iterations": len(it_bytes), "dram_bytes_per_iteration": sum(it_bytes) / max(len(it_bytes), 1),
                  "serialised_us_per_iteration": sum(it_ms) / max(len(it_ms), 1)}))
