"""Per-kernel summary of an ncu launch list captured with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv:
launches, mean duration, DRAM bytes per launch and GB/s.  python tools/traffic_summary.py CSV [top]"""
import collections
import csv
import sys

SCALE = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ki, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
d = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    if len(r) <= vi:
        continue
    d[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    names[r[ii]] = r[ki].split("(")[0][:70]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in d.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(v[1] for v in agg.values())
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("total kernel time %.1f us over %d launches" % (tot / 1e3, sum(v[0] for v in agg.values())))
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print("%-70s n%4d avg %7.1f us %7.1f MB %6.0f GB/s %5.1f%%" % (k, v[0], v[1] / v[0] / 1e3, v[2] / v[0] / 1e6,
                                                                 v[2] / v[1] if v[1] else 0, 100 * v[1] / tot))
