"""Summarise an ncu --csv launch list: per-kernel count, total/avg time, DRAM bytes, GB/s, share."""
import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    n = re.sub(r"\(.*", "", name) if not name.startswith("void ") else name[5:]
    n = re.sub(r"ibmgpu::|<unnamed>::|\(anonymous namespace\)::", "", n)
    m = re.match(r"([\w:]+)<(.*)>\(", n)
    if m:
        args = m.group(2)
        epi = re.findall(r"(Epi\w+|Body\w+|XJacobi|XPlain|LastDot|Fin\w+)", args)
        return m.group(1) + "<" + ",".join(dict.fromkeys(epi)) + ">"
    return re.sub(r"\(.*", "", n)


def main(path):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    hdr = rows[0]
    ix = {k: i for i, k in enumerate(hdr)}
    per = defaultdict(lambda: {"n": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0})
    seen = set()
    for r in rows[1:]:
        kid, name, metric, val = r[ix["ID"]], r[ix["Kernel Name"]], r[ix["Metric Name"]], r[ix["Metric Value"]]
        grid = r[ix["Grid Size"]]
        key = short(name) + " " + grid if "spmv" in name else short(name)
        v = float(val.replace(",", "")) if val else 0.0
        unit = r[ix["Metric Unit"]]
        d = per[key]
        if (kid, "id") not in seen:
            seen.add((kid, "id"))
            d["n"] += 1
        if metric == "gpu__time_duration.sum":
            d["ns"] += v * (1e3 if unit == "usecond" else 1e6 if unit == "msecond" else 1.0)
        elif metric == "dram__bytes_read.sum":
            d["rd"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        elif metric == "dram__bytes_write.sum":
            d["wr"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    tot = sum(d["ns"] for d in per.values())
    print(f"total kernel time {tot/1e6:.3f} ms over {sum(d['n'] for d in per.values())} launches")
    print(f"{'kernel':78s} {'n':>6s} {'tot ms':>9s} {'avg us':>8s} {'share':>6s} {'GB/s':>7s} {'MB/launch':>9s}")
    for k, d in sorted(per.items(), key=lambda kv: -kv[1]["ns"]):
        gbs = (d["rd"] + d["wr"]) / d["ns"] if d["ns"] else 0
        print(f"{k[:78]:78s} {d['n']:6d} {d['ns']/1e6:9.3f} {d['ns']/max(d['n'],1)/1e3:8.2f} "
              f"{100*d['ns']/tot:5.1f}% {gbs:7.0f} {(d['rd']+d['wr'])/max(d['n'],1)/1e6:9.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
