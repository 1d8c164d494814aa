"""Brief per-kernel summary of an ncu --set full report: duration, DRAM GB/s and bytes, occupancy,
IPC, instructions per launch and the top stall reasons.  python tools/ncu_brief.py REP [substr]"""
import csv, subprocess, sys

rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
units = rows[1]
col = {n: i for i, n in enumerate(h)}
SCALE = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1.0, "byte": 1.0,
         "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size"]
stalls = [n for n in h if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    if sub not in name:
        continue
    g = lambda n: (float(r[col[n]].replace(",", "")) * SCALE.get(units[col[n]], 1.0)
                   if n in col and r[col[n]] else 0.0)
    t = g("gpu__time_duration.sum")  # ns (units row says)
    by = g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
    st = sorted(((g(n), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]) for n in stalls),
                reverse=True)[:5]
    print("%-40s %8.1f us %7.1f MB %6.0f GB/s occ %4.1f%% ipc %.2f inst %.1fM regs %d grid %d | %s" % (
        name[:40], t / 1e3, by / 1e6, by / t if t else 0, g("sm__warps_active.avg.pct_of_peak_sustained_active"),
        g("sm__inst_executed.avg.per_cycle_active"), g("smsp__inst_executed.sum") / 1e6,
        g("launch__registers_per_thread"), g("launch__grid_size"), " ".join("%s %.1f" % (n, v) for v, n in st)))
