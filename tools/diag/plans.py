import os, sys
sys.path.insert(0, os.getcwd())
import bench
from paper_1109_3524_b200 import ibm
for wl in sys.argv[1:]:
    cfg, h, dt, _ = bench.workload(wl)
    st = ibm.Stepper(os.path.join("cases", cfg + ".cfg"), h_min=h, dt=dt)
    hh = st.hierarchy()
    for l in range(hh.n_levels):
        lv = hh.level(l)
        out = []
        for k in ("A", "P", "Pt"):
            m = lv[k]
            b, kind = m.format_bytes()
            out.append("%s %dx%d nnz %d kind %d bytes %.1fMB" % (k, m.rows(), m.cols(), m.nnz(), kind, b / 1e6))
        print(wl, "L%d" % l, " | ".join(out), flush=True)
