"""Column spans of the rows of P_l^T A_l (the first Galerkin product) per level: how many rows would
fit a dense window accumulator of W columns."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import scipy.sparse as sp
from paper_1109_3524_b200 import ibm
import bench
wl = sys.argv[1] if len(sys.argv) > 1 else "flapping"
cfg, h, dt, _ = bench.workload(wl)
st = ibm.Stepper(os.path.join("cases", cfg + ".cfg"), h_min=h, dt=dt)
hh = st.hierarchy()
def S(m):
    rp, ci, v = m.csr()
    return sp.csr_matrix((v, ci, rp), shape=(m.rows(), m.cols()))
for l in range(hh.n_levels):
    lv = hh.level(l)
    A, Pt = S(lv["A"]), S(lv["Pt"])
    T = (Pt @ A).tocsr()
    T.sort_indices()
    rp = T.indptr
    nz = np.diff(rp) > 0
    first = np.where(nz, T.indices[np.minimum(rp[:-1], len(T.indices) - 1)], 0)
    last = np.where(nz, T.indices[np.maximum(rp[1:] - 1, 0)], 0)
    span = last - first + 1
    prods = np.diff(rp)
    print(wl, "L%d" % l, "rows", T.shape[0], "cols", T.shape[1], "nnz/row %.0f" % (T.nnz / T.shape[0]),
          " ".join("span<=%d: %.3f" % (W, np.mean(span <= W)) for W in (4096, 12288, 16384, 32768)), flush=True)
