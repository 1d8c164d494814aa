"""Row-slab decomposition on CPU: the product's host halo planner
(ibmgpu_distplan_*, ibmgpu_partition_*) checked for local-SpMV exactness and send/recv
consistency, and a world_size-2 gloo run of the distributed SA-PCG algorithm of csrc/dist.cu —
same plans, same level switch, same reductions — on the reference's golden small-case hierarchy,
compared with the reference's own solve (tests/golden/small_case.npz bench_x / bench_iters)."""
import os
import socket

import numpy as np
import pytest

from paper_1109_3524_b200 import ibm
from tests import helpers as H


def _rand_csr(rng, rows, cols, density):
    rp, ci, v = [0], [], []
    for _ in range(rows):
        c = np.sort(rng.choice(cols, size=rng.integers(0, max(1, int(cols * density)) + 1), replace=False))
        ci.extend(c.tolist())
        v.extend(rng.standard_normal(len(c)).tolist())
        rp.append(len(ci))
    return np.array(rp, np.int32), np.array(ci, np.int32), np.array(v)


def _spmv_rows(rp, ci, v, x):
    """Row sums in stored order (the device kernels' order)."""
    y = np.zeros(len(rp) - 1)
    for i in range(len(rp) - 1):
        s = 0.0
        for k in range(rp[i], rp[i + 1]):
            s += v[k] * x[ci[k]]
        y[i] = s
    return y


@pytest.mark.parametrize("R", [1, 2, 3, 5])
def test_plan_local_spmv_and_exchange_consistency(R):
    rng = np.random.default_rng(7 + R)
    rows, cols = 120, 90
    rp, ci, v = _rand_csr(rng, rows, cols, 0.06)
    ro = rng.integers(0, R, rows).astype(np.int32)
    co = rng.integers(0, R, cols).astype(np.int32)
    x = rng.standard_normal(cols)
    y = _spmv_rows(rp, ci, v, x)
    plans = [ibm.DistPlan.build(rows, cols, rp, ci, v, ro, co, r, R) for r in range(R)]
    for r, P in enumerate(plans):
        assert np.array_equal(P.rows, np.flatnonzero(ro == r))
        assert np.array_equal(P.own, np.flatnonzero(co == r))
        # halo grouped by owner, ascending inside a group, and never owned
        for q in range(R):
            seg = P.halo[P.recv_off[q]:P.recv_off[q + 1]]
            assert np.all(co[seg] == q) and np.all(np.diff(seg) > 0)
            assert q != r or len(seg) == 0
        # local SpMV on [own | halo] reproduces the global rows bit for bit
        xe = np.concatenate([x[P.own], x[P.halo]])
        assert np.array_equal(_spmv_rows(P.rptr, P.cidx, P.val, xe), y[P.rows])
        # what r sends to q is exactly q's halo segment for r
        for q in range(R):
            sent = P.own[P.send_idx[P.send_off[q]:P.send_off[q + 1]]]
            Q = plans[q]
            assert np.array_equal(sent, Q.halo[Q.recv_off[r]:Q.recv_off[r + 1]])


def test_plan_rejects_bad_rank():
    rp, ci, v = np.array([0, 1], np.int32), np.array([0], np.int32), np.array([1.0])
    with pytest.raises(ValueError):
        ibm.DistPlan.build(1, 1, rp, ci, v, np.zeros(1, np.int32), np.zeros(1, np.int32), 2, 2)


def test_partition_lambda_slabs_and_bodies():
    nx, ny, R = 10, 7, 3
    bj = np.array([0, 3, 6, 6], np.int32)
    own = ibm.partition_lambda(nx, ny, bj, R)
    np_ = nx * ny
    slab = (np.arange(ny) * R) // ny
    assert np.array_equal(own[:np_].reshape(ny, nx), np.repeat(slab[:, None], nx, axis=1))
    assert np.array_equal(own[np_:np_ + 4], slab[bj]) and np.array_equal(own[np_ + 4:], slab[bj])
    counts = np.bincount(own[:np_], minlength=R)
    assert counts.max() - counts.min() <= nx


def test_partition_coarse_lowest_member():
    agg = np.array([1, 0, 1, 2, 0, 2], np.int32)
    of = np.array([2, 1, 0, 0, 1, 1, 3, 0], np.int32)  # 6 core rows + 2 tail
    oc = ibm.partition_coarse(agg, 6, 3, 2, of)
    assert oc.tolist() == [1, 2, 0, 3, 0]


# ------------------------------------------------------------------ gloo world_size 2
def _csr(d, key):
    return H.small_mat(d, key)


def _cell_j(y_faces, y):
    return np.clip(np.searchsorted(y_faces, y, side="right") - 1, 0, len(y_faces) - 2).astype(np.int32)


class _Rank:
    """numpy mirror of one rank of csrc/dist.cu (plans from the product's planner)."""

    def __init__(self, d, rank, R, min_rows):
        import torch.distributed as dist
        self.dist, self.rank, self.R = dist, rank, R
        nx, ny, n_b = int(d["dims"][0]), int(d["dims"][1]), int(d["dims"][4])
        A0 = _csr(d, "lhs2")
        self.L = int(d["n_levels"])
        lev = [dict(A=_csr(d, f"L{l}_A"), P=_csr(d, f"L{l}_P"), Pt=_csr(d, f"L{l}_Pt"), agg=d[f"L{l}_agg"],
                    omega=float(d[f"L{l}_omega"][0])) for l in range(self.L)]
        owner = [ibm.partition_lambda(nx, ny, _cell_j(d["grid_y_faces"], d["body_y"]), R)]
        D = 0
        while D < self.L and lev[D]["A"].rows >= min_rows:
            D += 1
        self.D = max(D, 1)
        for l in range(self.D):
            Al = lev[l]["A"]
            n_core = Al.rows - 2 * n_b
            owner.append(ibm.partition_coarse(lev[l]["agg"], n_core, int(lev[l]["agg"][:n_core].max()) + 1,
                                              2 * n_b, owner[l]))
        self.lev, self.owner = lev, owner

        def plan(M, ro, co):
            return ibm.DistPlan.build(M.rows, M.cols, M.rp, M.ci, M.v, ro, co, rank, R)

        self.pA = plan(A0, owner[0], owner[0])
        self.pl = []
        for l in range(self.D):
            M = lev[l]
            e = dict(A=plan(M["A"], owner[l], owner[l]))
            wd = M["omega"] / M["A"].diagonal()
            e["wd"] = np.concatenate([wd[e["A"].own], wd[e["A"].halo]])
            if l < self.D - 1:
                e["Pt"] = plan(M["Pt"], owner[l + 1], owner[l])
                e["P"] = plan(M["P"], owner[l], owner[l + 1])
            else:  # switch: rank-partial restriction, P against the full (replicated) coarse vector
                Pt = M["Pt"]
                keep = owner[l][Pt.ci] == rank
                g2l = -np.ones(Pt.cols, np.int64)
                g2l[owner[l] == rank] = np.arange(int(np.sum(owner[l] == rank)))
                rows_of = np.repeat(np.arange(Pt.rows), np.diff(Pt.rp))
                e["PtC"] = (rows_of[keep], g2l[Pt.ci[keep]], Pt.v[keep], Pt.rows)
                e["P"] = plan(M["P"], owner[l], np.full(M["P"].cols, rank, np.int32))
            self.pl.append(e)
        # replicated tail: full operators from level D, coarse solve dense
        Ac = lev[-1]["Pt"].dense() @ lev[-1]["A"].dense() @ lev[-1]["P"].dense()
        self.coarse_inv = np.linalg.inv(Ac)

    # --- communication (the NCCL calls of dist.cu, over gloo)
    def halo(self, P, x_own):
        import torch
        x_ext = np.concatenate([x_own, np.zeros(len(P.halo))])
        reqs, bufs = [], []
        for q in range(self.R):
            if q == self.rank:
                continue
            ns = P.send_off[q + 1] - P.send_off[q]
            nr = P.recv_off[q + 1] - P.recv_off[q]
            if ns:
                reqs.append(self.dist.isend(torch.from_numpy(x_own[P.send_idx[P.send_off[q]:P.send_off[q + 1]]].copy()), q))
            if nr:
                t = torch.zeros(nr, dtype=torch.float64)
                reqs.append(self.dist.irecv(t, q))
                bufs.append((P.recv_off[q], t))
        for rq in reqs:
            rq.wait()
        for off, t in bufs:
            x_ext[len(x_own) + off:len(x_own) + off + len(t)] = t.numpy()
        return x_ext

    def allreduce(self, a):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(a, np.float64).copy())
        self.dist.all_reduce(t)
        return t.numpy()

    @staticmethod
    def spmv(P, x_ext):
        return _spmv_rows(P.rptr, P.cidx, P.val, x_ext)

    # --- V-cycle (amg.hpp:198-225, distributed as dist.cu dist_vcycle)
    def vcycle_full(self, l, b):
        if l == self.L:
            return self.coarse_inv @ b
        M = self.lev[l]
        wd = M["omega"] / M["A"].diagonal()
        x = wd * b
        r = b - M["A"].spmv_np(x)
        x = x + M["P"].spmv_np(self.vcycle_full(l + 1, M["Pt"].spmv_np(r)))
        return x + wd * (b - M["A"].spmv_np(x))

    def vcycle(self, l, b_own):
        e = self.pl[l]
        PA = e["A"]
        n = len(PA.own)
        b_ext = self.halo(PA, b_own)
        x = e["wd"][:n] * b_own
        r = b_own - _spmv_rows(PA.rptr, PA.cidx, PA.val, e["wd"] * b_ext)
        if l < self.D - 1:
            bc = self.spmv(e["Pt"], self.halo(e["Pt"], r))
            xc_ext = self.halo(e["P"], self.vcycle(l + 1, bc))
        else:
            ri, ci, v, nrows = e["PtC"]
            part = np.zeros(nrows)
            np.add.at(part, ri, v * r[ci])
            xc_ext = self.vcycle_full(l + 1, self.allreduce(part))
        x = x + self.spmv(e["P"], xc_ext)
        return x + e["wd"][:n] * (b_own - self.spmv(PA, self.halo(PA, x)))

    def pcg(self, b_full, tol=1e-5, max_iters=200):
        """krylov.hpp:70-136 in dist.cu's single-reduction form: w = A z and ONE allreduce of
        {r.r, r.z, z.w, z.Ap_old} per iteration; A p = w + beta Ap_old, p.Ap by recurrence."""
        P = self.pA
        b = b_full[P.own]
        x = np.zeros(len(b))
        r = b - self.spmv(P, self.halo(P, x))
        bb, rr = self.allreduce([b @ b, r @ r])
        bnorm = np.sqrt(bb)
        if np.sqrt(rr) / bnorm <= tol:
            return x, 0
        p, Ap = np.zeros(len(b)), np.zeros(len(b))
        rz_old = pAp_old = 0.0
        it = 0
        while True:
            z = self.vcycle(0, r)
            w = self.spmv(P, self.halo(P, z))
            rr, rz, zw, zap = self.allreduce([r @ r, r @ z, z @ w, z @ Ap])
            if it > 0:
                if np.sqrt(rr) / bnorm <= tol or it >= max_iters:
                    return x, it
            beta = 0.0 if it == 0 else rz / rz_old
            pAp = zw if it == 0 else zw + 2.0 * beta * zap + beta * beta * pAp_old
            assert pAp > 0
            alpha = rz / pAp
            p = z + beta * p
            Ap = w + beta * Ap
            x += alpha * p
            r -= alpha * Ap
            rz_old, pAp_old = rz, pAp
            it += 1


def _worker(rank, R, port, min_rows, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=R)
    try:
        d = H.small()
        rk = _Rank(d, rank, R, min_rows)
        x_own, iters = rk.pcg(d["bench_b"])
        q.put((rank, rk.pA.own.tolist(), x_own.tolist(), iters, rk.D, len(rk.pA.halo)))
    except Exception as e:  # surface to the parent
        q.put((rank, None, repr(e), -1, -1, -1))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("min_rows", [0, 1000])
def test_gloo_world2_distributed_sa_pcg_matches_reference(min_rows):
    import torch.multiprocessing as mp
    R = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, R, port, min_rows, q)) for r in range(R)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(R)]
    for p in procs:
        p.join(timeout=60)
    d = H.small()
    n = len(d["bench_b"])
    x = np.full(n, np.nan)
    iters = set()
    for rank, own, xo, it, D, nh in sorted(out):
        assert own is not None, xo
        x[np.array(own, int)] = xo
        iters.add(it)
        assert nh > 0  # the slabs really exchange halos
    assert len(iters) == 1  # identical control flow on both ranks
    it = iters.pop()
    assert abs(it - int(np.ravel(d["bench_iters"])[0])) <= 2
    xr = d["bench_x"]
    assert np.linalg.norm(x - xr) <= 1e-5 * np.linalg.norm(xr)
