// assemble.cu — the grid operators of operators.hpp assembled on the device, bit-identical to the
// reference (and to csrc/host/case.cpp, which the CPU tests pin against it):
//   metric M        operators.hpp:75-84    u row: del_x[i_f-1] / dy[j]; v row: del_y[j_f-1] / dx[i]
//   diffusion L     operators.hpp:94-194   5-point rows in (south, west, diagonal, east, north)
//                                          order with exact zeros dropped, and the wall couplings
//                                          (BcCoupling) in the reference's per-row order
//   gradient G      operators.hpp:210-228  u row: -1 at p(i_f-1, j), +1 at p(i_f, j); v alike
// One thread per velocity unknown; every product/quotient/sum is an explicit round-to-nearest
// intrinsic in the reference's association order (no FMA contraction), so a 64M-cell grid's
// operators never exist on the host (time-to-first-step at C5-8192: SURVEY §8(f)4).
#include <algorithm>

#include "assemble.cuh"
#include "kern.cuh"

namespace ibmgpu {
namespace {

inline int nblk(long long n, int b = 256) { return (int)((n + b - 1) / b); }

struct DGrid {
    int nx, ny;
    const double *dx, *dy, *del_x, *del_y;
    __device__ int n_u() const { return (nx - 1) * ny; }
    __device__ int u_id(int i_f, int j) const { return (i_f - 1) + j * (nx - 1); }
    __device__ int v_id(int i, int j_f) const { return n_u() + i + (j_f - 1) * nx; }
};

__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double ml(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ad(double a, double b) { return __dadd_rn(a, b); }

// Wall slots of BcCoupling (boundary.hpp:36-40 order of BoundaryState arrays)
enum Slot { LU, RU, LV, RV, BV, TV, BU, TU };

struct Row {
    int n = 0, nb = 0;
    int c[5];
    double v[5];
    int bslot[4], bidx[4];
    double bcoef[4];
    __device__ void put(int col, double val) {
        if (val != 0.0) c[n] = col, v[n] = val, ++n;  // from_triplets drops exact zeros (sparse.hpp:59)
    }
    __device__ void wall(int slot, int idx, double coef) {
        bslot[nb] = slot, bidx[nb] = idx, bcoef[nb] = coef, ++nb;
    }
};

// operators.hpp:100-146 (u rows)
__device__ void u_row(const DGrid& g, int j, int i_f, Row& o) {
    const int nx = g.nx, ny = g.ny;
    const int row = g.u_id(i_f, j);
    const double sm = g.del_x[i_f - 1], dyj = g.dy[j];
    double dh = 0.0, wv = 0, ev = 0, sv = 0, nv = 0;
    const bool hw = i_f - 1 >= 1, he = i_f + 1 <= nx - 1, hs = j > 0, hn = j < ny - 1;
    {
        const double w_hat = dv(1.0, ml(sm, g.dx[i_f - 1]));
        dh = ad(dh, w_hat);
        if (hw) wv = dv(1.0, ml(dyj, g.dx[i_f - 1]));
        else o.wall(LU, j, ml(sm, w_hat));
    }
    {
        const double w_hat = dv(1.0, ml(sm, g.dx[i_f]));
        dh = ad(dh, w_hat);
        if (he) ev = dv(1.0, ml(dyj, g.dx[i_f]));
        else o.wall(RU, j, ml(sm, w_hat));
    }
    {
        const double span = hs ? g.del_y[j - 1] : ml(0.5, dyj);
        const double w_hat = dv(1.0, ml(dyj, span));
        dh = ad(dh, w_hat);
        if (hs) sv = dv(sm, ml(span, ml(dyj, g.dy[j - 1])));
        else o.wall(BU, i_f - 1, ml(sm, w_hat));
    }
    {
        const double span = hn ? g.del_y[j] : ml(0.5, dyj);
        const double w_hat = dv(1.0, ml(dyj, span));
        dh = ad(dh, w_hat);
        if (hn) nv = dv(sm, ml(span, ml(dyj, g.dy[j + 1])));
        else o.wall(TU, i_f - 1, ml(sm, w_hat));
    }
    if (hs) o.put(g.u_id(i_f, j - 1), sv);
    if (hw) o.put(g.u_id(i_f - 1, j), wv);
    o.put(row, dv(ml(-sm, dh), dyj));
    if (he) o.put(g.u_id(i_f + 1, j), ev);
    if (hn) o.put(g.u_id(i_f, j + 1), nv);
}

// operators.hpp:148-194 (v rows)
__device__ void v_row(const DGrid& g, int j_f, int i, Row& o) {
    const int nx = g.nx, ny = g.ny;
    const int row = g.v_id(i, j_f);
    const double sm = g.del_y[j_f - 1], dxi = g.dx[i];
    double dh = 0.0, wv = 0, ev = 0, sv = 0, nv = 0;
    const bool hs = j_f - 1 >= 1, hn = j_f + 1 <= ny - 1, hw = i > 0, he = i < nx - 1;
    {
        const double w_hat = dv(1.0, ml(sm, g.dy[j_f - 1]));
        dh = ad(dh, w_hat);
        if (hs) sv = dv(1.0, ml(dxi, g.dy[j_f - 1]));
        else o.wall(BV, i, ml(sm, w_hat));
    }
    {
        const double w_hat = dv(1.0, ml(sm, g.dy[j_f]));
        dh = ad(dh, w_hat);
        if (hn) nv = dv(1.0, ml(dxi, g.dy[j_f]));
        else o.wall(TV, i, ml(sm, w_hat));
    }
    {
        const double span = hw ? g.del_x[i - 1] : ml(0.5, dxi);
        const double w_hat = dv(1.0, ml(dxi, span));
        dh = ad(dh, w_hat);
        if (hw) wv = dv(sm, ml(span, ml(dxi, g.dx[i - 1])));
        else o.wall(LV, j_f - 1, ml(sm, w_hat));
    }
    {
        const double span = he ? g.del_x[i] : ml(0.5, dxi);
        const double w_hat = dv(1.0, ml(dxi, span));
        dh = ad(dh, w_hat);
        if (he) ev = dv(sm, ml(span, ml(dxi, g.dx[i + 1])));
        else o.wall(RV, j_f - 1, ml(sm, w_hat));
    }
    if (hs) o.put(g.v_id(i, j_f - 1), sv);
    if (hw) o.put(g.v_id(i - 1, j_f), wv);
    o.put(row, dv(ml(-sm, dh), dxi));
    if (he) o.put(g.v_id(i + 1, j_f), ev);
    if (hn) o.put(g.v_id(i, j_f + 1), nv);
}

__device__ void any_row(const DGrid& g, long long r, Row& o) {
    const long long nu = g.n_u();
    if (r < nu) {
        const int j = (int)(r / (g.nx - 1)), i_f = (int)(r % (g.nx - 1)) + 1;
        u_row(g, j, i_f, o);
    } else {
        const long long k = r - nu;
        const int j_f = (int)(k / g.nx) + 1, i = (int)(k % g.nx);
        v_row(g, j_f, i, o);
    }
}

// pass 1: entries and wall couplings per row; pass 2 (orp set): fill
__global__ void k_diffusion(long long n_q, DGrid g, int* __restrict__ cnt, int* __restrict__ bcnt,
                            const int* __restrict__ orp, const int* __restrict__ obo, int* __restrict__ oci,
                            double* __restrict__ ov, int* __restrict__ bslot, int* __restrict__ bidx,
                            double* __restrict__ bcoef) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_q) return;
    Row o;
    any_row(g, r, o);
    if (!orp) {
        cnt[r] = o.n;
        bcnt[r] = o.nb;
        return;
    }
    const int p = orp[r];
    for (int k = 0; k < o.n; ++k) oci[p + k] = o.c[k], ov[p + k] = o.v[k];
    const int q = obo[r];
    for (int k = 0; k < o.nb; ++k) bslot[q + k] = o.bslot[k], bidx[q + k] = o.bidx[k], bcoef[q + k] = o.bcoef[k];
}

__global__ void k_metric(long long n_q, DGrid g, double* __restrict__ m) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_q) return;
    const long long nu = g.n_u();
    if (r < nu) {
        const int j = (int)(r / (g.nx - 1)), i_f = (int)(r % (g.nx - 1)) + 1;
        m[r] = dv(g.del_x[i_f - 1], g.dy[j]);
    } else {
        const long long k = r - nu;
        const int j_f = (int)(k / g.nx) + 1, i = (int)(k % g.nx);
        m[r] = dv(g.del_y[j_f - 1], g.dx[i]);
    }
}

__global__ void k_gradient(long long n_q, DGrid g, int* __restrict__ rp, int* __restrict__ ci, double* __restrict__ v) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r > n_q) return;
    rp[r] = (int)(2 * r);
    if (r == n_q) return;
    const long long nu = g.n_u();
    int c0, c1;
    if (r < nu) {
        const int j = (int)(r / (g.nx - 1)), i_f = (int)(r % (g.nx - 1)) + 1;
        c0 = (i_f - 1) + j * g.nx, c1 = i_f + j * g.nx;
    } else {
        const long long k = r - nu;
        const int j_f = (int)(k / g.nx) + 1, i = (int)(k % g.nx);
        c0 = i + (j_f - 1) * g.nx, c1 = i + j_f * g.nx;
    }
    ci[2 * r] = c0, v[2 * r] = -1.0;
    ci[2 * r + 1] = c1, v[2 * r + 1] = 1.0;
}

// rows with wall couplings, compacted (the stepper's grouped viscous boundary terms)
__global__ void k_wall_rows(long long n_q, const int* __restrict__ bflag, const int* __restrict__ bpos,
                            const int* __restrict__ obo, int* __restrict__ rows, int* __restrict__ off) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_q || !bflag[r]) return;
    rows[bpos[r]] = (int)r;
    off[bpos[r]] = obo[r];
}
__global__ void k_flag(long long n, const int* __restrict__ cnt, int* __restrict__ flag) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) flag[r] = cnt[r] > 0;
}
__global__ void k_wall_pos(int nb, const int* __restrict__ bslot, const int* __restrict__ bidx, const int* slot_off,
                           int* __restrict__ pos) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nb) pos[k] = slot_off[bslot[k]] + bidx[k];
}

}  // namespace

GridOps assemble_grid_ops(Ctx* c, int nx, int ny, const double* dx, const double* dy, const double* del_x,
                          const double* del_y, const int slot_off[8]) {
    require((long long)(nx - 1) * ny + (long long)nx * (ny - 1) < (1ll << 30), "grid: too many unknowns");
    const DGrid g{nx, ny, dx, dy, del_x, del_y};
    const long long n_q = (long long)(nx - 1) * ny + (long long)nx * (ny - 1);
    const int nq = (int)n_q;
    GridOps o;
    // M
    o.M.alloc(c, (size_t)n_q);
    k_metric<<<nblk(n_q), 256, 0, c->stream>>>(n_q, g, o.M.p);
    CK_LAUNCH(c);
    // G: exactly two entries per row
    require(2 * n_q < (1ll << 31), "gradient: result exceeds int32 nonzero indexing");
    o.G = mat_new(c, nq, nx * ny, (int)(2 * n_q));
    k_gradient<<<nblk(n_q + 1), 256, 0, c->stream>>>(n_q, g, o.G->rp.p, o.G->ci.p, o.G->v.p);
    CK_LAUNCH(c);
    // L + wall couplings
    DBuf<int> cnt(c, (size_t)n_q + 1), bcnt(c, (size_t)n_q + 1), bo(c, (size_t)n_q + 1);
    k_diffusion<<<nblk(n_q), 256, 0, c->stream>>>(n_q, g, cnt.p, bcnt.p, nullptr, nullptr, nullptr, nullptr, nullptr,
                                                  nullptr, nullptr);
    CK_LAUNCH(c);
    o.L = mat_new(c, nq, nq, 0);
    exclusive_scan_total(c, cnt.p, o.L->rp.p, nq);
    exclusive_scan_total(c, bcnt.p, bo.p, nq);
    int tot[2];
    d2h(c, tot, o.L->rp.p + nq, 1);
    d2h(c, tot + 1, bo.p + nq, 1);
    sync(c);
    o.L->nnz = tot[0];
    o.n_wall = tot[1];
    o.L->ci.alloc(c, (size_t)std::max(tot[0], 1));
    o.L->v.alloc(c, (size_t)std::max(tot[0], 1));
    DBuf<int> bslot(c, (size_t)std::max(tot[1], 1)), bidx(c, (size_t)std::max(tot[1], 1));
    o.wall_coeff.alloc(c, (size_t)std::max(tot[1], 1) + 1);
    k_diffusion<<<nblk(n_q), 256, 0, c->stream>>>(n_q, g, nullptr, nullptr, o.L->rp.p, bo.p, o.L->ci.p, o.L->v.p,
                                                  bslot.p, bidx.p, o.wall_coeff.p);
    CK_LAUNCH(c);
    // grouped by row in list order (the reference builds the list row by row, u block then v block,
    // so it is already sorted by row): rows with couplings, their offsets, and the boundary slot of each
    DBuf<int> flag(c, (size_t)n_q + 1), fpos(c, (size_t)n_q + 1);
    k_flag<<<nblk(n_q), 256, 0, c->stream>>>(n_q, bcnt.p, flag.p);
    CK_LAUNCH(c);
    exclusive_scan_total(c, flag.p, fpos.p, nq);
    o.n_wall_rows = d2h_scalar(c, fpos.p + nq);
    o.wall_rows.alloc(c, (size_t)o.n_wall_rows + 1);
    o.wall_off.alloc(c, (size_t)o.n_wall_rows + 1);
    k_wall_rows<<<nblk(n_q), 256, 0, c->stream>>>(n_q, flag.p, fpos.p, bo.p, o.wall_rows.p, o.wall_off.p);
    CK_LAUNCH(c);
    h2d(c, o.wall_off.p + o.n_wall_rows, &o.n_wall, 1);
    DBuf<int> so(c, 8);
    h2d(c, so.p, slot_off, 8);
    o.wall_pos.alloc(c, (size_t)std::max(o.n_wall, 1) + 1);
    if (o.n_wall) {
        k_wall_pos<<<nblk(o.n_wall), 256, 0, c->stream>>>(o.n_wall, bslot.p, bidx.p, so.p, o.wall_pos.p);
        CK_LAUNCH(c);
    }
    sync(c);
    return o;
}

}  // namespace ibmgpu
