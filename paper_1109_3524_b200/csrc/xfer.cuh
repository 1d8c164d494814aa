// xfer.cuh — level-0 grid transfers of the V-cycle applied through the stencil (SURVEY §8(a)
// A19-A21: sa_apply / v_cycle at amg.hpp:198-225, P and P^T from amg.hpp:153-183).
//
// The reference forms the smoothed prolongator explicitly, P = (I - omega D^-1 A) T on the core
// rows (T: the normalised aggregate indicator, amg.hpp:153-166) and the identity on the body
// tail, and its V-cycle streams P^T and P once each per cycle. On the level-0 operator (the
// 5-point pressure stencil Q^T B^N Q, stored as band planes — kern.cuh k_spmv_stencil) the same
// linear maps are applied without P:
//   restriction  (P^T r)_a  = t_a sum_{m in a} [ r_m - sum_{i core} A_im (wd_i r_i) ]     (core a)
//                (P^T r)_{n_agg+t} = r_{n_core+t}                                        (tail)
//   prolongation (P e)_k    = y_k - wd_k (A y)_k,  y = T e (y = 0 on the tail)           (core k)
//                (P e)_{n_core+t} = e_{n_agg+t}                                           (tail)
// with wd = omega/diag(A) and t_a = 1/sqrt(|a|). The column sum in the restriction reads A's band
// transposed (row m-S's +S slot is A_{m-S,m}), so no symmetry is assumed. Core rows' extras are
// tail columns (checked by xfer0_setup), where y = 0, so only the band enters.
//
// Four kernels replace the four SpMVs of level 0 (K1 A, K2 P^T, K3 P, K4 A). A CTA of the two
// stencil kernels owns a tile of 28 grid columns x 30 lines: lane l of every warp is grid column
// i0 - 2 + l (lanes 2..29 produce output), warp w takes frame lines w, w + 8, ...; the i+-1
// neighbours come by warp shuffles, the j+-1 neighbours through shared memory, and all of a
// thread's loads (band, wd, b, aggregates) are issued together before their first use.
//   k_xfer_down      r1 = b - A (wd b) on the tile + 1 line, then s = r1 - A^T(wd r1) on the
//                    tile; the first CTAs compute r1 on the tail rows (one warp per row)
//   k_xfer_restrict  b_1[a] = t_a sum_{m in a} s_m (members in row order), b_1[tail] = r1_tail,
//                    and the next level's pre-smoothed iterate (w d)_1 b_1
//   k_xfer_up        y = T e on the tile + 2 lines, x = wd b + y - wd (A y) on the tile + 1,
//                    then the post-smooth z = x + wd (b - A x) and the PCG's r.z partial; x of
//                    the cells the tail rows couple to is kept for
//   k_xfer_up_tail   z on the tail rows (one warp per row; its r.z partials follow k_xfer_up's)
// Per cycle that removes P^T and P (~107 B per fine row at S-4M) and the r / x round trips.
// Same operator, different rounding (the reference sums P's entries, rounded at setup): results
// agree with the explicit path to ~1e-15 relative per cycle; IBMGPU_XFER0=0 restores it.
#pragma once
#include "kern.cuh"

namespace ibmgpu {

constexpr int kXOut = 28;        // output columns per tile (lanes 2..29)
#ifndef IBMGPU_XFER_TJ
#define IBMGPU_XFER_TJ 22
#endif
constexpr int kXTJ = IBMGPU_XFER_TJ;  // output lines per tile
constexpr int kXL1 = kXTJ + 2;   // band lines (tile + 1): 4 per warp
constexpr int kXL2 = kXTJ + 4;   // x / y frame lines (tile + 2)
#ifndef IBMGPU_XFER_WARPS
#define IBMGPU_XFER_WARPS 8
#endif
#ifndef IBMGPU_XFER_MINB
#define IBMGPU_XFER_MINB 3
#endif
constexpr int kXWarps = IBMGPU_XFER_WARPS;  // warps per tile CTA
constexpr int kXThreads = 32 * kXWarps;
constexpr int kXK1 = kXL1 / kXWarps;  // band lines per warp
constexpr int kXK2 = (kXL2 + kXWarps - 1) / kXWarps;
constexpr int kXTailRows = 8;    // tail rows per CTA (one warp each)
constexpr unsigned kXTailCol = 128u;  // stencil mask bit 7 (hierarchy copy of A_0): a tail row's column
static_assert(kXL1 % kXWarps == 0, "band lines per warp");

struct XferPlan {
    StencilPlan A;  // level-0 band planes + extras (n rows)
    int n, n_core, S, NY, n_agg;
    int n_ti, tiles, tail_ctas;  // tiles: n_ti across a line x ceil(NY / kXTJ); tail CTAs come first
    double* xk;                  // x of the core cells flagged kXTailCol (k_xfer_up -> _up_tail)
    const double* wd;    // omega / diag, n
    const int* agg;      // aggregate per core row
    const double* tagg;  // 1/sqrt(|a|) per aggregate
    const int* mrp;      // members of aggregate a: mem[mrp[a] .. mrp[a+1]), ascending rows
    const int* mem;
};

// Row sum of a tail row (band slots in slot order, then the extras: the stencil kernel's
// order) by one warp: lane j forms the product of entry j of each 32-entry chunk, lane-ordered
// shuffle adds. fx(col) gives the operand. Result on every lane.
template <class FX>
__device__ __forceinline__ double xfer_warp_row(const XferPlan& X, int row, FX fx, int lane) {
    const unsigned m = __ldg(X.A.mask + row);
    const int S = X.A.S1;
    const int off[5] = {-S, -1, 0, 1, S};
    double s = 0.0;
    if (m & 31u) {  // band slots (rare on tail rows)
        const double p = (lane < 5 && (m & (1u << lane))) ? mul(__ldg(X.A.v + (size_t)lane * X.n + row),
                                                                 fx(row + off[lane < 5 ? lane : 0]))
                                                          : 0.0;
        for (int q = 0; q < 5; ++q)
            if (m & (1u << q)) s = addd(s, __shfl_sync(kFull, p, q));
    }
    if (m & 32u) {
        const int b = __ldg(X.A.erp + row), e = __ldg(X.A.erp + row + 1);
        for (int k0 = b; k0 < e; k0 += 32) {
            const int k = k0 + lane;
            const double p = k < e ? mul(__ldg(X.A.ev + k), fx(__ldg(X.A.eci + k))) : 0.0;
            const int cnt = min(32, e - k0);
            for (int j = 0; j < cnt; ++j) s = addd(s, __shfl_sync(kFull, p, j));
        }
    }
    return s;
}

// Tile t: first output line j0 and this lane's grid column.
__device__ __forceinline__ void xfer_tile(const XferPlan& X, int t, int& j0, int& ic) {
    j0 = (t / X.n_ti) * kXTJ;
    ic = (t % X.n_ti) * kXOut - 2 + (threadIdx.x & 31);
}
__device__ __forceinline__ double shup(double v) { return __shfl_up_sync(kFull, v, 1); }    // lane - 1
__device__ __forceinline__ double shdn(double v) { return __shfl_down_sync(kFull, v, 1); }  // lane + 1

// K_D: s = r1 - A^T(wd r1) on core rows, r1 = b - A (wd b); r1 of the tail rows into r1t.
static __global__ void __launch_bounds__(kXThreads, IBMGPU_XFER_MINB) k_xfer_down(XferPlan X, const double* b, double* s_out,
                                                                double* r1t, const int* done) {
    __shared__ double sx[kXL2][32];  // x = wd b, frame lines j0-2 ..
    __shared__ double sq4[kXL1][32];  // A_{m,+S} u_m (read by the line below)
    __shared__ double sq0[kXL1][32];  // A_{m,-S} u_m (read by the line above)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (blockIdx.x < X.tail_ctas) {  // tail rows, one warp each
        if (w >= kXTailRows) return;
        const int t = blockIdx.x * kXTailRows + w;
        pdl_wait();
        if (done && flag_set(done)) return;
        if (t >= X.n - X.n_core) return;
        const int row = X.n_core + t;
        const double acc = xfer_warp_row(X, row, [&](int j) { return mul(__ldg(X.wd + j), ld_weak(b + j)); }, lane);
        if (lane == 0) r1t[t] = subd(ld_weak(b + row), acc);
        return;
    }
    int j0, ic;
    xfer_tile(X, blockIdx.x - X.tail_ctas, j0, ic);
    const bool col = ic >= 0 && ic < X.S;
    // constant operands: band + wd of this thread's band cells, wd of its frame cells
    int r1c[kXK1], r2c[kXK2];
    double p[kXK1][5], w1[kXK1], w2[kXK2];
    unsigned m1[kXK1];
#pragma unroll
    for (int k = 0; k < kXK1; ++k) {
        const int j = j0 - 1 + w + kXWarps * k;
        r1c[k] = (col && j >= 0 && j < X.NY) ? j * X.S + ic : -1;
#pragma unroll
        for (int q = 0; q < 5; ++q) p[k][q] = r1c[k] >= 0 ? __ldg(X.A.v + (size_t)q * X.n + r1c[k]) : 0.0;
        m1[k] = r1c[k] >= 0 ? __ldg(X.A.mask + r1c[k]) : 0u;
        w1[k] = r1c[k] >= 0 ? __ldg(X.wd + r1c[k]) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kXK2; ++k) {
        const int f = w + kXWarps * k, j = j0 - 2 + f;
        r2c[k] = (f < kXL2 && col && j >= 0 && j < X.NY) ? j * X.S + ic : -1;
        w2[k] = r2c[k] >= 0 ? __ldg(X.wd + r2c[k]) : 0.0;
    }
    pdl_wait();
    double b1[kXK1], b2[kXK2];  // issued with the done-flag load (one round trip, not two)
#pragma unroll
    for (int k = 0; k < kXK2; ++k) b2[k] = r2c[k] >= 0 ? ld_weak(b + r2c[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < kXK1; ++k) b1[k] = r1c[k] >= 0 ? ld_weak(b + r1c[k]) : 0.0;
    if (done && flag_set(done)) return;
#pragma unroll
    for (int k = 0; k < kXK2; ++k)
        if (w + kXWarps * k < kXL2) sx[w + kXWarps * k][lane] = mul(w2[k], b2[k]);
    __syncthreads();
    // r1 = b - A x on the band lines (column order -S, -1, 0, +1, +S, then tail-column extras)
    double r1[kXK1], c1[kXK1], c2[kXK1], c3[kXK1];
#pragma unroll
    for (int k = 0; k < kXK1; ++k) {
        const int f = w + kXWarps * k;  // band line f = frame line f + 1
        const double xm = sx[f + 1][lane];
        const double xl = shup(xm), xr = shdn(xm);
        double a = 0.0;
        a = addd(a, mul(p[k][0], sx[f][lane]));
        a = addd(a, mul(p[k][1], xl));
        a = addd(a, mul(p[k][2], xm));
        a = addd(a, mul(p[k][3], xr));
        a = addd(a, mul(p[k][4], sx[f + 2][lane]));
        if (m1[k] & 32u) {
            const int r = r1c[k], e = __ldg(X.A.erp + r + 1);
            for (int q = __ldg(X.A.erp + r); q < e; ++q) {
                const int cc = __ldg(X.A.eci + q);
                a = addd(a, mul(__ldg(X.A.ev + q), mul(__ldg(X.wd + cc), ld_weak(b + cc))));
            }
        }
        r1[k] = r1c[k] >= 0 ? subd(b1[k], a) : 0.0;
        const double u = mul(w1[k], r1[k]);
        c1[k] = mul(p[k][1], u);
        c2[k] = mul(p[k][2], u);
        c3[k] = mul(p[k][3], u);
        sq4[f][lane] = mul(p[k][4], u);
        sq0[f][lane] = mul(p[k][0], u);
    }
    __syncthreads();
    // s_m = r1_m - [A_{m-S,m} u + A_{m-1,m} u + A_mm u + A_{m+1,m} u + A_{m+S,m} u]
#pragma unroll
    for (int k = 0; k < kXK1; ++k) {
        const int f = w + kXWarps * k;
        const double cl = shup(c3[k]), cr = shdn(c1[k]);
        if (f >= 1 && f <= kXTJ && r1c[k] >= 0 && lane >= 2 && lane < 2 + kXOut) {
            double c = 0.0;
            c = addd(c, sq4[f - 1][lane]);
            c = addd(c, cl);
            c = addd(c, c2[k]);
            c = addd(c, cr);
            c = addd(c, sq0[f + 1][lane]);
            s_out[r1c[k]] = subd(r1[k], c);
        }
    }
    pdl_release();
}

// K_T: y[a] = t_a sum_{m in a} s_m (a < n_agg), y[n_agg + t] = r1t[t]; xj = wd1 y when the next
// level exists (EpiStoreJacobi's contract), else only y (the coarse right-hand side). Members are
// fetched eight at a time (indices, then gathers, then the in-order adds).
static __global__ void __launch_bounds__(kBlock) k_xfer_restrict(XferPlan X, int n_out, const double* s,
                                                                 const double* r1t, double* y, const double* wd1,
                                                                 double* xj, const int* done) {
    pdl_release_early(8);
    const int a = blockIdx.x * kBlock + threadIdx.x;
    const bool live = a < n_out;
    int b = 0, e = 0;
    double t = 0.0, w = 0.0;
    int mi[8];
    if (live && a < X.n_agg) {
        b = __ldg(X.mrp + a);
        e = __ldg(X.mrp + a + 1);
        t = __ldg(X.tagg + a);
#pragma unroll
        for (int q = 0; q < 8; ++q) mi[q] = b + q < e ? __ldg(X.mem + b + q) : -1;
    }
    if (live && xj) w = __ldg(wd1 + a);
    pdl_wait();
    if (done && flag_set(done)) return;
    if (live) {
        double v;
        if (a < X.n_agg) {
            double acc = 0.0;
            for (int k0 = b;;) {
                double sv[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    IBM_DCHECK(mi[q] < X.n_core);
                    sv[q] = mi[q] >= 0 ? ld_weak(s + mi[q]) : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (mi[q] >= 0) acc = addd(acc, sv[q]);
                k0 += 8;
                if (k0 >= e) break;
#pragma unroll
                for (int q = 0; q < 8; ++q) mi[q] = k0 + q < e ? __ldg(X.mem + k0 + q) : -1;
            }
            v = mul(t, acc);
        } else {
            v = ld_weak(r1t + (a - X.n_agg));
        }
        y[a] = v;
        if (xj) xj[a] = mul(w, v);
    }
    pdl_release_late(8);
}

// Post-smooth sinks of k_xfer_up: the plain V-cycle (sa_apply) or the PCG's fused r.z.
struct XSinkPlain {
    static constexpr int NR = 0;
    double* z;
    const int* done;
    __device__ bool skip() const { return done && flag_set(done); }
    __device__ void row(int i, double, double zi, double*) const { z[i] = zi; }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};
template <class Fin>
struct XSinkDot {
    static constexpr int NR = 1;
    double* z;
    const int* done;
    RedSlot rs;
    Fin f;
    __device__ bool skip() const { return done && flag_set(done); }
    __device__ void row(int i, double bi, double zi, double* acc) const {
        z[i] = zi;
        acc[0] += bi * zi;
    }
    __device__ RedSlot slot() const { return rs; }
    __device__ void fin(double* tot) const { f(tot); }
};

// K_U: z = x + wd (b - A x), x = wd b + P e, with P e applied through the stencil (see top).
template <class Sink>
__global__ void __launch_bounds__(kXThreads, IBMGPU_XFER_MINB) k_xfer_up(XferPlan X, const double* b, const double* e, Sink sink) {
    __shared__ double sy[kXL2][32];  // y = T e, frame lines j0-2 ..
    __shared__ double sx[kXL1][32];  // x, band lines j0-1 ..
    constexpr int NR = Sink::NR;
    double acc[NR > 0 ? NR : 1];
#pragma unroll
    for (int q = 0; q < (NR > 0 ? NR : 1); ++q) acc[q] = 0.0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int j0, ic;
    xfer_tile(X, blockIdx.x, j0, ic);
    const bool col = ic >= 0 && ic < X.S;
    int r1c[kXK1], a2[kXK2];
    double p[kXK1][5], w1[kXK1], t2[kXK2];
    unsigned m1[kXK1];
#pragma unroll
    for (int k = 0; k < kXK2; ++k) {
        const int f = w + kXWarps * k, j = j0 - 2 + f;
        a2[k] = (f < kXL2 && col && j >= 0 && j < X.NY) ? __ldg(X.agg + j * X.S + ic) : -1;
        IBM_DCHECK(a2[k] < X.n_agg);
    }
#pragma unroll
    for (int k = 0; k < kXK1; ++k) {
        const int j = j0 - 1 + w + kXWarps * k;
        r1c[k] = (col && j >= 0 && j < X.NY) ? j * X.S + ic : -1;
#pragma unroll
        for (int q = 0; q < 5; ++q) p[k][q] = r1c[k] >= 0 ? __ldg(X.A.v + (size_t)q * X.n + r1c[k]) : 0.0;
        m1[k] = r1c[k] >= 0 ? __ldg(X.A.mask + r1c[k]) : 0u;
        w1[k] = r1c[k] >= 0 ? __ldg(X.wd + r1c[k]) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kXK2; ++k) t2[k] = a2[k] >= 0 ? __ldg(X.tagg + a2[k]) : 0.0;
    pdl_wait();
    double e2[kXK2], b1[kXK1];  // issued before the done flag is tested
#pragma unroll
    for (int k = 0; k < kXK2; ++k) e2[k] = a2[k] >= 0 ? ld_weak(e + a2[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < kXK1; ++k) b1[k] = r1c[k] >= 0 ? ld_weak(b + r1c[k]) : 0.0;
    const bool skip = sink.skip();
#pragma unroll
    for (int k = 0; k < kXK2; ++k)
        if (w + kXWarps * k < kXL2) sy[w + kXWarps * k][lane] = mul(t2[k], e2[k]);
    __syncthreads();
    // x = wd b + (y - wd (A y)) on the band lines (core extras are tail columns: y = 0 there)
    double x[kXK1];
#pragma unroll
    for (int k = 0; k < kXK1; ++k) {
        const int f = w + kXWarps * k;
        const double ym = sy[f + 1][lane];
        const double yl = shup(ym), yr = shdn(ym);
        double a = 0.0;
        a = addd(a, mul(p[k][0], sy[f][lane]));
        a = addd(a, mul(p[k][1], yl));
        a = addd(a, mul(p[k][2], ym));
        a = addd(a, mul(p[k][3], yr));
        a = addd(a, mul(p[k][4], sy[f + 2][lane]));
        x[k] = r1c[k] >= 0 ? addd(mul(w1[k], b1[k]), subd(ym, mul(w1[k], a))) : 0.0;
        sx[f][lane] = x[k];
    }
    __syncthreads();
    // z = x + wd (b - A x) on the tile
#pragma unroll
    for (int k = 0; k < kXK1; ++k) {
        const int f = w + kXWarps * k;
        const double xl = shup(x[k]), xr = shdn(x[k]);
        const int r = r1c[k];
        if (skip || f < 1 || f > kXTJ || r < 0 || lane < 2 || lane >= 2 + kXOut) continue;
        double c = 0.0;
        c = addd(c, mul(p[k][0], sx[f - 1][lane]));
        c = addd(c, mul(p[k][1], xl));
        c = addd(c, mul(p[k][2], x[k]));
        c = addd(c, mul(p[k][3], xr));
        c = addd(c, mul(p[k][4], sx[f + 1][lane]));
        if (m1[k] & 32u) {  // tail columns: x = wd b + e_tail
            const int q1 = __ldg(X.A.erp + r + 1);
            for (int q = __ldg(X.A.erp + r); q < q1; ++q) {
                const int cc = __ldg(X.A.eci + q);
                const double xc =
                    addd(mul(__ldg(X.wd + cc), ld_weak(b + cc)), ld_weak(e + X.n_agg + (cc - X.n_core)));
                c = addd(c, mul(__ldg(X.A.ev + q), xc));
            }
        }
        IBM_DCHECK(r < X.n_core);
        if (m1[k] & kXTailCol) X.xk[r] = x[k];
        sink.row(r, b1[k], addd(x[k], mul(w1[k], subd(b1[k], c))), acc);
    }
    pdl_release();
    if (skip) return;
    if constexpr (NR > 0) block_partial<NR>(acc, sink.slot());
}

// z on the tail rows: x_t = wd b + e_tail, core columns' x from k_xfer_up (X.xk). Partials go to
// slots `slot0 + blockIdx.x` (after k_xfer_up's).
template <class Sink>
__global__ void __launch_bounds__(kBlock) k_xfer_up_tail(XferPlan X, const double* b, const double* e, Sink sink,
                                                         int slot0) {
    pdl_release_early(8);
    constexpr int NR = Sink::NR;
    double acc[NR > 0 ? NR : 1];
#pragma unroll
    for (int q = 0; q < (NR > 0 ? NR : 1); ++q) acc[q] = 0.0;
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x * kXTailRows + (threadIdx.x >> 5);
    pdl_wait();
    if (sink.skip()) return;
    if (t < X.n - X.n_core) {
        const int row = X.n_core + t;
        const double ax = xfer_warp_row(
            X, row,
            [&](int k) {
                return k < X.n_core ? ld_weak(X.xk + k)
                                    : addd(mul(__ldg(X.wd + k), ld_weak(b + k)), ld_weak(e + X.n_agg + (k - X.n_core)));
            },
            lane);
        if (lane == 0) {
            const double bi = ld_weak(b + row), wdi = __ldg(X.wd + row);
            const double xi = addd(mul(wdi, bi), ld_weak(e + X.n_agg + t));
            sink.row(row, bi, addd(xi, mul(wdi, subd(bi, ax))), acc);
        }
    }
    pdl_release_late(8);
    if constexpr (NR > 0) {
        RedSlot rs = sink.slot();
        rs.partials += (size_t)slot0 * NR;
        block_partial<NR>(acc, rs);
    }
}

}  // namespace ibmgpu
