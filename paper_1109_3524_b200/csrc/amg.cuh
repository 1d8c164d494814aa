// amg.cuh — smoothed-aggregation hierarchy on the device and the fused V(1,1) cycle.
//
// Reference: amg.hpp:33-52 (SaLevel/SaHierarchy), :198-225 (v_cycle). Per level l (n_l rows):
//   K1  x = (w d) .* b ; r = b - A x           one SpMV over A_l, x gathered as (w d_j) b_j
//   K2  b_{l+1} = P^T r                         SpMV over the explicit P^T (amg.hpp:183)
//   ... recurse; coarsest: x_c = A_c^{-1} b_c   dense symmetric inverse GEMV (dense.hpp)
//   K3  x += P x_{l+1}                          SpMV over P, in-place add
//   K4  out = x + (w d) .* (b - A x)            SpMV over A_l; at level 0 the PCG's r.z partial
//                                               is reduced in the same kernel
// The products (w d) use the stored omega*inv_diag, which rounds exactly like the reference's
// L.omega * L.inv_diag[i] (amg.hpp:210, :224); SELL levels therefore reproduce v_cycle bit for bit
// up to the coarse solve.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <memory>
#include <vector>

#include "coarse.cuh"
#include "internal.cuh"
#include "kern.cuh"
#include "xfer.cuh"

struct ibmgpu_hier;

namespace ibmgpu {

struct Level {
    Mat* A = nullptr;  // owned
    Mat* P = nullptr;
    Mat* Pt = nullptr;
    double omega = 0.0;
    int n_core = 0, n_agg = 0;
    DBuf<double> invd, wd;  // 1/diag(A), omega/diag(A)
    DBuf<int> agg;          // aggregate id per core row
    DBuf<double> b, x, r, xo;  // V-cycle work vectors (b unused at level 0)
    DBuf<double> xj;           // levels >= 1: (omega d) .* b, written by the restriction above
    ~Level() {
        delete A;
        delete P;
        delete Pt;
    }
};

// Level-0 transfers through the stencil (xfer.cuh / xfer.cu); on = false: the explicit P / P^T
struct Xfer0 {
    bool on = false;
    bool built = false;  // plan and buffers exist (on may be switched off and back)
    int S = 0, NY = 0, n_ti = 0, tiles = 0, tail_ctas = 0;
    DBuf<double> tagg, r1t;
    DBuf<int> mrp, mem;
};

}  // namespace ibmgpu

struct ibmgpu_hier {
    std::vector<std::unique_ptr<ibmgpu::Level>> levels;
    ibmgpu::Mat* coarse_A = nullptr;
    int n_c = 0;
    ibmgpu::DBuf<double> coarse_inv;  // n_c x n_c row-major, symmetric
    ibmgpu::DBuf<double> coarse_tiles, prow, pcol;  // packed lower-triangle tiles + SYMV partials
    ibmgpu::DBuf<double> cb, cx;      // coarse rhs / solution (n_dense)
    // fold.cu: the last n_fold levels folded into one dense operator of dimension n_dense (the
    // coarse solve then applies it; n_fold = 0: n_dense = n_c, the coarse inverse itself)
    int n_fold = 0, n_dense = 0;
    ibmgpu::DBuf<double> dense;       // n_dense x n_dense row-major (freed once packed)
    int active_levels() const { return (int)levels.size() - n_fold; }
    // fused coarse sub-cycle (coarse.cuh): levels [fuse_from, L) + dense solve in one launch
    int fuse_from = 0;
    int n_phases = 0, coarse_grid = 0;
    ibmgpu::DBuf<ibmgpu::Phase> phases;
    ibmgpu::DBuf<unsigned> bar;       // {count, generation}
    ibmgpu::Xfer0 x0;
    bool stalled = false;
    long long id = 0;
    int built_at_step = -1;
    ~ibmgpu_hier() { delete coarse_A; }
};

namespace ibmgpu {
using Hier = ibmgpu_hier;

// A hierarchy built on a helper stream (the stepper's operator pipeline) handed to the main
// stream: every buffer is then freed in main-stream order (see mat_rehome).
inline void hier_rehome(Hier* h, cudaStream_t s) {
    auto set = [s](auto& b) {
        if (b.p) b.s = s;
    };
    for (auto& lv : h->levels) {
        for (Mat* m : {lv->A, lv->P, lv->Pt})
            if (m) mat_rehome(m, s);
        set(lv->invd), set(lv->wd), set(lv->agg), set(lv->b), set(lv->x), set(lv->r), set(lv->xo), set(lv->xj);
    }
    if (h->coarse_A) mat_rehome(h->coarse_A, s);
    set(h->coarse_inv), set(h->coarse_tiles), set(h->prow), set(h->pcol), set(h->cb), set(h->cx), set(h->dense);
    set(h->phases), set(h->bar);
    set(h->x0.tagg), set(h->x0.r1t), set(h->x0.mrp), set(h->x0.mem);
}

// Aggregates of the previous build, per level, keyed by the strength graph they came from.
// aggregate() (amg.hpp:79-107) is a function of the strength graph alone, so when a rebuild's
// graph is identical to the cached one the cached aggregates ARE the result (moving bodies: the
// level-0 graph lives on the pressure block, which body motion never changes).
struct AggCache {
    struct Lv {
        int n_core = -1, nnz = -1, n_agg = 0;
        DBuf<int> rp, ci, agg;
    };
    std::vector<Lv> lv;
    long long hits = 0, misses = 0;
    void rehome(cudaStream_t s) {  // buffers freed in the order of the stream that uses them next
        for (auto& l : lv)
            for (DBuf<int>* b : {&l.rp, &l.ci, &l.agg})
                if (b->p) b->s = s;
    }
};

// xfer.cu
bool xfer0_enabled();
void xfer0_setup(Ctx* c, Hier* h);
inline XferPlan xfer_plan(const Hier* h) {
    const Level& lv = *h->levels[0];
    const Mat* A = lv.A;
    return XferPlan{StencilPlan{A->st_v.p, A->st_mask.p, A->st_erp.p, A->st_eci.p, A->st_ev.p, A->st_S1, A->st_S2},
                    A->rows, lv.n_core, h->x0.S, h->x0.NY, lv.n_agg, h->x0.n_ti, h->x0.tiles, h->x0.tail_ctas,
                    lv.x.p, lv.wd.p, lv.agg.p, h->x0.tagg.p, h->x0.mrp.p, h->x0.mem.p};
}

// amg_setup.cu
Hier* sa_build(Ctx* c, const Mat* A, const ibm_sa_options& o, AggCache* cache = nullptr);
int aggregate_device(Ctx* c, const Mat* A, double theta, int n_core, DBuf<int>& agg,
                     AggCache::Lv* cache = nullptr, bool* hit = nullptr, int grid_S = 0);
// dense.cu
void dense_spd_inverse(Ctx* c, const Mat* Ac, double* inv);  // factor (dense.hpp:20-40) + inverse
void launch_dense_gemv(Ctx* c, int n, const double* Ainv, const double* x, double* y, const int* done,
                       cudaStream_t s);
void pack_symmetric_tiles(Ctx* c, int n, const double* full, double* tiles);
constexpr int kSymvTile = 64;  // packed SYMV tile edge (dense.cu)
// fold.cu
void fold_tail(Ctx* c, Hier* h, int tile);
size_t packed_tiles_doubles(int n);
size_t packed_partials_doubles(int n);
void launch_symv_packed(Ctx* c, int n, const double* tiles, const double* x, double* y, double* prow, double* pcol,
                        const int* done, cudaStream_t s);

// coarsest level: y = A_c^{-1} x from the packed symmetric inverse (each element read once)
inline void coarse_solve(Ctx* c, Hier* h, const double* x, double* y, const int* done, cudaStream_t s) {
    launch_symv_packed(c, h->n_dense, h->coarse_tiles.p, x, y, h->prow.p, h->pcol.p, done, s);
}

// ---------------------------------------------------------------- V-cycle epilogues
struct EpiJacobiResidual {  // K1: x_i = wd_i b_i ; r_i = b_i - s
    static constexpr int NR = 0;
    const double* wd;
    const double* b;
    double* x;
    double* r;
    const int* done;
    __device__ bool skip() const { return done && flag_set(done); }
    __device__ void touch(int i) const {
        pf(wd + i);
        pf(b + i);
    }
    __device__ void row(int i, double s, double*) const {
        const double bi = b[i];
        x[i] = mul(wd[i], bi);
        r[i] = subd(bi, s);
    }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

struct EpiStoreSkip {  // K2: b_{l+1} = s
    static constexpr int NR = 0;
    double* y;
    const int* done;
    __device__ bool skip() const { return done && flag_set(done); }
    __device__ void row(int i, double s, double*) const { y[i] = s; }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

struct EpiStoreJacobi {  // K2 into level l+1: b_i = s and the pre-smoothed iterate xj_i = (w d)_i b_i
    static constexpr int NR = 0;
    double* y;
    const double* wd;
    double* xj;
    const int* done;
    __device__ bool skip() const { return done && flag_set(done); }
    __device__ void touch(int i) const { pf(wd + i); }
    __device__ void row(int i, double s, double*) const {
        y[i] = s;
        xj[i] = mul(wd[i], s);
    }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

struct EpiAddInPlace {  // K3: x_i += s
    static constexpr int NR = 0;
    double* x;
    const int* done;
    __device__ bool skip() const { return done && flag_set(done); }
    __device__ void touch(int i) const { pf(x + i); }
    __device__ void row(int i, double s, double*) const { x[i] = addd(x[i], s); }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

struct EpiPostSmooth {  // K4: out_i = x_i + wd_i (b_i - s)
    static constexpr int NR = 0;
    const double* wd;
    const double* b;
    const double* x;
    double* out;
    const int* done;
    __device__ bool skip() const { return done && flag_set(done); }
    __device__ void touch(int i) const {
        pf(wd + i);
        pf(b + i);
    }
    __device__ void row(int i, double s, double*) const { out[i] = addd(x[i], mul(wd[i], subd(b[i], s))); }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

// K4 at level 0 with the PCG's r.z reduction fused: Fin receives tot[0] = sum r_i z_i.
template <class Fin>
struct EpiPostSmoothDot {
    static constexpr int NR = 1;
    const double* wd;
    const double* b;  // == PCG r
    const double* x;
    double* out;      // == PCG z
    const int* done;
    RedSlot rs;
    Fin f;
    __device__ bool skip() const { return done && flag_set(done); }
    __device__ void touch(int i) const {
        pf(wd + i);
        pf(b + i);
    }
    __device__ void row(int i, double s, double* acc) const {
        const double bi = b[i];
        const double z = addd(x[i], mul(wd[i], subd(bi, s)));
        out[i] = z;
        acc[0] += bi * z;
    }
    __device__ RedSlot slot() const { return rs; }
    __device__ void fin(double* tot) const { f(tot); }
};

// One V(1,1) cycle: z = M^{-1} r. `lastfin` customises the level-0 post-smooth epilogue
// (PCG fusion); `done` (nullable) lets every kernel early-exit once a solve has finished.
template <class LastEpi>
inline void vcycle_launch(Ctx* c, Hier* h, const double* r_in, double* z_out, const int* done, LastEpi last,
                          cudaStream_t s) {
    const int L = h->active_levels();
    if (L == 0) {
        coarse_solve(c, h, r_in, z_out, done, s);
        return;
    }
    int F = h->n_phases ? h->fuse_from : L;  // levels >= F run inside the fused kernel
    // IBMGPU_DEBUG_VDEPTH=k (timing experiments only; results are wrong): run levels < k and no
    // coarse solve unless k > L, to measure each level's in-graph cost by difference
    static const int vdepth = std::getenv("IBMGPU_DEBUG_VDEPTH") ? std::atoi(std::getenv("IBMGPU_DEBUG_VDEPTH")) : 0;
    const bool truncated = vdepth > 0 && vdepth <= L;
    if (truncated) F = std::min(F, vdepth);
    for (int l = 0; l < F; ++l) {
        Level& lv = *h->levels[l];
        const double* b = l == 0 ? r_in : lv.b.p;
        if (l == 0 && h->x0.on) {  // stencil transfers (xfer.cuh): s into lv.r, then b_1 = P^T r1
            const XferPlan X = xfer_plan(h);
            launch_k(c, k_xfer_down, h->x0.tail_ctas + h->x0.tiles, kXThreads, s, X, b, lv.r.p, h->x0.r1t.p, done);
            const int n1 = l + 1 < L ? h->levels[1]->A->rows : h->n_dense;
            const int g = (n1 + kBlock - 1) / kBlock;
            if (l + 1 < L) {
                Level& nx = *h->levels[1];
                launch_k(c, k_xfer_restrict, g, kBlock, s, X, n1, (const double*)lv.r.p, (const double*)h->x0.r1t.p,
                         nx.b.p, (const double*)nx.wd.p, nx.xj.p, done);
            } else {
                launch_k(c, k_xfer_restrict, g, kBlock, s, X, n1, (const double*)lv.r.p, (const double*)h->x0.r1t.p,
                         h->cb.p, (const double*)nullptr, (double*)nullptr, done);
            }
            continue;
        }
        // level 0 forms x_j = (w d)_j r_j inside the gather; deeper levels gather the iterate the
        // restriction above already wrote (one gather per entry instead of two)
        if (l == 0)
            launch_spmv(c, lv.A, XJacobi{lv.wd.p, b}, EpiJacobiResidual{lv.wd.p, b, lv.x.p, lv.r.p, done}, s);
        else
            launch_spmv(c, lv.A, XPlain{lv.xj.p}, EpiJacobiResidual{lv.wd.p, b, lv.x.p, lv.r.p, done}, s);
        if (l + 1 < L) {
            Level& nx = *h->levels[l + 1];
            launch_spmv(c, lv.Pt, XPlain{lv.r.p}, EpiStoreJacobi{nx.b.p, nx.wd.p, nx.xj.p, done}, s);
        } else {
            launch_spmv(c, lv.Pt, XPlain{lv.r.p}, EpiStoreSkip{h->cb.p, done}, s);
        }
    }
    if (truncated) {
    } else if (F < L) {
        k_coarse_cycle<<<h->coarse_grid, kBlock, 0, s>>>(CoarsePlan{h->phases.p, h->n_phases, h->bar.p, h->bar.p + 1},
                                                         done);
        CK_LAUNCH(c);
    } else {
        coarse_solve(c, h, h->cb.p, h->cx.p, done, s);
    }
    for (int l = F - 1; l >= 0; --l) {
        Level& lv = *h->levels[l];
        const double* b = l == 0 ? r_in : lv.b.p;
        const double* ec = l + 1 < L ? h->levels[l + 1]->xo.p : h->cx.p;
        if (l == 0 && h->x0.on) {
            last.xfer(h, b, ec, z_out);
            continue;
        }
        launch_spmv(c, lv.P, XPlain{ec}, EpiAddInPlace{lv.x.p, done}, s);
        if (l > 0) {
            launch_spmv(c, lv.A, XPlain{lv.x.p}, EpiPostSmooth{lv.wd.p, b, lv.x.p, lv.xo.p, done}, s);
        } else {
            last(lv, b, z_out);
        }
    }
}

// Plain level-0 finish (sa_apply without a fused reduction).
struct LastPlain {
    Ctx* c;
    const int* done;
    cudaStream_t s;
    void operator()(Level& lv, const double* b, double* z) const {
        launch_spmv(c, lv.A, XPlain{lv.x.p}, EpiPostSmooth{lv.wd.p, b, lv.x.p, z, done}, s);
    }
    void xfer(Hier* h, const double* b, const double* e, double* z) const {
        const XSinkPlain sink{z, done};
        launch_k(c, k_xfer_up<XSinkPlain>, h->x0.tiles, kXThreads, s, xfer_plan(h), b, e, sink);
        if (h->x0.tail_ctas)
            launch_k(c, k_xfer_up_tail<XSinkPlain>, h->x0.tail_ctas, kBlock, s, xfer_plan(h), b, e, sink, h->x0.tiles);
    }
};

// kernels launched by one V-cycle (for launch accounting)
inline int vcycle_kernels(const Hier* h) {
    if (h->levels.empty()) return 1;
    const int F = h->n_phases ? h->fuse_from : h->active_levels();
    return 4 * F + 2 - (h->x0.on && !h->x0.tail_ctas ? 1 : 0);  // + the two SYMV kernels
}

}  // namespace ibmgpu
