// pcg.cu — preconditioned CG (krylov.hpp:70-136) as one CUDA-graph launch per solve.
//
// Every scalar of the recurrence (alpha, beta, r.z, p.Ap, ||r||/||b||, the iteration counter,
// the status) lives in device memory and is produced by the last block of the kernel that
// reduces it (kern.cuh grid_sum_last), so the host never sits inside the iteration. The loop is
// a graph conditional WHILE node whose handle is cleared by the kernel that detects convergence,
// breakdown or the iteration cap. Per iteration:
//   B1  Ap = A p                   + p.Ap            -> alpha (or breakdown)
//   B2  x += alpha p, r -= alpha Ap + r.r (+ r.z)     -> rel, converged?  (diag/identity: beta)
//   B3  z = V-cycle(r)             + r.z fused in the last V-cycle kernel -> beta   (SA only)
//   B4  p = z + beta p
// Semantics follow krylov.hpp exactly: b = 0 returns x = 0; convergence is tested on the
// recursive residual before preconditioning; pAp <= 0 is breakdown with iterations = it-1;
// iterations counts the SpMVs after the initial residual.
#include <map>
#include <mutex>
#include <vector>
#include <memory>
#include <tuple>

#include "amg.cuh"
#include "internal.cuh"
#include "kern.cuh"
#include "pcg.cuh"

namespace ibmgpu {

namespace {

// ---------------------------------------------------------------- epilogues / bodies
struct EpiInitResidual {  // r_i = b_i - (A x)_i ; reduce b.b and r.r
    static constexpr int NR = 2;
    const double* b;
    double* r;
    RedSlot rs;
    PcgState* st;
    __device__ bool skip() const { return false; }
    __device__ void row(int i, double s, double* acc) const {
        const double bi = b[i];
        const double ri = subd(bi, s);
        r[i] = ri;
        acc[0] += bi * bi;
        acc[1] += ri * ri;
    }
    __device__ RedSlot slot() const { return rs; }
    __device__ void fin(double* tot) const {
        PcgState& S = *st;
        S.it = 1;
        S.bnorm = __dsqrt_rn(tot[0]);
        if (S.bnorm == 0.0) {  // krylov.hpp:85-89
            S.status = 0;
            S.iterations = 0;
            S.rel = 0.0;
            S.done = 1;
            S.zero_x = 1;
            if (S.use_cond) cudaGraphSetConditional(S.cond, 0);
            return;
        }
        S.rel = __ddiv_rn(__dsqrt_rn(tot[1]), S.bnorm);
        if (S.hist) S.hist[0] = S.rel;
        S.hist_len = 1;
        if (S.rel <= S.rel_tol) {  // krylov.hpp:97-100
            S.status = 0;
            S.iterations = 0;
            S.done = 1;
            if (S.use_cond) cudaGraphSetConditional(S.cond, 0);
        }
    }
};

struct BodyZeroX {
    static constexpr int NR = 0;
    double* x;
    const PcgState* st;
    __device__ bool skip() const { return !st->zero_x; }
    __device__ void row(int i, double*) const { x[i] = 0.0; }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

// initial z = M r, p = z, rz = r.z for identity / diagonal preconditioners
struct BodyInitZ {
    static constexpr int NR = 1;
    const double* r;
    const double* invd;  // null: identity
    double* z;
    double* p;
    RedSlot rs;
    PcgState* st;
    __device__ bool skip() const { return flag_set(&st->done); }
    __device__ void row(int i, double* acc) const {
        const double ri = r[i];
        const double zi = invd ? mul(ri, invd[i]) : ri;
        z[i] = zi;
        p[i] = zi;
        acc[0] += ri * zi;
    }
    __device__ RedSlot slot() const { return rs; }
    __device__ void fin(double* tot) const { st->rz = tot[0]; }
};

struct BodyCopy {  // p = z (after the initial V-cycle)
    static constexpr int NR = 0;
    const double* z;
    double* p;
    const PcgState* st;
    __device__ bool skip() const { return flag_set(&st->done); }
    __device__ void row(int i, double*) const { p[i] = z[i]; }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

struct FinInitRz {  // initial V-cycle's r.z
    PcgState* st;
    __device__ void operator()(double* tot) const { st->rz = tot[0]; }
};

struct EpiSpmvPAp {  // B1
    static constexpr int NR = 1;
    const double* p;
    double* Ap;
    RedSlot rs;
    PcgState* st;
    __device__ bool skip() const { return flag_set(&st->done); }
    __device__ void touch(int i) const { pf(p + i); }
    __device__ void row(int i, double s, double* acc) const {
        Ap[i] = s;
        acc[0] += p[i] * s;
    }
    __device__ RedSlot slot() const { return rs; }
    __device__ void fin(double* tot) const {
        PcgState& S = *st;
        S.pAp = tot[0];
        if (!(S.pAp > 0.0)) {  // krylov.hpp:109-114
            S.status = 2;
            S.iterations = S.it - 1;
            S.done = 1;
            if (S.use_cond) cudaGraphSetConditional(S.cond, 0);
            return;
        }
        S.alpha = __ddiv_rn(S.rz, S.pAp);
    }
};

__device__ __forceinline__ void finish_iteration(PcgState& S) {
    // end of iteration `it` (krylov.hpp:126-131 + loop bound)
    if (S.it >= S.max_iters) {
        S.status = 1;
        S.iterations = S.max_iters;
        S.done = 1;
        if (S.use_cond) cudaGraphSetConditional(S.cond, 0);
        return;
    }
    ++S.it;
}

struct BodyUpdate {  // B2
    static constexpr int NR = 2;
    double* x;
    double* r;
    const double* p;
    const double* Ap;
    const double* invd;  // diag preconditioner (null otherwise)
    double* z;           // written for identity/diag (z = M r)
    int kind;
    RedSlot rs;
    PcgState* st;
    __device__ bool skip() const { return flag_set(&st->done); }
    __device__ void row(int i, double* acc) const {
        const double a = st->alpha;
        x[i] = addd(x[i], mul(a, p[i]));           // axpy(alpha, p, x)
        const double ri = addd(r[i], mul(-a, Ap[i]));  // axpy(-alpha, Ap, r)
        r[i] = ri;
        acc[0] += ri * ri;
        if (kind != IBMGPU_PC_SA) {
            const double zi = kind == IBMGPU_PC_DIAGONAL ? mul(ri, invd[i]) : ri;
            z[i] = zi;
            acc[1] += ri * zi;
        }
    }
    __device__ RedSlot slot() const { return rs; }
    __device__ void fin(double* tot) const {
        PcgState& S = *st;
        S.rel = __ddiv_rn(__dsqrt_rn(tot[0]), S.bnorm);
        if (S.hist) S.hist[S.it] = S.rel;
        S.hist_len = S.it + 1;
        if (S.rel <= S.rel_tol) {
            S.status = 0;
            S.iterations = S.it;
            S.done = 1;
            if (S.use_cond) cudaGraphSetConditional(S.cond, 0);
            return;
        }
        if (kind != IBMGPU_PC_SA) {
            S.beta = __ddiv_rn(tot[1], S.rz);
            S.rz = tot[1];
            finish_iteration(S);
        }
    }
};

struct FinBeta {  // B3 (SA): beta from the fused r.z of the V-cycle's last kernel
    PcgState* st;
    __device__ void operator()(double* tot) const {
        PcgState& S = *st;
        S.beta = __ddiv_rn(tot[0], S.rz);
        S.rz = tot[0];
        finish_iteration(S);
    }
};

struct BodyP {  // B4: p = z + beta p
    static constexpr int NR = 0;
    const double* z;
    double* p;
    const PcgState* st;
    __device__ bool skip() const { return flag_set(&st->done); }
    __device__ void row(int i, double*) const { p[i] = addd(z[i], mul(st->beta, p[i])); }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

// V-cycle last kernel adapter for the PCG
template <class Fin>
struct LastDot {
    Ctx* c;
    const int* done;
    RedSlot rs;
    Fin f;
    cudaStream_t s;
    void operator()(Level& lv, const double* b, double* z) const {
        launch_spmv(c, lv.A, XPlain{lv.x.p}, EpiPostSmoothDot<Fin>{lv.wd.p, b, lv.x.p, z, done, rs, f}, s);
    }
    void xfer(Hier* h, const double* b, const double* e, double* z) const {
        const XSinkDot<Fin> sink{z, done, rs, f};
        const XferPlan X = xfer_plan(h);
        launch_k(c, k_xfer_up<XSinkDot<Fin>>, h->x0.tiles, kXThreads, s, X, b, e, sink);
        if (h->x0.tail_ctas)
            launch_k(c, k_xfer_up_tail<XSinkDot<Fin>>, h->x0.tail_ctas, kBlock, s, X, b, e, sink, h->x0.tiles);
        launch_k(c, k_finalize<XSinkDot<Fin>>, 1, kFinThreads, s, sink, h->x0.tiles + h->x0.tail_ctas);
    }
};

template <class Fin>
struct BodyDotAfterCoarse {  // no-level hierarchy: r.z after the dense solve
    static constexpr int NR = 1;
    const double* r;
    const double* z;
    const int* done;
    RedSlot rs;
    Fin f;
    __device__ bool skip() const { return done && flag_set(done); }
    __device__ void row(int i, double* acc) const { acc[0] += r[i] * z[i]; }
    __device__ RedSlot slot() const { return rs; }
    __device__ void fin(double* tot) const { f(tot); }
};

}  // namespace

// ---------------------------------------------------------------- plan
// Pinned PcgState slots are recycled instead of freed: cudaFreeHost synchronises the whole device,
// and a moving body retires one solve-2 plan per step — each retirement stalled the solve stream
// behind the operator pipeline's kernels. A slot is reused once the event recorded on its plan's
// last stream at retirement has completed (its final device-to-host copy has landed).
namespace {
struct PinSlot {
    PcgState* p;
    cudaEvent_t ev;
};
std::mutex g_pin_mu;
std::vector<PinSlot> g_pin_free;

PcgState* pin_acquire() {
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        for (size_t i = 0; i < g_pin_free.size(); ++i) {
            if (cudaEventQuery(g_pin_free[i].ev) == cudaSuccess) {
                PinSlot sl = g_pin_free[i];
                g_pin_free.erase(g_pin_free.begin() + (long)i);
                cudaEventDestroy(sl.ev);
                return sl.p;
            }
        }
    }
    PcgState* p = nullptr;
    CK(cudaMallocHost(&p, sizeof(PcgState)));
    return p;
}

void pin_release(PcgState* p, cudaStream_t last) {
    cudaEvent_t ev = nullptr;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return;  // leak one slot
    if (cudaEventRecord(ev, last) != cudaSuccess) {
        cudaEventDestroy(ev);
        return;
    }
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back({p, ev});
}
}  // namespace

PcgPlan::PcgPlan(Ctx* c, Mat* A_, int kind_, Hier* h_) : A(A_), kind(kind_), h(h_) {
    require(A->rows == A->cols, "pcg: dimension mismatch");
    if (!A->planned) mat_plan(c, A);
    const size_t n = (size_t)A->rows;
    hier_id = h ? h->id : 0;
    b.alloc(c, n);
    x.alloc(c, n);
    r.alloc(c, n);
    z.alloc(c, n);
    p.alloc(c, n);
    Ap.alloc(c, n);
    if (kind == IBMGPU_PC_DIAGONAL) {
        DBuf<double> d(c, n);
        diag_of(c, A, d.p);
        std::vector<double> hd(n);
        d2h(c, hd.data(), d.p, n);
        sync(c);
        for (size_t i = 0; i < n; ++i) {
            if (hd[i] == 0.0) fail(IBMGPU_EINVAL, "diagonal preconditioner: zero diagonal entry");
            hd[i] = 1.0 / hd[i];
        }
        invd.alloc(c, n);
        h2d(c, invd.p, hd.data(), n);
    }
    st.alloc(c, 1);
    int g = std::max(spmv_grid(A), elem_grid(c, (long long)n));
    if (h)
        for (auto& lv : h->levels) g = std::max(g, spmv_grid(lv->A));
    if (h && h->x0.on) g = std::max(g, h->x0.tiles + h->x0.tail_ctas);
    partials.alloc(c, (size_t)std::max(g, 1) * 2);
    counter.alloc(c, 1);
    CK(cudaMemsetAsync(counter.p, 0, sizeof(unsigned), c->stream));
    host_st = pin_acquire();
    last_stream = c->stream;
    build_graph(c);
}

PcgPlan::~PcgPlan() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (host_st) pin_release(host_st, last_stream);
}

void PcgPlan::enqueue_init(Ctx* c, cudaStream_t s) {
    const int n = A->rows;
    const RedSlot rs{partials.p, counter.p};
    PcgState* S = st.p;
    const int* done = &S->done;
    launch_spmv(c, A, XPlain{x.p}, EpiInitResidual{b.p, r.p, rs, S}, s);
    const int eg = elem_grid(c, n);
    launch_elem(c, n, eg, BodyZeroX{x.p, S}, s);
    if (kind == IBMGPU_PC_SA) {
        if (h->levels.empty()) {
            coarse_solve(c, h, r.p, z.p, done, s);
            launch_elem(c, n, eg, BodyDotAfterCoarse<FinInitRz>{r.p, z.p, done, rs, FinInitRz{S}}, s);
        } else {
            vcycle_launch(c, h, r.p, z.p, done, LastDot<FinInitRz>{c, done, rs, FinInitRz{S}, s}, s);
        }
        launch_elem(c, n, eg, BodyCopy{z.p, p.p, S}, s);
    } else {
        launch_elem(c, n, eg, BodyInitZ{r.p, kind == IBMGPU_PC_DIAGONAL ? invd.p : nullptr, z.p, p.p, rs, S}, s);
    }
}

void PcgPlan::enqueue_body(Ctx* c, cudaStream_t s) {
    const int n = A->rows;
    const RedSlot rs{partials.p, counter.p};
    PcgState* S = st.p;
    const int* done = &S->done;
    const int eg = elem_grid(c, n);
    launch_spmv(c, A, XPlain{p.p}, EpiSpmvPAp{p.p, Ap.p, rs, S}, s);
    launch_elem(c, n, eg,
                BodyUpdate{x.p, r.p, p.p, Ap.p, kind == IBMGPU_PC_DIAGONAL ? invd.p : nullptr, z.p, kind, rs, S}, s);
    if (kind == IBMGPU_PC_SA) {
        if (h->levels.empty()) {
            coarse_solve(c, h, r.p, z.p, done, s);
            launch_elem(c, n, eg, BodyDotAfterCoarse<FinBeta>{r.p, z.p, done, rs, FinBeta{S}}, s);
        } else {
            vcycle_launch(c, h, r.p, z.p, done, LastDot<FinBeta>{c, done, rs, FinBeta{S}, s}, s);
        }
    }
    launch_elem(c, n, eg, BodyP{z.p, p.p, S}, s);
}

void PcgPlan::build_graph(Ctx* c) {
    cudaStream_t s = c->stream;
    const long long l0 = c->launches;
    CK(cudaGraphCreate(&graph, 0));
    CK(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
    // write the handle into the state before anything reads it
    CK(cudaStreamBeginCaptureToGraph(s, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    enqueue_init(c, s);
    const long long l1 = c->launches;
    // conditional WHILE node after the init nodes
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    cudaGraph_t capg;
    CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &capg, &deps, &ndeps));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    CK(cudaGraphAddNode(&cnode, capg, deps, ndeps, &cp));
    CK(cudaStreamUpdateCaptureDependencies(s, &cnode, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
    cudaStream_t s2;
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    CK(cudaStreamBeginCaptureToGraph(s2, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    enqueue_body(c, s2);
    const long long l2 = c->launches;
    CK(cudaStreamEndCapture(s2, &bodyg));
    CK(cudaStreamDestroy(s2));
    CK(cudaStreamEndCapture(s, &graph));
    CK(cudaGraphInstantiate(&exec, graph, 0));
    kernels_init = (int)(l1 - l0);
    kernels_iter = (int)(l2 - l1);
    c->launches = l0;  // capture is not execution
}

void PcgPlan::run(Ctx* c, const ibm_solver_params& prm, double* hist_dev) {
    last_stream = c->stream;
    PcgState& H = *host_st;
    H = PcgState{};
    H.rel_tol = prm.rel_tol;
    H.max_iters = prm.max_iters;
    H.hist = hist_dev;
    H.cond = cond;
    H.use_cond = c->eager ? 0 : 1;
    CK(cudaMemcpyAsync(st.p, &H, sizeof(PcgState), cudaMemcpyHostToDevice, c->stream));
    last_eager = c->eager != 0;
    if (!last_eager) {
        CK(cudaGraphLaunch(exec, c->stream));
    } else {
        // Profiling mode (IBMGPU_EAGER=1): the same kernels launched from the host, 8 iterations
        // between done-flag checks (ncu cannot profile kernel nodes of conditional graphs).
        enqueue_init(c, c->stream);
        for (int it = 0; it <= prm.max_iters + 8; it += 8) {
            for (int k = 0; k < 8; ++k) enqueue_body(c, c->stream);
            CK(cudaMemcpyAsync(host_st, st.p, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
            sync(c);
            if (host_st->done) break;
        }
    }
    CK(cudaMemcpyAsync(host_st, st.p, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
}

void PcgPlan::finish(Ctx* c, ibm_solve_result* res) {
    sync(c);
    const PcgState& H = *host_st;
    // iterations executed: init + one body per started iteration (eager mode counted at launch)
    if (!last_eager) c->launches += kernels_init + (long long)kernels_iter * std::max(H.it, 0);
    if (res) {
        res->iterations = H.iterations;
        res->rel_residual = H.rel;
        res->status = H.status;
        res->history_len = H.hist_len;
    }
}

// ---------------------------------------------------------------- plan cache
namespace {
struct Cache {
    std::map<std::tuple<const Mat*, int, long long>, std::unique_ptr<PcgPlan>> plans;
};
Cache& cache_of(Ctx* c) {
    if (!c->pcg_cache) c->pcg_cache = new Cache();
    return *static_cast<Cache*>(c->pcg_cache);
}
}  // namespace

PcgPlan* pcg_plan(Ctx* c, Mat* A, int kind, Hier* h) {
    auto& C = cache_of(c);
    const auto key = std::make_tuple((const Mat*)A, kind, h ? h->id : 0ll);
    auto it = C.plans.find(key);
    if (it != C.plans.end()) return it->second.get();
    auto plan = std::make_unique<PcgPlan>(c, A, kind, h);
    auto* raw = plan.get();
    C.plans[key] = std::move(plan);
    return raw;
}

void pcg_forget(Ctx* c, const Mat* A, const Hier* h) {
    if (!c->pcg_cache) return;
    auto& C = cache_of(c);
    for (auto it = C.plans.begin(); it != C.plans.end();) {
        if ((A && std::get<0>(it->first) == A) || (h && it->second->h == h))
            it = C.plans.erase(it);
        else
            ++it;
    }
}

void pcg_cache_free(Ctx* c) {
    if (c->pcg_cache) delete static_cast<Cache*>(c->pcg_cache);
    c->pcg_cache = nullptr;
}

void validate_params(const ibm_solver_params& p) {
    // krylov.hpp:21-24
    if (!(p.rel_tol > 0.0 && p.rel_tol < 1.0)) fail(IBMGPU_EINVAL, "solver: rel_tol must be in (0,1)");
    if (p.max_iters < 1) fail(IBMGPU_EINVAL, "solver: max_iters must be >= 1");
}

void pcg_solve(Ctx* c, Mat* A, int kind, Hier* h, const double* b, double* x, const ibm_solver_params& prm,
               ibm_solve_result* res, double* hist_host) {
    validate_params(prm);
    require(A->rows == A->cols, "pcg: dimension mismatch");
    require(kind >= 0 && kind <= 2, "pcg: unknown preconditioner");
    require(kind != IBMGPU_PC_SA || h != nullptr, "pcg: SA preconditioner needs a hierarchy");
    require(kind != IBMGPU_PC_SA || h->levels.empty() ? (kind != IBMGPU_PC_SA || h->n_c == A->rows)
                                                      : h->levels[0]->A->rows == A->rows,
            "pcg: hierarchy size does not match the matrix");
    if (prm.check_symmetry) require(is_symmetric(c, A, 1e-12), "pcg: matrix is not symmetric");
    const int n = A->rows;
    if (n == 0) {
        if (res) *res = ibm_solve_result{0, 0.0, 0, 0};
        return;
    }
    PcgPlan* P = pcg_plan(c, A, kind, h);
    d2d(c, P->b.p, b, (size_t)n);
    d2d(c, P->x.p, x, (size_t)n);
    DBuf<double> hist;
    if (prm.record_history) hist.alloc(c, (size_t)prm.max_iters + 1);
    P->run(c, prm, prm.record_history ? hist.p : nullptr);
    d2d(c, x, P->x.p, (size_t)n);
    P->finish(c, res);
    if (prm.record_history && hist_host && res) d2h(c, hist_host, hist.p, (size_t)res->history_len), sync(c);
}

}  // namespace ibmgpu

// ---------------------------------------------------------------- pcg with a caller's preconditioner
// krylov.hpp:70-136 with M = the caller's apply (the reference's virtual Preconditioner::apply,
// krylov.hpp:39-43). The preconditioner is opaque, so the loop is host-driven: one SpMV, the
// vector updates and fixed-order (deterministic) dot products per iteration, the scalars read
// back as the reference's loop reads them.
namespace ibmgpu {
namespace {
constexpr int kDotBlocks = 592;  // 4 x 148 SMs
__global__ void __launch_bounds__(256) k_dot_part(int n, const double* __restrict__ a, const double* __restrict__ b,
                                                  double* __restrict__ part) {
    __shared__ double sh[256];
    double s = 0.0;
    for (int i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) s = addd(s, mul(a[i], b[i]));
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] = addd(sh[threadIdx.x], sh[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void k_dot_fin(int nb, const double* __restrict__ part, double* __restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int k = 0; k < nb; ++k) s = addd(s, part[k]);
        *out = s;
    }
}
__global__ void k_resid(int n, const double* __restrict__ b, const double* __restrict__ ax, double* __restrict__ r) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) r[i] = subd(b[i], ax[i]);
}
__global__ void k_xr_update(int n, double alpha, const double* __restrict__ p, const double* __restrict__ ap,
                            double* __restrict__ x, double* __restrict__ r) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        x[i] = addd(x[i], mul(alpha, p[i]));   // axpy(alpha, p, x)
        r[i] = addd(r[i], mul(-alpha, ap[i]));  // axpy(-alpha, Ap, r)
    }
}
__global__ void k_p_update(int n, double beta, const double* __restrict__ z, double* __restrict__ p) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = addd(z[i], mul(beta, p[i]));
}
inline int eb(int n) { return (n + 255) / 256; }
}  // namespace

void pcg_callback(Ctx* c, Mat* A, ibmgpu_apply_fn apply, void* user, const double* b, double* x,
                  const ibm_solver_params& prm, ibm_solve_result* res, double* hist_host) {
    validate_params(prm);
    require(A->rows == A->cols, "pcg: dimension mismatch");
    require(apply != nullptr, "pcg: null preconditioner");
    if (prm.check_symmetry) require(is_symmetric(c, A, 1e-12), "pcg: matrix is not symmetric");
    if (!A->planned) mat_plan(c, A);
    const int n = A->rows;
    ibm_solve_result out{0, 0.0, 0, 0};
    auto finish = [&] {
        if (res) *res = out;
    };
    if (n == 0) return finish();
    DBuf<double> r(c, n), z(c, n), p(c, n), ap(c, n), part(c, kDotBlocks), scal(c, 1);
    auto dot = [&](const double* u, const double* v) {
        k_dot_part<<<kDotBlocks, 256, 0, c->stream>>>(n, u, v, part.p);
        CK_LAUNCH(c);
        k_dot_fin<<<1, 32, 0, c->stream>>>(kDotBlocks, part.p, scal.p);
        CK_LAUNCH(c);
        return d2h_scalar(c, scal.p);
    };
    auto record = [&](double rel) {
        if (prm.record_history && hist_host && out.history_len <= prm.max_iters) hist_host[out.history_len++] = rel;
    };
    auto precondition = [&] {
        sync(c);
        if (apply(user, n, r.p, z.p) != 0) fail(IBMGPU_EINVAL, "pcg: preconditioner apply failed");
    };
    const double bnorm = std::sqrt(dot(b, b));
    if (bnorm == 0.0) {  // krylov.hpp:85-89
        CK(cudaMemsetAsync(x, 0, sizeof(double) * (size_t)n, c->stream));
        sync(c);
        return finish();
    }
    spmv(c, A, x, ap.p);
    k_resid<<<eb(n), 256, 0, c->stream>>>(n, b, ap.p, r.p);
    CK_LAUNCH(c);
    double rel = std::sqrt(dot(r.p, r.p)) / bnorm;
    out.rel_residual = rel;
    record(rel);
    if (rel <= prm.rel_tol) return finish();
    precondition();
    d2d(c, p.p, z.p, (size_t)n);
    double rz = dot(r.p, z.p);
    for (int it = 1; it <= prm.max_iters; ++it) {
        spmv(c, A, p.p, ap.p);
        const double pAp = dot(p.p, ap.p);
        if (pAp <= 0.0) {  // krylov.hpp:110-115
            out.iterations = it - 1;
            out.status = 2;
            return finish();
        }
        const double alpha = rz / pAp;
        k_xr_update<<<eb(n), 256, 0, c->stream>>>(n, alpha, p.p, ap.p, x, r.p);
        CK_LAUNCH(c);
        rel = std::sqrt(dot(r.p, r.p)) / bnorm;
        out.rel_residual = rel;
        record(rel);
        if (rel <= prm.rel_tol) {
            out.iterations = it;
            return finish();
        }
        precondition();
        const double rz_new = dot(r.p, z.p);
        const double beta = rz_new / rz;
        rz = rz_new;
        k_p_update<<<eb(n), 256, 0, c->stream>>>(n, beta, z.p, p.p);
        CK_LAUNCH(c);
    }
    out.iterations = prm.max_iters;
    out.status = 1;
    sync(c);
    finish();
}
}  // namespace ibmgpu

// ---------------------------------------------------------------- amg_solve (amg.hpp:250-280)
namespace ibmgpu {
namespace {
struct EpiResidNorm {  // r_i = b_i - s ; reduce r.r (and b.b)
    static constexpr int NR = 2;
    const double* b;
    double* r;
    RedSlot rs;
    double* out;  // [bb, rr]
    __device__ bool skip() const { return false; }
    __device__ void row(int i, double s, double* acc) const {
        const double ri = subd(b[i], s);
        r[i] = ri;
        acc[0] += b[i] * b[i];
        acc[1] += ri * ri;
    }
    __device__ RedSlot slot() const { return rs; }
    __device__ void fin(double* tot) const {
        out[0] = tot[0];
        out[1] = tot[1];
    }
};
struct BodyAxpy1 {
    static constexpr int NR = 0;
    const double* z;
    double* x;
    __device__ bool skip() const { return false; }
    __device__ void row(int i, double*) const { x[i] = addd(x[i], z[i]); }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};
}  // namespace

void amg_solve(Ctx* c, Mat* A, Hier* h, const double* b, double* x, const ibm_solver_params& prm,
               ibm_solve_result* res) {
    validate_params(prm);
    require(A->rows == A->cols, "amg_solve: dimension mismatch");
    if (!A->planned) mat_plan(c, A);
    const int n = A->rows;
    DBuf<double> r(c, (size_t)n), z(c, (size_t)n), part(c, (size_t)std::max(spmv_grid(A), 1) * 2), nrm(c, 2);
    DBuf<unsigned> cnt(c, 1);
    CK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned), c->stream));
    ibm_solve_result R{0, 0.0, 1, 0};
    double bnorm = -1.0;
    for (int it = 0; it <= prm.max_iters; ++it) {
        launch_spmv(c, A, XPlain{x}, EpiResidNorm{b, r.p, RedSlot{part.p, cnt.p}, nrm.p}, c->stream);
        double hn[2];
        d2h(c, hn, nrm.p, 2);
        sync(c);
        if (bnorm < 0.0) {
            bnorm = std::sqrt(hn[0]);
            if (bnorm == 0.0) {
                CK(cudaMemsetAsync(x, 0, sizeof(double) * (size_t)n, c->stream));
                R = ibm_solve_result{0, 0.0, 0, 0};
                break;
            }
        }
        const double rel = std::sqrt(hn[1]) / bnorm;
        static const bool dbg = std::getenv("IBMGPU_DEBUG_AMG") != nullptr;
        if (dbg && (it < 12 || it % 1000 == 0)) std::fprintf(stderr, "[amg] it %d rel %.6e bb %.6e\n", it, rel, hn[0]);
        R.rel_residual = rel;
        R.iterations = it;
        if (rel <= prm.rel_tol) {
            R.status = 0;
            break;
        }
        if (it == prm.max_iters) break;
        vcycle_launch(c, h, r.p, z.p, nullptr, LastPlain{c, nullptr, c->stream}, c->stream);
        launch_elem(c, n, elem_grid(c, n), BodyAxpy1{z.p, x}, c->stream);
    }
    sync(c);
    if (res) *res = R;
}
}  // namespace ibmgpu
