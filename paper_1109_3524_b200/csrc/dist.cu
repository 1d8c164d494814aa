// dist.cu — row-slab multi-GPU PCG for the modified Poisson solve.
//
// Decomposition. Rows of the solve are owned by ranks (pressure rows by j-slab, body rows by the
// slab that contains the point; host/dist_plan.cpp). Every rank builds the full operators and the
// full SA hierarchy (deterministic, so identical on all ranks) and keeps, per distributed level,
// its owned rows of A_l, P_l and P_l^T with halo-extended column numbering. Coarse aggregates
// follow the owner of their lowest-index member, so most of P's and P^T's entries stay local.
// Levels with fewer than `min_rows` rows — the latency-bound tail of the cycle — are replicated:
// the rank-partial restriction P^T r is summed across ranks (one allreduce of the level-D vector),
// and every rank runs the remaining V-cycle on full vectors (amg.cuh kernels unchanged).
//
// Per PCG iteration (SA): 1 + 4 D halo exchanges, 1 vector allreduce at the level switch, and ONE
// scalar allreduce: the single-reduction recurrence applies the SpMV to z
// (w = A z) and reduces {r.r, r.z, z.w, z.Ap_old} together; A p follows as w + beta Ap_old and
// p.Ap from the recurrence. Because every local matrix keeps the global entry order inside a row,
// every distributed SpMV rounds exactly like the single-GPU one; the dot products (sums of
// per-rank partials), the recurrence for p.Ap and the switch restriction differ in rounding.
//
// Communication backends: NCCL (one process per GPU; grouped ncclSend/ncclRecv for halos,
// ncclAllReduce for scalars and the switch vector), or loopback — all ranks of the partition
// emulated in one context on one GPU, halos moved by device copies, so the same decomposition is
// testable without peers. Neither backend has kernels waiting on other ranks' kernels.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>

#include "amg.cuh"
#include "dist.cuh"
#include "host/dist_plan.hpp"
#include "internal.cuh"
#include "kern.cuh"
#include "pcg.cuh"

namespace ibmgpu {

// ---------------------------------------------------------------- NCCL, loaded on first use
namespace {
struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
};

const NcclApi& nccl_api() {
    static NcclApi api;
    static bool loaded = false;
    if (loaded) return api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) fail(IBMGPU_ENCCL, std::string("NCCL not loadable: ") + dlerror());
    auto sym = [&](auto& fn, const char* name) {
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
        if (!fn) fail(IBMGPU_ENCCL, std::string("NCCL symbol missing: ") + name);
    };
    sym(api.getUniqueId, "ncclGetUniqueId");
    sym(api.commInitRank, "ncclCommInitRank");
    sym(api.commDestroy, "ncclCommDestroy");
    sym(api.send, "ncclSend");
    sym(api.recv, "ncclRecv");
    sym(api.groupStart, "ncclGroupStart");
    sym(api.groupEnd, "ncclGroupEnd");
    sym(api.allReduce, "ncclAllReduce");
    sym(api.errorString, "ncclGetErrorString");
    loaded = true;
    return api;
}
}  // namespace

#define NK(call)                                                                                     \
    do {                                                                                             \
        ncclResult_t r_ = (call);                                                                    \
        if (r_ != ncclSuccess) fail(IBMGPU_ENCCL, std::string(#call) + ": " + nccl_api().errorString(r_)); \
    } while (0)

void nccl_comm_init(Ctx* c, const void* id) {
    const auto& N = nccl_api();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    ncclComm_t comm = nullptr;
    NK(N.commInitRank(&comm, c->nranks, uid, c->rank));
    c->nccl = comm;
}

void nccl_comm_free(Ctx* c) {
    if (c->nccl) nccl_api().commDestroy(static_cast<ncclComm_t>(c->nccl));
    c->nccl = nullptr;
}

void nccl_unique_id(void* out) {
    ncclUniqueId uid;
    NK(nccl_api().getUniqueId(&uid));
    std::memcpy(out, &uid, sizeof uid);
}

namespace {

// ---------------------------------------------------------------- small kernels
struct BodyPack {  // out[k] = v[idx[k]]
    static constexpr int NR = 0;
    const int* idx;
    const double* v;
    double* out;
    __device__ bool skip() const { return false; }
    __device__ void row(int k, double*) const { out[k] = v[idx[k]]; }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};
struct BodyScatter {  // full[idx[k]] = v[k]
    static constexpr int NR = 0;
    const int* idx;
    const double* v;
    double* full;
    __device__ bool skip() const { return false; }
    __device__ void row(int k, double*) const { full[idx[k]] = v[k]; }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};
constexpr int kMaxLoop = 16;
struct RankPtrs {
    double* p[kMaxLoop];
    int R;
};
struct BodySumRanks {  // loopback allreduce: every rank's buffer := sum over ranks (rank order)
    static constexpr int NR = 0;
    RankPtrs P;
    __device__ bool skip() const { return false; }
    __device__ void row(int i, double*) const {
        double s = P.p[0][i];
        for (int r = 1; r < P.R; ++r) s += P.p[r][i];
        for (int r = 0; r < P.R; ++r) P.p[r][i] = s;
    }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

template <int NR>
struct FinStore {
    double* red;
    __device__ void operator()(double* tot) const {
#pragma unroll
        for (int r = 0; r < NR; ++r) red[r] = tot[r];
    }
};

__device__ __forceinline__ bool is_done(const PcgState* S) { return flag_set(&S->done); }

struct EpiDInit {  // r = b - A x ; partial b.b, r.r
    static constexpr int NR = 2;
    const double* b;
    double* r;
    RedSlot rs;
    double* red;
    __device__ bool skip() const { return false; }
    __device__ void row(int i, double s, double* acc) const {
        const double bi = b[i];
        const double ri = subd(bi, s);
        r[i] = ri;
        acc[0] += bi * bi;
        acc[1] += ri * ri;
    }
    __device__ RedSlot slot() const { return rs; }
    __device__ void fin(double* tot) const { FinStore<2>{red}(tot); }
};

struct BodyDZeroX {
    static constexpr int NR = 0;
    double* x;
    const PcgState* st;
    __device__ bool skip() const { return !st->zero_x; }
    __device__ void row(int i, double*) const { x[i] = 0.0; }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

struct BodyDPrecond {  // z = M r for the identity / diagonal preconditioners (krylov.hpp:46-66)
    static constexpr int NR = 0;
    const double* r;
    const double* invd;
    double* z;
    const PcgState* st;
    __device__ bool skip() const { return is_done(st); }
    __device__ void row(int i, double*) const { z[i] = invd ? mul(r[i], invd[i]) : r[i]; }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

// w = A z with the iteration's four partial sums r.r, r.z, z.w, z.Ap_old — everything the
// single-reduction recurrence needs, so one allreduce per iteration
struct EpiDFused {
    static constexpr int NR = 4;
    const double* r;
    const double* z;
    const double* Ap;
    double* w;
    RedSlot rs;
    double* red;
    const PcgState* st;
    __device__ bool skip() const { return is_done(st); }
    __device__ void touch(int i) const {
        pf(r + i);
        pf(Ap + i);
    }
    __device__ void row(int i, double s, double* acc) const {
        w[i] = s;
        const double ri = r[i], zi = z[i];
        acc[0] += ri * ri;
        acc[1] += ri * zi;
        acc[2] += zi * s;
        acc[3] += zi * Ap[i];
    }
    __device__ RedSlot slot() const { return rs; }
    __device__ void fin(double* tot) const { FinStore<4>{red}(tot); }
};

// p = z + beta p, Ap = w + beta Ap (A p without a second SpMV), x += alpha p, r -= alpha Ap
struct BodyDUpd {
    static constexpr int NR = 0;
    double* x;
    double* r;
    double* p;
    double* Ap;
    const double* z;
    const double* w;
    const PcgState* st;
    __device__ bool skip() const { return is_done(st); }
    __device__ void row(int i, double*) const {
        const double b = st->beta, a = st->alpha;
        const double pi = b == 0.0 ? z[i] : addd(z[i], mul(b, p[i]));  // first direction: p = z
        const double api = b == 0.0 ? w[i] : addd(w[i], mul(b, Ap[i]));
        p[i] = pi;
        Ap[i] = api;
        x[i] = addd(x[i], mul(a, pi));
        r[i] = addd(r[i], mul(-a, api));
    }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

// Scalar recurrence from the globally reduced sums. PH_INIT: krylov.hpp:85-100 on r0.
// PH_FUSED (sums r.r, r.z, z.w, z.Ap_old of iteration `it` = updates done so far):
//   convergence of r_it exactly where krylov.hpp:126-127 tests it (it > 0), then
//   beta = rz/rz_old, pAp = z.w + 2 beta z.Ap_old + beta^2 pAp_old  (= p.Ap for symmetric A),
//   breakdown if pAp <= 0 (krylov.hpp:109-114), alpha = rz/pAp.
// The iterates are krylov.hpp's up to rounding; `iterations` counts updates as the reference does.
enum { PH_INIT = 0, PH_FUSED = 1 };

__global__ void k_dscal(PcgState* Sp, const double* red, int phase) {
    pdl_wait();
    PcgState& S = *Sp;
    if (phase == PH_INIT) {
        S.it = 0;
        S.bnorm = __dsqrt_rn(red[0]);
        if (S.bnorm == 0.0) {
            S.status = 0, S.iterations = 0, S.rel = 0.0, S.done = 1, S.zero_x = 1;
            return;
        }
        S.rel = __ddiv_rn(__dsqrt_rn(red[1]), S.bnorm);
        if (S.hist) S.hist[0] = S.rel;
        S.hist_len = 1;
        if (S.rel <= S.rel_tol) S.status = 0, S.iterations = 0, S.done = 1;
        return;
    }
    if (S.done) return;
    const double rr = red[0], rz = red[1], zw = red[2], zap = red[3];
    if (S.it > 0) {
        S.rel = __ddiv_rn(__dsqrt_rn(rr), S.bnorm);
        if (S.hist) S.hist[S.it] = S.rel;
        S.hist_len = S.it + 1;
        if (S.rel <= S.rel_tol) {
            S.status = 0, S.iterations = S.it, S.done = 1;
            return;
        }
        if (S.it >= S.max_iters) {
            S.status = 1, S.iterations = S.max_iters, S.done = 1;
            return;
        }
    }
    const double beta = S.it == 0 ? 0.0 : __ddiv_rn(rz, S.rz);
    const double pAp = S.it == 0 ? zw : addd(addd(zw, mul(mul(2.0, beta), zap)), mul(mul(beta, beta), S.pAp));
    if (!(pAp > 0.0)) {
        S.status = 2, S.iterations = S.it, S.done = 1;
        return;
    }
    S.beta = beta;
    S.alpha = __ddiv_rn(rz, pAp);
    S.rz = rz;
    S.pAp = pAp;
    ++S.it;
}

// ---------------------------------------------------------------- distributed pieces
struct DMat {
    Mat* m = nullptr;
    int n_own = 0, n_halo = 0;
    std::vector<int> send_off, recv_off;  // nranks + 1 (host)
    DBuf<int> send_idx;
    DBuf<double> send_buf;
    ~DMat() { delete m; }
    int sends() const { return send_off.empty() ? 0 : send_off.back(); }
};

void dmat_from_plan(Ctx* c, DMat& d, const ibmhost::DistPlan& P) {
    d.n_own = P.n_own;
    d.n_halo = P.n_halo();
    d.m = mat_upload(c, (int)P.rows.size(), P.n_own + P.n_halo(), (int)P.ci.size(), P.rp.data(), P.ci.data(),
                     P.v.data());
    d.send_off = P.send_off;
    d.recv_off = P.recv_off;
    d.send_idx.alloc(c, std::max<size_t>(P.send_idx.size(), 1));
    h2d(c, d.send_idx.p, P.send_idx.data(), P.send_idx.size());
    d.send_buf.alloc(c, std::max<size_t>(P.send_idx.size(), 1));
}

struct HostCsr {
    int rows = 0, cols = 0;
    std::vector<int> rp, ci;
    std::vector<double> v;
};
HostCsr download(Ctx* c, const Mat* m) {
    HostCsr h;
    h.rows = m->rows, h.cols = m->cols;
    h.rp.resize((size_t)m->rows + 1);
    h.ci.resize((size_t)m->nnz);
    h.v.resize((size_t)m->nnz);
    mat_download(c, m, h.rp.data(), h.ci.data(), h.v.data());
    return h;
}

// rows of M restricted to entries whose column this rank owns (columns renumbered to the owned
// index); every row of M is kept. Used for the rank-partial restriction at the level switch.
Mat* colsplit(Ctx* c, const HostCsr& M, const std::vector<int>& col_owner, int rank) {
    std::vector<int> g2l((size_t)M.cols, -1);
    int n_own = 0;
    for (int j = 0; j < M.cols; ++j)
        if (col_owner[j] == rank) g2l[j] = n_own++;
    std::vector<int> rp(1, 0), ci;
    std::vector<double> v;
    for (int r = 0; r < M.rows; ++r) {
        for (int k = M.rp[r]; k < M.rp[r + 1]; ++k)
            if (g2l[M.ci[k]] >= 0) ci.push_back(g2l[M.ci[k]]), v.push_back(M.v[k]);
        rp.push_back((int)ci.size());
    }
    return mat_upload(c, M.rows, n_own, (int)ci.size(), rp.data(), ci.data(), v.data());
}

struct DLev {
    DMat A, P, Pt;        // P: own(l) x ext(l+1) or full level D ; Pt: own(l+1) x ext(l), or colsplit at the switch
    bool switch_below = false;
    int n_own = 0, cap = 0;
    DBuf<double> wd;      // omega/diag in A's extended layout
    DBuf<double> b, x, r, xo;
};

struct RankData {
    int rank = 0;
    int n_own = 0;  // level 0
    std::vector<int> own0;
    DBuf<int> own0_dev;
    DMat A;  // the PCG matrix
    std::vector<std::unique_ptr<DLev>> lev;
    DBuf<double> b, x, r, z, p, Ap, w, invd;  // x, r, z extended (A0 halo)
    DBuf<double> bD, xD;                    // full level-D vectors (replicated part)
    DBuf<PcgState> st;
    DBuf<double> red, partials;
    PcgState* host_st = nullptr;
    ~RankData() {
        if (host_st) cudaFreeHost(host_st);
    }
};

}  // namespace
}  // namespace ibmgpu

struct ibmgpu_dist {
    ibmgpu::Ctx* c = nullptr;
    ibmgpu::Mat* A = nullptr;
    ibmgpu::Hier* h = nullptr;
    int kind = 0;
    int R = 1;           // ranks of the partition
    bool loop = false;   // loopback (all ranks local)
    bool loop_nccl = false;  // loopback whose halos travel as NCCL send/recv to self (1-rank comm)
    int D = 0;           // distributed levels
    int n = 0;
    std::vector<std::unique_ptr<ibmgpu::RankData>> ranks;  // local ranks
    std::vector<std::vector<int>> owner;                   // per level (0..D), host
    ibmgpu::DBuf<int> allown;                              // NCCL: all ranks' level-0 own lists
    std::vector<int> own_off;                              // R + 1
    ibmgpu::DBuf<double> gather_buf;                       // NCCL: R * max_own
    int max_own = 0;
    cudaGraphExec_t iter_exec = nullptr;                   // one captured PCG iteration
    bool no_graph = false;                                 // capture failed: eager iterations
    int iter_kernels = 0;
    int* done_host = nullptr;                              // pinned, 2 slots
    cudaEvent_t ev[2] = {};
    ~ibmgpu_dist() {
        if (iter_exec) cudaGraphExecDestroy(iter_exec);
        if (done_host) cudaFreeHost(done_host);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
    }
};

namespace ibmgpu {
namespace {
using Dist = ibmgpu_dist;

template <class GetM, class GetV>
void exchange(Dist* d, GetM gm, GetV gv) {
    Ctx* c = d->c;
    cudaStream_t s = c->stream;
    for (auto& rk : d->ranks) {
        DMat& M = gm(*rk);
        const int ns = M.sends();
        if (ns) launch_elem(c, ns, elem_grid(c, ns), BodyPack{M.send_idx.p, gv(*rk), M.send_buf.p}, s);
    }
    if (d->R == 1) return;
    if (d->loop) {
#ifdef IBMGPU_TIMING_EXPERIMENTS
        // IBMGPU_DIST_NOCOPY=1 (timing builds only, results are wrong): skip the loopback halo
        // copies to separate their cost from the ranks' own work. Never compiled into the product.
        static const bool nocopy = std::getenv("IBMGPU_DIST_NOCOPY") != nullptr;
        if (nocopy) return;
#endif
        if (d->loop_nccl) {
            // every virtual rank's halo through the NCCL p2p path: send/recv pairs to self, issued
            // in the same order so the k-th send matches the k-th receive
            const auto& N = nccl_api();
            auto comm = static_cast<ncclComm_t>(c->nccl);
            NK(N.groupStart());
            for (int r = 0; r < d->R; ++r) {
                DMat& Mr = gm(*d->ranks[r]);
                double* dst = gv(*d->ranks[r]) + Mr.n_own;
                for (int q = 0; q < d->R; ++q) {
                    if (q == r) continue;
                    DMat& Mq = gm(*d->ranks[q]);
                    const int cnt = Mr.recv_off[q + 1] - Mr.recv_off[q];
                    require(cnt == Mq.send_off[r + 1] - Mq.send_off[r], "dist: inconsistent halo plan");
                    if (!cnt) continue;
                    NK(N.send(Mq.send_buf.p + Mq.send_off[r], (size_t)cnt, ncclDouble, c->rank, comm, s));
                    NK(N.recv(dst + Mr.recv_off[q], (size_t)cnt, ncclDouble, c->rank, comm, s));
                }
            }
            NK(N.groupEnd());
            return;
        }
        for (int r = 0; r < d->R; ++r) {
            DMat& Mr = gm(*d->ranks[r]);
            double* dst = gv(*d->ranks[r]) + Mr.n_own;
            for (int q = 0; q < d->R; ++q) {
                if (q == r) continue;
                DMat& Mq = gm(*d->ranks[q]);
                const int cnt = Mr.recv_off[q + 1] - Mr.recv_off[q];
                require(cnt == Mq.send_off[r + 1] - Mq.send_off[r], "dist: inconsistent halo plan");
                d2d(c, dst + Mr.recv_off[q], Mq.send_buf.p + Mq.send_off[r], (size_t)cnt);
            }
        }
    } else {
        const auto& N = nccl_api();
        auto comm = static_cast<ncclComm_t>(c->nccl);
        RankData& rk = *d->ranks[0];
        DMat& M = gm(rk);
        double* dst = gv(rk) + M.n_own;
        NK(N.groupStart());
        for (int q = 0; q < d->R; ++q) {
            if (q == rk.rank) continue;
            const int ns = M.send_off[q + 1] - M.send_off[q];
            const int nr = M.recv_off[q + 1] - M.recv_off[q];
            if (ns) NK(N.send(M.send_buf.p + M.send_off[q], (size_t)ns, ncclDouble, q, comm, s));
            if (nr) NK(N.recv(dst + M.recv_off[q], (size_t)nr, ncclDouble, q, comm, s));
        }
        NK(N.groupEnd());
    }
}

template <class GetV>
void allreduce(Dist* d, GetV gv, int n) {
    if (n == 0 || (d->loop && d->R == 1)) return;
    Ctx* c = d->c;
    if (d->loop) {
        RankPtrs P{};
        P.R = d->R;
        for (int r = 0; r < d->R; ++r) P.p[r] = gv(*d->ranks[r]);
        launch_elem(c, n, elem_grid(c, n), BodySumRanks{P}, c->stream);
    } else {
        double* buf = gv(*d->ranks[0]);
        NK(nccl_api().allReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, static_cast<ncclComm_t>(c->nccl),
                                c->stream));
    }
}

// Replicated tail: V-cycle from level D (full vectors, amg.cuh kernels) — b_in -> out.
void vcycle_from(Ctx* c, Hier* h, int D, const double* b_in, double* out, const int* done, cudaStream_t s) {
    const int L = h->active_levels();
    if (D == L) {
        coarse_solve(c, h, b_in, out, done, s);
        return;
    }
    for (int l = D; l < L; ++l) {
        Level& lv = *h->levels[l];
        const double* b = l == D ? b_in : lv.b.p;
        if (l == D)
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
    coarse_solve(c, h, h->cb.p, h->cx.p, done, s);
    for (int l = L - 1; l >= D; --l) {
        Level& lv = *h->levels[l];
        const double* b = l == D ? b_in : lv.b.p;
        const double* ec = l + 1 < L ? h->levels[l + 1]->xo.p : h->cx.p;
        launch_spmv(c, lv.P, XPlain{ec}, EpiAddInPlace{lv.x.p, done}, s);
        launch_spmv(c, lv.A, XPlain{lv.x.p}, EpiPostSmooth{lv.wd.p, b, lv.x.p, l == D ? out : lv.xo.p, done}, s);
    }
}

// SpMV with a fused reduction into rk.red; a rank without rows contributes zeros
template <class XF, class Epi>
void spmv_red(Ctx* c, const Mat* M, double* red, XF xf, Epi epi, cudaStream_t s) {
    if (M->rows == 0) {
        CK(cudaMemsetAsync(red, 0, sizeof(double) * Epi::NR, s));
        return;
    }
    launch_spmv(c, M, xf, epi, s);
}

// level l's restriction feeds the replicated part
inline bool rk_switch(const Dist* d, int l) { return l == d->D - 1; }

// One distributed V(1,1) cycle z = M^{-1} r on every local rank.
void dist_vcycle(Dist* d) {
    Ctx* c = d->c;
    cudaStream_t s = c->stream;
    const int D = d->D;
    for (int l = 0; l < D; ++l) {
        auto bvec = [l](RankData& rk) -> double* { return l == 0 ? rk.r.p : rk.lev[l]->b.p; };
        exchange(d, [l](RankData& rk) -> DMat& { return rk.lev[l]->A; }, bvec);
        for (auto& rk : d->ranks) {
            DLev& L = *rk->lev[l];
            const int* done = &rk->st.p->done;
            launch_spmv(c, L.A.m, XJacobi{L.wd.p, bvec(*rk)}, EpiJacobiResidual{L.wd.p, bvec(*rk), L.x.p, L.r.p, done},
                        s);
        }
        if (!rk_switch(d, l)) {
            exchange(d, [l](RankData& rk) -> DMat& { return rk.lev[l]->Pt; }, [l](RankData& rk) { return rk.lev[l]->r.p; });
            for (auto& rk : d->ranks) {
                DLev& L = *rk->lev[l];
                launch_spmv(c, L.Pt.m, XPlain{L.r.p}, EpiStoreSkip{rk->lev[l + 1]->b.p, &rk->st.p->done}, s);
            }
        } else {
            for (auto& rk : d->ranks) {
                DLev& L = *rk->lev[l];
                launch_spmv(c, L.Pt.m, XPlain{L.r.p}, EpiStoreSkip{rk->bD.p, &rk->st.p->done}, s);
            }
            allreduce(d, [](RankData& rk) { return rk.bD.p; }, (int)d->ranks[0]->bD.n);
        }
    }
    for (auto& rk : d->ranks) vcycle_from(c, d->h, D, rk->bD.p, rk->xD.p, &rk->st.p->done, s);
    for (int l = D - 1; l >= 0; --l) {
        if (!rk_switch(d, l)) {
            exchange(d, [l](RankData& rk) -> DMat& { return rk.lev[l]->P; },
                     [l](RankData& rk) { return rk.lev[l + 1]->xo.p; });
        }
        for (auto& rk : d->ranks) {
            DLev& L = *rk->lev[l];
            const double* ec = rk_switch(d, l) ? rk->xD.p : rk->lev[l + 1]->xo.p;
            launch_spmv(c, L.P.m, XPlain{ec}, EpiAddInPlace{L.x.p, &rk->st.p->done}, s);
        }
        exchange(d, [l](RankData& rk) -> DMat& { return rk.lev[l]->A; }, [l](RankData& rk) { return rk.lev[l]->x.p; });
        for (auto& rk : d->ranks) {
            DLev& L = *rk->lev[l];
            const int* done = &rk->st.p->done;
            if (l > 0) {
                launch_spmv(c, L.A.m, XPlain{L.x.p}, EpiPostSmooth{L.wd.p, L.b.p, L.x.p, L.xo.p, done}, s);
            } else {  // z (r.z is reduced with the next SpMV's sums)
                launch_spmv(c, L.A.m, XPlain{L.x.p}, EpiPostSmooth{L.wd.p, rk->r.p, L.x.p, rk->z.p, done}, s);
            }
        }
    }
}

}  // namespace
}  // namespace ibmgpu

// ---------------------------------------------------------------- one PCG iteration
namespace ibmgpu {
namespace {

void scal_all(Dist* d, int phase) {
    for (auto& rk : d->ranks) launch_k(d->c, k_dscal, 1, 1, d->c->stream, rk->st.p, (const double*)rk->red.p, phase);
}

// One iteration of the single-reduction PCG on every local rank; scalars stay on the device.
void enqueue_iteration(Dist* d) {
    Ctx* c = d->c;
    cudaStream_t s = c->stream;
    auto red = [](RankData& rk) { return rk.red.p; };
    auto rslot = [](RankData& rk) { return RedSlot{rk.partials.p, nullptr}; };
    if (d->kind == IBMGPU_PC_SA) {
        dist_vcycle(d);
    } else {
        for (auto& rk : d->ranks)
            if (rk->n_own)
                launch_elem(c, rk->n_own, elem_grid(c, rk->n_own), BodyDPrecond{rk->r.p, rk->invd.p, rk->z.p, rk->st.p},
                            s);
    }
    exchange(d, [](RankData& rk) -> DMat& { return rk.A; }, [](RankData& rk) { return rk.z.p; });
    for (auto& rk : d->ranks)
        spmv_red(c, rk->A.m, rk->red.p, XPlain{rk->z.p},
                 EpiDFused{rk->r.p, rk->z.p, rk->Ap.p, rk->w.p, rslot(*rk), rk->red.p, rk->st.p}, s);
    allreduce(d, red, 4);  // the iteration's only scalar collective
    scal_all(d, PH_FUSED);
    for (auto& rk : d->ranks)
        if (rk->n_own)
            launch_elem(c, rk->n_own, elem_grid(c, rk->n_own),
                        BodyDUpd{rk->x.p, rk->r.p, rk->p.p, rk->Ap.p, rk->z.p, rk->w.p, rk->st.p}, s);
}

void capture_iteration(Dist* d) {
    Ctx* c = d->c;
    const long long l0 = c->launches;
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
        enqueue_iteration(d);
    } catch (...) {  // leave the stream usable: end (and drop) the broken capture
        cudaStreamEndCapture(c->stream, &g);
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        c->launches = l0;
        throw;
    }
    CK(cudaStreamEndCapture(c->stream, &g));
    CK(cudaGraphInstantiate(&d->iter_exec, g, 0));
    CK(cudaGraphDestroy(g));
    d->iter_kernels = (int)(c->launches - l0);
    c->launches = l0;  // capture is not execution
}

}  // namespace
}  // namespace ibmgpu

// ---------------------------------------------------------------- setup
namespace ibmgpu {
namespace {

std::vector<double> download_vec(Ctx* c, const double* p, size_t n) {
    std::vector<double> h(n);
    d2h(c, h.data(), p, n);
    sync(c);
    return h;
}

// values of a full vector at the extended layout of a plan (own entries, then halo)
void upload_ext(Ctx* c, DBuf<double>& dst, const std::vector<double>& full, const ibmhost::DistPlan& P) {
    std::vector<double> e;
    e.reserve(P.own.size() + P.halo.size());
    for (int g : P.own) e.push_back(full[(size_t)g]);
    for (int g : P.halo) e.push_back(full[(size_t)g]);
    dst.alloc(c, std::max<size_t>(e.size(), 1));
    h2d(c, dst.p, e.data(), e.size());
}

ibmhost::DistPlan plan_of(const HostCsr& M, const std::vector<int>& ro, const std::vector<int>& co, int r, int R) {
    return ibmhost::make_dist_plan(M.rows, M.cols, M.rp.data(), M.ci.data(), M.v.data(), ro.data(), co.data(), r, R);
}

}  // namespace

Dist* dist_create(Ctx* c, Mat* A, int kind, Hier* h, const int* owner0, int virtual_ranks, int min_rows) {
    require(A->rows == A->cols, "dist: matrix must be square");
    require(kind >= 0 && kind <= 2, "dist: unknown preconditioner");
    require(kind != IBMGPU_PC_SA || h != nullptr, "dist: SA preconditioner needs a hierarchy");
    auto d = std::make_unique<Dist>();
    d->c = c;
    d->A = A;
    d->h = kind == IBMGPU_PC_SA ? h : nullptr;
    d->kind = kind;
    // a one-rank NCCL communicator with virtual ranks runs the loopback decomposition with its
    // halos moved by NCCL send/recv (the p2p path exercised on a single GPU)
    d->loop = c->nccl == nullptr || (c->nranks == 1 && virtual_ranks > 1);
    d->loop_nccl = d->loop && c->nccl != nullptr;
    d->R = d->loop ? std::max(1, virtual_ranks) : c->nranks;
    require(!d->loop || d->R <= kMaxLoop, "dist: at most 16 loopback ranks");
    const int R = d->R;
    const int n = A->rows;
    d->n = n;
    d->owner.emplace_back(owner0, owner0 + n);
    for (int o : d->owner[0]) require(o >= 0 && o < R, "dist: owner out of range");
    if (d->h) {
        const int L = h->active_levels();  // folded tail levels are part of the dense coarse solve
        if (L == 0) fail(IBMGPU_ESUPPORT, "dist: hierarchy has no levels to distribute");
        require(h->levels[0]->A->rows == n, "dist: hierarchy size does not match the matrix");
        int D = 0;
        while (D < L && h->levels[D]->A->rows >= min_rows) ++D;
        d->D = std::max(D, 1);
        for (int l = 0; l < d->D; ++l) {
            Level& lv = *h->levels[l];
            std::vector<int> agg((size_t)std::max(lv.n_core, 1));
            d2h(c, agg.data(), lv.agg.p, (size_t)lv.n_core);
            sync(c);
            d->owner.push_back(ibmhost::partition_coarse(d->owner[l], agg.data(), lv.n_core, lv.n_agg,
                                                         lv.A->rows - lv.n_core));
        }
    }
    // host copies of the operators (every rank holds the full ones)
    const HostCsr Ah = download(c, A);
    std::vector<HostCsr> Al, Pl, Ptl;
    std::vector<std::vector<double>> wdl;
    for (int l = 0; l < d->D; ++l) {
        Level& lv = *h->levels[l];
        Al.push_back(download(c, lv.A));
        Pl.push_back(download(c, lv.P));
        Ptl.push_back(download(c, lv.Pt));
        wdl.push_back(download_vec(c, lv.wd.p, (size_t)lv.A->rows));
    }
    std::vector<double> invd_full;
    if (kind == IBMGPU_PC_DIAGONAL) {
        DBuf<double> dg(c, (size_t)std::max(n, 1));
        diag_of(c, A, dg.p);
        invd_full = download_vec(c, dg.p, (size_t)n);
        for (double& v : invd_full) {
            if (v == 0.0) fail(IBMGPU_EINVAL, "diagonal preconditioner: zero diagonal entry");
            v = 1.0 / v;
        }
    }
    const int nD = d->h ? (d->D < h->active_levels() ? h->levels[d->D]->A->rows : h->n_dense) : 0;
    std::vector<int> local_ranks;
    if (d->loop)
        for (int r = 0; r < R; ++r) local_ranks.push_back(r);
    else
        local_ranks.push_back(c->rank);
    for (int r : local_ranks) {
        auto rk = std::make_unique<RankData>();
        rk->rank = r;
        const auto PA = plan_of(Ah, d->owner[0], d->owner[0], r, R);
        dmat_from_plan(c, rk->A, PA);
        rk->own0 = PA.own;
        rk->n_own = PA.n_own;
        const size_t no = (size_t)std::max(PA.n_own, 1);
        rk->own0_dev.alloc(c, no);
        h2d(c, rk->own0_dev.p, PA.own.data(), PA.own.size());
        rk->b.alloc(c, no);
        rk->z.alloc(c, no + (size_t)PA.n_halo());
        rk->Ap.alloc(c, no);
        rk->w.alloc(c, no);
        rk->x.alloc(c, no + (size_t)PA.n_halo());
        rk->p.alloc(c, no);
        if (kind == IBMGPU_PC_DIAGONAL) {
            std::vector<double> iv;
            for (int g : PA.own) iv.push_back(invd_full[(size_t)g]);
            rk->invd.alloc(c, no);
            h2d(c, rk->invd.p, iv.data(), iv.size());
        }
        int rcap = PA.n_own;
        int grid = std::max(spmv_grid(rk->A.m), elem_grid(c, PA.n_own));
        int prev_p_halo = 0;
        for (int l = 0; l < d->D; ++l) {
            auto L = std::make_unique<DLev>();
            const bool sw = l == d->D - 1;
            L->switch_below = sw;
            const auto PAl = plan_of(Al[l], d->owner[l], d->owner[l], r, R);
            dmat_from_plan(c, L->A, PAl);
            upload_ext(c, L->wd, wdl[l], PAl);
            int pt_halo = 0;
            if (!sw) {
                const auto PPt = plan_of(Ptl[l], d->owner[l + 1], d->owner[l], r, R);
                dmat_from_plan(c, L->Pt, PPt);
                pt_halo = PPt.n_halo();
                const auto PP = plan_of(Pl[l], d->owner[l], d->owner[l + 1], r, R);
                dmat_from_plan(c, L->P, PP);
            } else {
                L->Pt.m = colsplit(c, Ptl[l], d->owner[l], r);
                const std::vector<int> all_mine((size_t)Pl[l].cols, r);
                const auto PP = plan_of(Pl[l], d->owner[l], all_mine, r, R);
                dmat_from_plan(c, L->P, PP);
            }
            L->n_own = PAl.n_own;
            const size_t own = (size_t)std::max(PAl.n_own, 1);
            L->b.alloc(c, own + (size_t)PAl.n_halo());
            L->x.alloc(c, own + (size_t)PAl.n_halo());
            L->r.alloc(c, own + (size_t)pt_halo);
            L->xo.alloc(c, own + (size_t)prev_p_halo);
            prev_p_halo = L->P.n_halo;
            if (l == 0) rcap = std::max(rcap, PAl.n_own + PAl.n_halo());
            grid = std::max(grid, spmv_grid(L->A.m));
            rk->lev.push_back(std::move(L));
        }
        rk->r.alloc(c, (size_t)std::max(rcap, 1));
        if (d->h) {
            rk->bD.alloc(c, (size_t)nD);
            rk->xD.alloc(c, (size_t)nD);
        }
        rk->st.alloc(c, 1);
        rk->red.alloc(c, 4);
        rk->partials.alloc(c, (size_t)std::max(grid, 1) * 4);
        CK(cudaMallocHost(&rk->host_st, sizeof(PcgState)));
        d->ranks.push_back(std::move(rk));
    }
    CK(cudaMallocHost(&d->done_host, 2 * sizeof(int)));
    for (auto& e : d->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    sync(c);
    return d.release();
}

void dist_solve(Dist* d, const double* b_full, double* x_full, const ibm_solver_params& prm, ibm_solve_result* res,
                double* hist_host) {
    validate_params(prm);
    Ctx* c = d->c;
    cudaStream_t s = c->stream;
    if (d->n == 0) {
        if (res) *res = ibm_solve_result{0, 0.0, 0, 0};
        return;
    }
    DBuf<double> hist;
    if (prm.record_history) hist.alloc(c, (size_t)prm.max_iters + 1);
    for (auto& rk : d->ranks) {
        const int no = rk->n_own;
        if (no) {
            launch_elem(c, no, elem_grid(c, no), BodyPack{rk->own0_dev.p, b_full, rk->b.p}, s);
            launch_elem(c, no, elem_grid(c, no), BodyPack{rk->own0_dev.p, x_full, rk->x.p}, s);
        }
        PcgState& H = *rk->host_st;
        H = PcgState{};
        H.rel_tol = prm.rel_tol;
        H.max_iters = prm.max_iters;
        H.hist = rk == d->ranks[0] ? hist.p : nullptr;
        CK(cudaMemcpyAsync(rk->st.p, &H, sizeof(PcgState), cudaMemcpyHostToDevice, s));
    }
    auto red = [](RankData& rk) { return rk.red.p; };
    auto rslot = [](RankData& rk) { return RedSlot{rk.partials.p, nullptr}; };
    for (auto& rk : d->ranks)
        if (rk->n_own) {  // the recurrence reads p and Ap of "iteration -1" with beta = 0
            CK(cudaMemsetAsync(rk->p.p, 0, sizeof(double) * (size_t)rk->n_own, s));
            CK(cudaMemsetAsync(rk->Ap.p, 0, sizeof(double) * (size_t)rk->n_own, s));
        }
    // r = b - A x0
    exchange(d, [](RankData& rk) -> DMat& { return rk.A; }, [](RankData& rk) { return rk.x.p; });
    for (auto& rk : d->ranks)
        spmv_red(c, rk->A.m, rk->red.p, XPlain{rk->x.p}, EpiDInit{rk->b.p, rk->r.p, rslot(*rk), rk->red.p}, s);
    allreduce(d, red, 2);
    scal_all(d, PH_INIT);
    for (auto& rk : d->ranks)
        if (rk->n_own) launch_elem(c, rk->n_own, elem_grid(c, rk->n_own), BodyDZeroX{rk->x.p, rk->st.p}, s);
    PcgState* H0 = d->ranks[0]->host_st;
    CK(cudaMemcpyAsync(H0, d->ranks[0]->st.p, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    sync(c);
    if (!H0->done) {
        if (!c->eager && !d->iter_exec && !d->no_graph) {
            try {
                capture_iteration(d);
            } catch (const Error&) {
                d->no_graph = true;  // e.g. a communicator that cannot be captured: run eagerly
            }
        }
        if (c->eager || d->no_graph) {
            // profiling mode (IBMGPU_EAGER=1): kernels launched from the host, checked every iteration
            for (;;) {
                enqueue_iteration(d);
                CK(cudaMemcpyAsync(H0, d->ranks[0]->st.p, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
                sync(c);
                if (H0->done) break;
            }
        } else {
            // one graph launch per iteration (NCCL calls captured with the kernels); the done flag
            // of iteration k is read while iteration k+1 is already queued, so the GPU never idles
            // on the host check — the extra iteration's kernels see `done` and exit at once
            const int* done_dev = &d->ranks[0]->st.p->done;
            for (int k = 0;; ++k) {
                CK(cudaGraphLaunch(d->iter_exec, s));
                c->launches += d->iter_kernels;
                CK(cudaMemcpyAsync(d->done_host + (k & 1), done_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
                CK(cudaEventRecord(d->ev[k & 1], s));
                if (k > 0) {
                    CK(cudaEventSynchronize(d->ev[(k - 1) & 1]));
                    if (d->done_host[(k - 1) & 1]) break;
                }
                require(k <= prm.max_iters + 2, "dist: iteration loop did not terminate");
            }
        }
    }
    // x (owned rows) back into the full vector on every rank
    if (d->loop) {
        for (auto& rk : d->ranks)
            if (rk->n_own)
                launch_elem(c, rk->n_own, elem_grid(c, rk->n_own), BodyScatter{rk->own0_dev.p, rk->x.p, x_full}, s);
    } else {
        RankData& rk = *d->ranks[0];
        CK(cudaMemsetAsync(x_full, 0, sizeof(double) * (size_t)d->n, s));
        if (rk.n_own) launch_elem(c, rk.n_own, elem_grid(c, rk.n_own), BodyScatter{rk.own0_dev.p, rk.x.p, x_full}, s);
        NK(nccl_api().allReduce(x_full, x_full, (size_t)d->n, ncclDouble, ncclSum, static_cast<ncclComm_t>(c->nccl), s));
    }
    CK(cudaMemcpyAsync(H0, d->ranks[0]->st.p, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    sync(c);
    if (res) {
        res->iterations = H0->iterations;
        res->rel_residual = H0->rel;
        res->status = H0->status;
        res->history_len = H0->hist_len;
    }
    if (prm.record_history && hist_host && res) d2h(c, hist_host, hist.p, (size_t)res->history_len), sync(c);
}

void dist_info(const Dist* d, int* info8) {
    const RankData& rk = *d->ranks[0];
    info8[0] = d->R;
    info8[1] = d->D;
    info8[2] = d->loop_nccl ? 2 : d->loop ? 1 : 0;
    info8[3] = rk.n_own;
    info8[4] = rk.A.n_halo;
    info8[5] = (int)d->ranks.size();
    info8[6] = d->h ? (int)d->h->levels.size() : 0;
    info8[7] = rk.A.m ? rk.A.m->kind : -1;
}

}  // namespace ibmgpu

namespace ibmgpu {
Ctx* dist_ctx(const Dist* d) { return d->c; }
void dist_destroy(Dist* d) {
    if (!d) return;
    sync(d->c);
    delete d;
}
}  // namespace ibmgpu
