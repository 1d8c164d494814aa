// capi.cu — extern "C" entry points of include/ibmgpu.h (context, memory, CSR, solvers).
// Every call is wrapped so that C++ exceptions become IBMGPU_E* codes + ibmgpu_last_error().
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "amg.cuh"
#include "dist.cuh"
#include "internal.cuh"
#include "kern.cuh"
#include "pcg.cuh"

using namespace ibmgpu;

namespace {
thread_local std::string g_noctx_err;

template <class F>
int guard(ibmgpu_ctx* c, F&& f) {
    try {
        f();
        return IBMGPU_OK;
    } catch (const Error& e) {
        (c ? c->err : g_noctx_err) = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        (c ? c->err : g_noctx_err) = "out of host memory";
        return IBMGPU_ENOMEM;
    } catch (const std::exception& e) {
        (c ? c->err : g_noctx_err) = e.what();
        return IBMGPU_ECUDA;
    }
}
void need(bool ok, const char* what) {
    if (!ok) fail(IBMGPU_EINVAL, what);
}
}  // namespace

namespace ibmgpu {
void ctx_free_extras(Ctx* c);  // stepper.cu / dist hooks
}

extern "C" {

const char* ibmgpu_version(void) { return "ibmgpu 0.1 (sm_100a)"; }

int ibmgpu_init(int device, int nranks, int rank, const void* nccl_id, ibmgpu_ctx_t* out) {
    auto* c = new ibmgpu_ctx();
    const int rc = guard(nullptr, [&] {
        need(out != nullptr, "init: null output");
        need(nranks >= 1 && rank >= 0 && rank < nranks, "init: bad rank/nranks");
        c->device = device;
        c->nranks = nranks;
        c->rank = rank;
        CK(cudaSetDevice(device));
        // the solve stream at the highest priority: the stepper's operator-pipeline workers (lowest
        // priority streams) then fill only the SMs the solves leave idle
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi));
        CK(cudaEventCreate(&c->t0));
        CK(cudaEventCreate(&c->t1));
        CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
        const char* eg = std::getenv("IBMGPU_EAGER");
        c->eager = eg && eg[0] == '1';
        // A private stream-ordered pool: freed blocks stay cached for the context's own reuse, and
        // nothing process-wide (the device's default pool, other allocators) is touched.
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        CK(cudaMemPoolCreate(&c->pool, &props));
        unsigned long long thr = ~0ull;  // keep freed blocks cached in this pool
        CK(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr));
        // Pre-map part of the pool for the first context on a device: the SpGEMM sort buffers of
        // a hierarchy rebuild (up to ~2 GB at 600k rows) otherwise map fresh pages mid-setup,
        // which made identical rebuilds vary 65-500 ms (IBMGPU_POOL_RESERVE_MB, default 8192;
        // 0 disables). The once-per-device claim is an atomic exchange (thread-safe).
        static std::atomic<bool> reserved[64] = {};
        const char* rv = std::getenv("IBMGPU_POOL_RESERVE_MB");
        const size_t mb = rv ? std::strtoull(rv, nullptr, 10) : 8192;
        if (mb && device >= 0 && device < 64 && !reserved[device].exchange(true)) {
            size_t free_b = 0, total_b = 0;
            CK(cudaMemGetInfo(&free_b, &total_b));
            const size_t want = std::min(mb << 20, free_b / 4);
            void* p = nullptr;
            if (cudaMallocFromPoolAsync(&p, want, c->pool, c->stream) == cudaSuccess) {
                CK(cudaFreeAsync(p, c->stream));
                CK(cudaStreamSynchronize(c->stream));
            } else {
                cudaGetLastError();
            }
        }
        need(nranks == 1 || nccl_id != nullptr, "init: multi-rank context needs an NCCL unique id");
        // nranks == 1 with an id: a one-rank NCCL communicator (exercises the NCCL code path)
        if (nranks > 1 || nccl_id) nccl_comm_init(c, nccl_id);
    });
    if (rc) {
        if (out) *out = nullptr;
        delete c;
        return rc;
    }
    *out = c;
    return 0;
}

int ibmgpu_destroy(ibmgpu_ctx_t c) {
    if (!c) return 0;
    cudaStreamSynchronize(c->stream);
    pcg_cache_free(c);
    zero_scratch_free(c);
    ctx_free_extras(c);
    nccl_comm_free(c);
    cudaEventDestroy(c->t0);
    cudaEventDestroy(c->t1);
    cudaStreamDestroy(c->stream);
    if (c->pool) cudaMemPoolDestroy(c->pool);  // released once its last allocation is freed
    delete c;
    return 0;
}

const char* ibmgpu_last_error(ibmgpu_ctx_t c) { return c ? c->err.c_str() : g_noctx_err.c_str(); }

int ibmgpu_synchronize(ibmgpu_ctx_t c) {
    return guard(c, [&] { sync(c); });
}

int ibmgpu_vec_alloc(ibmgpu_ctx_t c, size_t n, double** dev) {
    return guard(c, [&] {
        CK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(dev), sizeof(double) * (n ? n : 1), c->pool, c->stream));
        CK(cudaMemsetAsync(*dev, 0, sizeof(double) * (n ? n : 1), c->stream));
    });
}
int ibmgpu_vec_free(ibmgpu_ctx_t c, double* dev) {
    return guard(c, [&] {
        if (dev) CK(cudaFreeAsync(dev, c->stream));
    });
}
int ibmgpu_h2d(ibmgpu_ctx_t c, double* dev, const double* host, size_t n) {
    return guard(c, [&] {
        h2d(c, dev, host, n);
        sync(c);
    });
}
int ibmgpu_d2h(ibmgpu_ctx_t c, double* host, const double* dev, size_t n) {
    return guard(c, [&] {
        d2h(c, host, dev, n);
        sync(c);
    });
}
int ibmgpu_timer_start(ibmgpu_ctx_t c) {
    return guard(c, [&] { CK(cudaEventRecord(c->t0, c->stream)); });
}
int ibmgpu_timer_stop(ibmgpu_ctx_t c, float* ms) {
    return guard(c, [&] {
        CK(cudaEventRecord(c->t1, c->stream));
        CK(cudaEventSynchronize(c->t1));
        CK(cudaEventElapsedTime(ms, c->t0, c->t1));
    });
}
int ibmgpu_launch_count(ibmgpu_ctx_t c, long long* n) {
    *n = c->launches;
    return 0;
}

// ---------------------------------------------------------------- CSR
int ibmgpu_csr_upload(ibmgpu_ctx_t c, int rows, int cols, int nnz, const int* rp, const int* ci, const double* v,
                      ibmgpu_mat_t* out) {
    return guard(c, [&] {
        need(out && rp, "csr_upload: null argument");
        *out = mat_upload(c, rows, cols, nnz, rp, ci, v);
    });
}

int ibmgpu_csr_from_triplets(ibmgpu_ctx_t c, int rows, int cols, int n, const int* r, const int* cc, const double* v,
                             ibmgpu_mat_t* out) {
    return guard(c, [&] {
        need(out && n >= 0, "from_triplets: bad argument");
        DBuf<int> dr(c, (size_t)n), dc(c, (size_t)n);
        DBuf<double> dv(c, (size_t)n);
        h2d(c, dr.p, r, (size_t)n);
        h2d(c, dc.p, cc, (size_t)n);
        h2d(c, dv.p, v, (size_t)n);
        *out = from_triplets(c, rows, cols, (size_t)n, dr.p, dc.p, dv.p);
    });
}

int ibmgpu_csr_info(ibmgpu_mat_t m, int* rows, int* cols, int* nnz) {
    if (!m) return IBMGPU_EINVAL;
    if (rows) *rows = m->rows;
    if (cols) *cols = m->cols;
    if (nnz) *nnz = m->nnz;
    return 0;
}

int ibmgpu_csr_format_bytes(ibmgpu_ctx_t c, ibmgpu_mat_t m, long long* bytes, int* kind) {
    return guard(c, [&] {
        need(m && bytes, "csr_format_bytes: null argument");
        if (!m->planned) mat_plan(c, m);
        const long long n = m->rows, cols = m->cols;
        long long b = 8 * cols + 8 * n;  // x gathered once, y written once
        switch (m->kind) {
            case SPMV_STENCIL:  // 5 band planes + mask byte per row, CSR tail (row ptr + entries)
                b += 41 * n + 4 * (n + 1) + 12 * (long long)m->st_eci.n;
                break;
            case SPMV_SELL:  // padded 32-row slices (16- or 32-bit columns) + slice offsets + row lengths
                b += (m->c16 ? 10 : 12) * (long long)m->sell_v.n + 4 * (long long)m->sell_off.n + 4 * (n + 1) +
                     4 * (long long)m->sell_cbase.n;
                break;
            case SPMV_SELLW:  // SELL-sigma slices + slot->row permutation + long rows in CSR
                b += (m->c16 ? 10 : 12) * (long long)m->sell_v.n + 4 * (long long)m->sell_off.n +
                     4 * (long long)m->perm.n + 4 * (n + 1) + 4 * (long long)m->sell_cbase.n;
                break;
            default:  // CSR-adaptive: the CSR itself + chunk metadata
                b += 12 * (long long)m->nnz + 4 * (n + 1) + 16 * (long long)m->n_blocks;
                break;
        }
        *bytes = b;
        if (kind) *kind = m->kind | (m->c16 ? 16 : 0);
    });
}

int ibmgpu_csr_download(ibmgpu_ctx_t c, ibmgpu_mat_t m, int* rp, int* ci, double* v) {
    return guard(c, [&] {
        need(m != nullptr, "csr_download: null matrix");
        mat_download(c, m, rp, ci, v);
    });
}

int ibmgpu_csr_destroy(ibmgpu_ctx_t c, ibmgpu_mat_t m) {
    return guard(c, [&] {
        if (!m) return;
        need(!m->borrowed, "csr_destroy: matrix is owned by a hierarchy or stepper");
        pcg_forget(c, m, nullptr);
        delete m;
    });
}

int ibmgpu_spmv(ibmgpu_ctx_t c, ibmgpu_mat_t A, const double* x, double* y) {
    return guard(c, [&] {
        need(A && x && y, "spmv: null argument");
        spmv(c, A, x, y);
    });
}

int ibmgpu_spmv_timed(ibmgpu_ctx_t c, ibmgpu_mat_t A, const double* x, double* y, int reps, double* us) {
    return guard(c, [&] {
        need(A && x && y && us && reps > 0, "spmv_timed: bad argument");
        if (!A->planned) mat_plan(c, A);
        spmv(c, A, x, y);  // warm: plan buffers, instruction cache
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < reps; ++i) spmv(c, A, x, y);
        CK(cudaStreamEndCapture(c->stream, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaGraphLaunch(ge, c->stream));
        CK(cudaEventRecord(e0, c->stream));
        CK(cudaGraphLaunch(ge, c->stream));
        CK(cudaEventRecord(e1, c->stream));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        *us = 1e3 * ms / reps;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
    });
}

int ibmgpu_spmv_host(ibmgpu_ctx_t c, ibmgpu_mat_t A, const double* x, double* y) {
    return guard(c, [&] {
        need(A != nullptr, "spmv: null matrix");
        DBuf<double> dx(c, (size_t)A->cols), dy(c, (size_t)A->rows);
        h2d(c, dx.p, x, (size_t)A->cols);
        spmv(c, A, dx.p, dy.p);
        d2h(c, y, dy.p, (size_t)A->rows);
        sync(c);
    });
}

int ibmgpu_transpose(ibmgpu_ctx_t c, ibmgpu_mat_t A, ibmgpu_mat_t* out) {
    return guard(c, [&] { *out = transpose(c, A); });
}
int ibmgpu_spmm(ibmgpu_ctx_t c, ibmgpu_mat_t A, ibmgpu_mat_t B, ibmgpu_mat_t* out) {
    return guard(c, [&] { *out = spmm_rows(c, A, 0, A->rows, B); });
}
int ibmgpu_triple_product(ibmgpu_ctx_t c, ibmgpu_mat_t A, ibmgpu_mat_t B, ibmgpu_mat_t C, int slice,
                          ibmgpu_mat_t* out, long long* peak, int* slices) {
    return guard(c, [&] { *out = triple_product(c, A, B, C, slice, peak, slices); });
}
int ibmgpu_add(ibmgpu_ctx_t c, double a, ibmgpu_mat_t A, double b, ibmgpu_mat_t B, ibmgpu_mat_t* out) {
    return guard(c, [&] { *out = add(c, a, A, b, B); });
}
int ibmgpu_symmetrized(ibmgpu_ctx_t c, ibmgpu_mat_t A, ibmgpu_mat_t* out) {
    return guard(c, [&] { *out = symmetrized(c, A); });
}
int ibmgpu_pin(ibmgpu_ctx_t c, ibmgpu_mat_t A, int p, ibmgpu_mat_t* out) {
    return guard(c, [&] { *out = pin(c, A, p); });
}
int ibmgpu_is_symmetric(ibmgpu_ctx_t c, ibmgpu_mat_t A, double tol, int* result) {
    return guard(c, [&] { *result = is_symmetric(c, A, tol) ? 1 : 0; });
}
int ibmgpu_scale(ibmgpu_ctx_t c, ibmgpu_mat_t A, int mode, double a, const double* d_host, ibmgpu_mat_t* out) {
    return guard(c, [&] {
        need(mode >= 0 && mode <= 2, "scale: bad mode");
        DBuf<double> d;
        if (mode) {
            need(d_host != nullptr, "scale: missing vector");
            const size_t n = (size_t)(mode == 1 ? A->rows : A->cols);
            d.alloc(c, n);
            h2d(c, d.p, d_host, n);
        }
        *out = scale(c, A, mode, a, d.p);
    });
}

// ---------------------------------------------------------------- solvers
int ibmgpu_pcg(ibmgpu_ctx_t c, ibmgpu_mat_t A, int precond, ibmgpu_hier_t h, const double* b, double* x,
               const ibm_solver_params* prm, ibm_solve_result* res, double* hist) {
    return guard(c, [&] {
        need(A && b && x && prm, "pcg: null argument");
        pcg_solve(c, A, precond, h, b, x, *prm, res, hist);
    });
}

int ibmgpu_pcg_callback(ibmgpu_ctx_t c, ibmgpu_mat_t A, ibmgpu_apply_fn apply, void* user, const double* b,
                        double* x, const ibm_solver_params* prm, ibm_solve_result* res, double* hist) {
    return guard(c, [&] {
        need(A && b && x && prm, "pcg: null argument");
        pcg_callback(c, A, apply, user, b, x, *prm, res, hist);
    });
}

int ibmgpu_sa_build(ibmgpu_ctx_t c, ibmgpu_mat_t A, const ibm_sa_options* o, ibmgpu_hier_t* out) {
    return guard(c, [&] {
        need(A && o && out, "sa_build: null argument");
        *out = sa_build(c, A, *o);
    });
}

int ibmgpu_sa_destroy(ibmgpu_ctx_t c, ibmgpu_hier_t h) {
    return guard(c, [&] {
        if (!h) return;
        sync(c);
        pcg_forget(c, nullptr, h);
        delete h;
    });
}

int ibmgpu_sa_apply(ibmgpu_ctx_t c, ibmgpu_hier_t h, const double* r, double* z) {
    return guard(c, [&] {
        need(h && r && z, "sa_apply: null argument");
        vcycle_launch(c, h, r, z, nullptr, LastPlain{c, nullptr, c->stream}, c->stream);
    });
}

int ibmgpu_hier_info(ibmgpu_hier_t h, int* n_levels, int* stalled, int* coarse_rows) {
    if (!h) return IBMGPU_EINVAL;
    if (n_levels) *n_levels = (int)h->levels.size();
    if (stalled) *stalled = h->stalled ? 1 : 0;
    if (coarse_rows) *coarse_rows = h->n_c;
    return 0;
}

int ibmgpu_hier_folded(ibmgpu_hier_t h, int* n_fold, int* dense_rows) {
    if (!h) return IBMGPU_EINVAL;
    if (n_fold) *n_fold = h->n_fold;
    if (dense_rows) *dense_rows = h->n_dense;
    return 0;
}

int ibmgpu_hier_transfers(ibmgpu_ctx_t c, ibmgpu_hier_t h, int mode, int* active) {
    return guard(c, [&] {
        need(h != nullptr, "hier_transfers: null hierarchy");
        if (mode == 0) h->x0.on = false;
        if (mode == 1 && !h->x0.on) xfer0_setup(c, h);
        if (active) *active = h->x0.on ? 1 : 0;
    });
}

int ibmgpu_hier_level(ibmgpu_hier_t h, int l, ibmgpu_mat_t* A, ibmgpu_mat_t* P, ibmgpu_mat_t* Pt, double* omega) {
    if (!h || l < 0 || l > (int)h->levels.size()) return IBMGPU_EINVAL;
    if (l == (int)h->levels.size()) {
        h->coarse_A->borrowed = true;
        if (A) *A = h->coarse_A;
        if (P) *P = nullptr;
        if (Pt) *Pt = nullptr;
        if (omega) *omega = 0.0;
        return 0;
    }
    Level& lv = *h->levels[l];
    lv.A->borrowed = lv.P->borrowed = lv.Pt->borrowed = true;
    if (A) *A = lv.A;
    if (P) *P = lv.P;
    if (Pt) *Pt = lv.Pt;
    if (omega) *omega = lv.omega;
    return 0;
}

int ibmgpu_hier_aggregates(ibmgpu_ctx_t c, ibmgpu_hier_t h, int l, int* agg_host, int* n_agg) {
    return guard(c, [&] {
        need(h && l >= 0 && l < (int)h->levels.size(), "hier_aggregates: bad level");
        Level& lv = *h->levels[l];
        if (agg_host) d2h(c, agg_host, lv.agg.p, (size_t)lv.n_core);
        sync(c);
        if (n_agg) *n_agg = lv.n_agg;
    });
}

int ibmgpu_aggregate(ibmgpu_ctx_t c, ibmgpu_mat_t A, double theta, int n_core, int* agg_host, int* n_agg) {
    return guard(c, [&] {
        need(A && n_core >= 0 && n_core <= A->rows, "aggregate: bad argument");
        DBuf<int> agg;
        const int n = aggregate_device(c, A, theta, n_core, agg);
        if (agg_host) d2h(c, agg_host, agg.p, (size_t)n_core);
        sync(c);
        if (n_agg) *n_agg = n;
    });
}

}  // extern "C"

namespace ibmgpu {
void amg_solve(Ctx* c, Mat* A, Hier* h, const double* b, double* x, const ibm_solver_params& prm,
               ibm_solve_result* res);
}
extern "C" int ibmgpu_amg_solve(ibmgpu_ctx_t c, ibmgpu_mat_t A, ibmgpu_hier_t h, const double* b, double* x,
                                const ibm_solver_params* prm, ibm_solve_result* res) {
    return guard(c, [&] {
        need(A && h && b && x && prm, "amg_solve: null argument");
        amg_solve(c, A, h, b, x, *prm, res);
    });
}

// ---------------------------------------------------------------- row-slab multi-GPU (dist.cu)
extern "C" {

int ibmgpu_nccl_unique_id(void* id128) {
    return guard(nullptr, [&] {
        need(id128 != nullptr, "nccl_unique_id: null output");
        nccl_unique_id(id128);
    });
}

int ibmgpu_dist_create(ibmgpu_ctx_t c, ibmgpu_mat_t A, int precond, ibmgpu_hier_t hier, const int* owner,
                       int virtual_ranks, int min_dist_rows, ibmgpu_dist_t* out) {
    return guard(c, [&] {
        need(A && owner && out, "dist_create: null argument");
        need(!c->nccl || c->nranks == 1 || virtual_ranks <= 1, "dist_create: virtual ranks need a single-rank context");
        *out = dist_create(c, A, precond, hier, owner, virtual_ranks, min_dist_rows);
    });
}

int ibmgpu_dist_info(ibmgpu_dist_t d, int* info8) {
    if (!d || !info8) return IBMGPU_EINVAL;
    dist_info(d, info8);
    return 0;
}

int ibmgpu_dist_pcg(ibmgpu_dist_t d, const double* b_dev, double* x_dev, const ibm_solver_params* prm,
                    ibm_solve_result* res, double* history_host) {
    if (!d) return IBMGPU_EINVAL;
    Ctx* c = dist_ctx(d);
    return guard(c, [&] {
        need(b_dev && x_dev && prm, "dist_pcg: null argument");
        dist_solve(d, b_dev, x_dev, *prm, res, history_host);
    });
}

int ibmgpu_dist_destroy(ibmgpu_dist_t d) {
    if (!d) return 0;
    Ctx* c = dist_ctx(d);
    return guard(c, [&] { dist_destroy(d); });
}

}  // extern "C"
