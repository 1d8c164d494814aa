// internal.cuh — shared internals of libibmgpu (context, memory, device CSR, errors).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ibmgpu.h"

namespace ibmgpu {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool ok, const std::string& msg) {
    if (!ok) fail(IBMGPU_EINVAL, msg);
}

#define CK(call)                                                                                        \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess)                                                                          \
            ::ibmgpu::fail(e_ == cudaErrorMemoryAllocation ? IBMGPU_ENOMEM : IBMGPU_ECUDA,               \
                           std::string(#call) + ": " + cudaGetErrorString(e_) + " (" + __FILE__ + ":" +   \
                               std::to_string(__LINE__) + ")");                                         \
    } while (0)

// Every plain <<<>>> launch goes through CK_LAUNCH, which raises the context's PDL fence: the
// next launch_k (kern.cuh) then runs without programmatic stream serialization. Plain launches
// are where matrices and plans get written (assembly, SpGEMM, plan fills), and the PDL SpMV
// kernels read their constant matrix BEFORE griddepcontrol.wait — the fence guarantees they
// never overlap the kernel that wrote it.
#define CK_LAUNCH(ctx)                 \
    do {                               \
        CK(cudaGetLastError());        \
        ++(ctx)->launches;             \
        (ctx)->pdl_fence = 1;          \
    } while (0)

}  // namespace ibmgpu

struct ibmgpu_ctx {
    int device = 0;
    int nranks = 1, rank = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    std::string err;
    long long launches = 0;
    int num_sms = 148;
    void* nccl = nullptr;       // ncclComm_t when nranks > 1
    void* pcg_cache = nullptr;  // pcg.cu plan cache
    int eager = 0;              // IBMGPU_EAGER=1: host-looped solves (profiling only)
    int pdl_fence = 0;          // set by plain launches: the next launch_k skips PDL (CK_LAUNCH)
    cudaMemPool_t pool = nullptr;  // the context's own stream-ordered pool (capi.cu ibmgpu_init)
    // zero-filled scratch kept across calls (sparse_ops.cu windowed dense SpGEMM: its kernels leave
    // it zero again), so no call allocates and clears hundreds of MB; freed with the context
    void* zscratch = nullptr;
    size_t zscratch_bytes = 0;
};

namespace ibmgpu {

using Ctx = ibmgpu_ctx;

// Stream-ordered device buffer (cudaMallocAsync on the context's pool).
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(Ctx* c, size_t count) { alloc(c, count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr, o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p, n = o.n, s = o.s;
            o.p = nullptr, o.n = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(Ctx* c, size_t count) {
        release();
        s = c->stream;
        n = count;
        if (count) {
            if (c->pool)
                CK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, c->pool, s));
            else
                CK(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, s));
        }
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
    operator T*() const { return p; }
};

template <class T>
inline void h2d(Ctx* c, T* dst, const T* src, size_t n) {
    if (n) CK(cudaMemcpyAsync(dst, src, sizeof(T) * n, cudaMemcpyHostToDevice, c->stream));
}
template <class T>
inline void d2h(Ctx* c, T* dst, const T* src, size_t n) {
    if (n) CK(cudaMemcpyAsync(dst, src, sizeof(T) * n, cudaMemcpyDeviceToHost, c->stream));
}
template <class T>
inline void d2d(Ctx* c, T* dst, const T* src, size_t n) {
    if (n) CK(cudaMemcpyAsync(dst, src, sizeof(T) * n, cudaMemcpyDeviceToDevice, c->stream));
}
inline void sync(Ctx* c) { CK(cudaStreamSynchronize(c->stream)); }

// The context's zero-filled scratch, grown (and cleared once) when a call needs more.
inline void* zero_scratch(Ctx* c, size_t bytes) {
    if (bytes > c->zscratch_bytes) {
        if (c->zscratch) CK(cudaFreeAsync(c->zscratch, c->stream));
        c->zscratch = nullptr;
        c->zscratch_bytes = 0;
        CK(cudaMallocFromPoolAsync(&c->zscratch, bytes, c->pool, c->stream));
        CK(cudaMemsetAsync(c->zscratch, 0, bytes, c->stream));
        c->zscratch_bytes = bytes;
    }
    return c->zscratch;
}
inline void zero_scratch_free(Ctx* c) {
    if (c->zscratch) cudaFreeAsync(c->zscratch, c->stream);
    c->zscratch = nullptr;
    c->zscratch_bytes = 0;
}

// A kernel's dynamic shared-memory limit, raised once to the device's opt-in maximum (minus its
// static shared memory). Setting it per launch to that launch's size races when two host threads
// (the stepper's operator-pipeline workers) launch the same kernel with different sizes.
template <class K>
inline void smem_optin_once(std::once_flag& f, K kernel, int device) {
    std::call_once(f, [&] {
        int mx = 0;
        CK(cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        cudaFuncAttributes fa{};
        CK(cudaFuncGetAttributes(&fa, kernel));
        CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx - (int)fa.sharedSizeBytes));
    });
}
#define IBM_SMEM_OPTIN(c, kernel)                                 \
    do {                                                          \
        static std::once_flag ibm_smem_flag_;                     \
        ::ibmgpu::smem_optin_once(ibm_smem_flag_, kernel, (c)->device); \
    } while (0)

template <class T>
inline T d2h_scalar(Ctx* c, const T* src) {
    T v;
    d2h(c, &v, src, 1);
    sync(c);
    return v;
}

// SpMV execution plan chosen at construction from the row-length profile.
enum SpmvKind { SPMV_SELL = 0, SPMV_VECTOR = 1, SPMV_SELLW = 2, SPMV_STENCIL = 3 };

}  // namespace ibmgpu

// Device CSR (sparse.hpp:214-219 layout: int32 row_ptr/col_idx, f64 values) plus the
// SpMV-side SELL-32 copy (column-major within 32-row slices, padded to the slice width).
struct ibmgpu_mat {
    int rows = 0, cols = 0, nnz = 0;
    ibmgpu::DBuf<int> rp, ci;
    ibmgpu::DBuf<double> v;
    // SpMV plan
    int kind = ibmgpu::SPMV_SELL;
    int tpr = 1;  // threads per row (vector kind)
    int max_row = 0;
    ibmgpu::DBuf<int> sell_off;  // n_slices + 1 element offsets
    ibmgpu::DBuf<int> sell_ci;
    ibmgpu::DBuf<double> sell_v;
    // 16-bit column codes (csr.cu try_c16): code < 0x8000 -> slice base + code, else
    // c16_tail0 + code - 0x8000 (the last 32768 columns: the body tail of the SA levels). When a
    // matrix's columns fit, sell_ci is dropped and the SELL kernels stream 10 B per entry, not 12.
    bool c16 = false;
    int c16_tail0 = 0;
    ibmgpu::DBuf<unsigned short> sell_c16;
    ibmgpu::DBuf<int> sell_cbase;  // per slice
    ibmgpu::DBuf<int> perm;              // SELL-sigma: slot -> original row
    int n_short = 0;                     // SELL-sigma slots (rows <= 96 entries)
    int n_long = 0;                      // rows > 96 entries: one warp each, in-order sum
    ibmgpu::DBuf<int> long_rows;
    // stencil (DIA-hybrid) plan: 5-point band {i-S, i-1, i, i+1, i+S} as 5 value planes + a
    // per-row presence mask (bit 6 selects the second stride), extras (columns > i+S, or whole
    // rows that do not fit the band) in a CSR tail — summation order equals CSR column order
    int st_S1 = 0, st_S2 = 0;
    ibmgpu::DBuf<double> st_v;           // 5 * rows, plane-major
    ibmgpu::DBuf<unsigned char> st_mask; // rows
    ibmgpu::DBuf<int> st_erp, st_eci;    // extras CSR
    ibmgpu::DBuf<double> st_ev;
    int n_blocks = 0;                   // CSR-adaptive plan (kern.cuh k_spmv_adapt)
    int n_lrows = 0;                    // its split long rows (each owns a reduction slot)
    ibmgpu::DBuf<int4> blk_meta;         // per CTA: {r0, r1, tpr, 0} | {row, chunk, 0, long-row id}
    ibmgpu::DBuf<int2> lrow;             // per long row: {partial base, chunks}
    ibmgpu::DBuf<double> lpart;          // long-row chunk partials
    ibmgpu::DBuf<unsigned> lcnt;         // long-row arrival counters
    bool planned = false;
    bool borrowed = false;  // owned by a hierarchy / stepper; ibmgpu_csr_destroy refuses
};

namespace ibmgpu {
using Mat = ibmgpu_mat;

// Device buffers are freed on the stream they were allocated on; a matrix planned on a helper
// stream is handed back to the main stream with this before anything else uses it.
inline void mat_rehome(Mat* m, cudaStream_t s) {
    auto set = [s](auto& b) {
        if (b.p) b.s = s;
    };
    set(m->rp), set(m->ci), set(m->v), set(m->sell_off), set(m->sell_ci), set(m->sell_v), set(m->perm);
    set(m->sell_c16), set(m->sell_cbase);
    set(m->long_rows), set(m->st_v), set(m->st_mask), set(m->st_erp), set(m->st_eci), set(m->st_ev);
    set(m->blk_meta), set(m->lrow), set(m->lpart), set(m->lcnt);
}

// csr.cu
Mat* mat_new(Ctx* c, int rows, int cols, int nnz);
void mat_plan(Ctx* c, Mat* m);              // build the SpMV plan (SELL copy or vector width)
void mat_plan_adaptive(Ctx* c, Mat* m);     // CSR-adaptive chunk plan (also used by the fused coarse cycle)
void plan_adaptive_from(Ctx* c, Mat* m, const std::vector<int>& rp);
void spmv(Ctx* c, Mat* A, const double* x, double* y);
Mat* mat_upload(Ctx* c, int rows, int cols, int nnz, const int* rp, const int* ci, const double* v);
void mat_download(Ctx* c, const Mat* m, int* rp, int* ci, double* v);
void diag_of(Ctx* c, const Mat* A, double* d);  // (*this)(i,i) by binary search (sparse.hpp:163)
double max_abs(Ctx* c, const Mat* A);

// sparse_ops.cu
Mat* transpose(Ctx* c, const Mat* A);
Mat* spmm_rows(Ctx* c, const Mat* A, int r0, int r1, const Mat* B);
Mat* triple_product(Ctx* c, const Mat* A, const Mat* B, const Mat* C, int slice, long long* peak, int* slices);
Mat* add(Ctx* c, double a, const Mat* A, double b, const Mat* B);
Mat* symmetrized(Ctx* c, const Mat* A);
Mat* pin(Ctx* c, const Mat* A, int p);
Mat* scale(Ctx* c, const Mat* A, int mode, double a, const double* d_dev);
Mat* from_triplets(Ctx* c, int rows, int cols, size_t n, const int* r_dev, const int* c_dev, const double* v_dev);
Mat* concat_cols(Ctx* c, const Mat* G, const Mat* Et);
Mat* identity_tail_append(Ctx* c, const Mat* Pcore, int n_core, int n_agg, int tail);
bool is_symmetric(Ctx* c, const Mat* A, double tol);
Mat* diag_matrix(Ctx* c, int n, const double* d_dev);

// scan helper (cub) — exclusive scan of n ints into out (n+1 entries, out[n] = total)
void exclusive_scan_total(Ctx* c, const int* in, int* out, int n);
long long exclusive_scan_total64(Ctx* c, const long long* in, long long* out, int n);

}  // namespace ibmgpu
