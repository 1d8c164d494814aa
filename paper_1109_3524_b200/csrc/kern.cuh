// kern.cuh — device building blocks shared by the hot-path kernels:
//   * bit-exact scalar arithmetic (no FMA contraction: the reference is built without -march,
//     proj/CMakeLists.txt:9, so every a*b+c rounds twice),
//   * deterministic block reductions with a "last block finalises" epilogue (fixed order for a
//     fixed grid, so results are run-to-run reproducible without host round trips),
//   * the SpMV kernels (SELL-32 thread-per-row; CSR vector for long rows) with pluggable
//     operand gathers and fused epilogues.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.cuh"

namespace ibmgpu {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double addd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double subd(double a, double b) { return __dsub_rn(a, b); }

constexpr int kBlock = 256;

// Device-side invariant checks of the checked build (make CHECKED=1): a violated bound traps the
// kernel (cudaErrorIllegalInstruction at the next sync), so the test that ran it fails loudly.
#if defined(IBMGPU_CHECKED)
#define IBM_DCHECK(cond)        \
    do {                        \
        if (!(cond)) __trap();  \
    } while (0)
#else
#define IBM_DCHECK(cond) \
    do {                 \
    } while (0)
#endif
constexpr unsigned kFull = 0xffffffffu;

// L1 prefetch of an epilogue operand, issued before the row loop so its DRAM latency overlaps
// the matrix stream (epilogues opt in by defining touch(i)).
__device__ __forceinline__ void pf(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// The PCG's done flag, written by the previous kernel of the graph: after griddepcontrol.wait a
// weak L2 load (ld.global.cg) sees it. A volatile load compiles to a system-scope strong load
// (LDG.E.STRONG.SYS) whose latency stalled every warp of the coarse-level SpMVs (ncu: 15% of the
// stall samples of the level-3 adaptive kernel at S-4M).
__device__ __forceinline__ bool flag_set(const int* p) { return __ldcg(p) != 0; }

// Programmatic dependent launch: every hot-path kernel is launched with programmatic stream
// serialization, waits for its predecessor's completion + memory flush before touching memory
// (griddepcontrol.wait), and releases its successor when its own block is done — so the next
// kernel's launch and CTA rasterisation overlap this kernel's tail instead of following it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" :::); }
// Grids that fit in one wave release their dependents as soon as every CTA has started, so the
// next kernel's CTAs become resident and stream their (constant) matrix data while this kernel
// runs; larger grids release at the end of each CTA (early dependents would take the slots of
// this grid's later waves).
// `bps` is the kernel's resident CTAs per SM (its launch bounds); 148 SMs on B200.
constexpr int kNumSms = 148;
__device__ __forceinline__ bool pdl_early(int bps) { return gridDim.x <= kNumSms * bps; }
__device__ __forceinline__ void pdl_release_early(int bps) {
#if !defined(IBMGPU_NO_EARLY_RELEASE)
    if (pdl_early(bps)) pdl_release();
#endif
}
__device__ __forceinline__ void pdl_release_late(int bps) {
#if !defined(IBMGPU_NO_EARLY_RELEASE)
    if (!pdl_early(bps)) pdl_release();
#else
    pdl_release();
#endif
}

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("IBMGPU_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <class... KArgs, class... Args>
inline void launch_k(Ctx* c, void (*kernel)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    // PDL invariant: SpMV kernels load their matrix before griddepcontrol.wait, which is only
    // safe when the predecessor did not write it; after any plain launch (CK_LAUNCH sets the
    // fence) this launch waits for full completion instead
    cfg.numAttrs = pdl_enabled() && !c->pdl_fence ? 1 : 0;
    c->pdl_fence = 0;
    CK(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
    ++c->launches;
}

// ---------------------------------------------------------------- reductions
template <int NR>
struct Vals {
    double v[NR];
};

// Deterministic sum of NR values over the block (fixed shuffle tree, fixed warp order).
// Result valid in thread 0.
template <int NR>
__device__ __forceinline__ void block_sum(double (&v)[NR]) {
    __shared__ double sh[NR][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[r] += __shfl_down_sync(kFull, v[r], o);
    }
    __syncthreads();  // protect sh from a previous use
    if (lane == 0)
#pragma unroll
        for (int r = 0; r < NR; ++r) sh[r][w] = v[r];
    __syncthreads();
    if (w == 0) {
        const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            double t = lane < nw ? sh[r][lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(kFull, t, o);
            v[r] = t;
        }
    }
}

// Grid-wide reduction slot: per-block partials + arrival counter (self-resetting).
struct RedSlot {
    double* partials;   // >= gridDim.x * NR
    unsigned* counter;  // zero-initialised once
};

// Every block contributes v; returns true in thread 0 of the last block to arrive, with v
// holding the grid totals (summed in block-index order by a fixed tree).
template <int NR>
__device__ __forceinline__ bool grid_sum_last(double (&v)[NR], RedSlot slot) {
    __shared__ bool is_last;
    block_sum<NR>(v);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int r = 0; r < NR; ++r) slot.partials[(size_t)blockIdx.x * NR + r] = v[r];
        __threadfence();
        const unsigned prev = atomicAdd(slot.counter, 1u);
        is_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return false;
    __threadfence();
    double t[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) t[r] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
#pragma unroll
        for (int r = 0; r < NR; ++r) t[r] += __ldcg(slot.partials + (size_t)b * NR + r);
    block_sum<NR>(t);
    if (threadIdx.x == 0) {
        *slot.counter = 0;
#pragma unroll
        for (int r = 0; r < NR; ++r) v[r] = t[r];
    }
    return threadIdx.x == 0;
}

// Per-block partial only (no fence, no atomic): the grid total is formed by k_finalize, launched
// right after on the same stream — the kernel boundary provides visibility. (A per-block
// __threadfence + arrival atomic costs ~40% of a 16k-block SpMV on B200: the SC fence also
// invalidates the SM's L1, evicting co-resident blocks' gather reuse.)
template <int NR>
__device__ __forceinline__ void block_partial(double (&v)[NR], RedSlot slot) {
    block_sum<NR>(v);
    if (threadIdx.x == 0)
#pragma unroll
        for (int r = 0; r < NR; ++r) slot.partials[(size_t)blockIdx.x * NR + r] = v[r];
}

// One CTA of kFinThreads: sum the partials of `nblocks` blocks in a fixed order and run
// epi.fin(tot). 8 independent loads in flight per thread keep it at ~2 L2 round trips for 16k
// partials.
constexpr int kFinThreads = 1024;

template <class Epi>
__global__ void __launch_bounds__(kFinThreads) k_finalize(Epi epi, int nblocks) {
    pdl_release_early(1);
    constexpr int NR = Epi::NR;
    constexpr int U = 8;
    pdl_wait();
    // the done flag is read alongside the partials (one L2 round trip, not two); a converged
    // solve skips only the epilogue
    const bool skip = epi.skip();
    const RedSlot slot = epi.slot();
    double t[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) t[r] = 0.0;
    int b = threadIdx.x;
    for (; b + (U - 1) * kFinThreads < nblocks; b += U * kFinThreads) {
        double u[U][NR];
#pragma unroll
        for (int q = 0; q < U; ++q)
#pragma unroll
            for (int r = 0; r < NR; ++r) u[q][r] = slot.partials[(size_t)(b + kFinThreads * q) * NR + r];
#pragma unroll
        for (int q = 0; q < U; ++q)
#pragma unroll
            for (int r = 0; r < NR; ++r) t[r] += u[q][r];
    }
    for (; b < nblocks; b += kFinThreads)
#pragma unroll
        for (int r = 0; r < NR; ++r) t[r] += slot.partials[(size_t)b * NR + r];
    block_sum<NR>(t);
    if (!skip && threadIdx.x == 0) epi.fin(t);
}

// ---------------------------------------------------------------- operand gathers
// Gathers of vectors produced by the previous kernel: a weak coherent load (ld.global), not the
// non-coherent __ldg path. Under PDL the producer runs while this grid is already resident, and
// ld.global.nc assumes the data are read-only for the grid's lifetime — it can return a line
// cached before the producer wrote it (seen as a diverging amg_solve on a 3758-row system).
// griddepcontrol.wait makes the producer's writes visible to weak loads.
__device__ __forceinline__ double ld_weak(const double* p) { return *p; }  // LDG.E.64 (not .CONSTANT)
#if defined(IBMGPU_X_CG)
#define IBM_XLD __ldcg
#elif defined(IBMGPU_X_NC)
#define IBM_XLD __ldg
#else
#define IBM_XLD ld_weak
#endif
struct XPlain {
    const double* x;
    __device__ __forceinline__ double operator()(int j) const { return IBM_XLD(x + j); }
};
// x_j = (omega d_j) * b_j  — the damped-Jacobi pre-smoothed iterate of amg.hpp:210 computed on the fly
struct XJacobi {
    const double* wd;
    const double* b;
    __device__ __forceinline__ double operator()(int j) const { return mul(__ldg(wd + j), IBM_XLD(b + j)); }
};

// ---------------------------------------------------------------- SpMV kernels
// Row contract: epi.row(i, s) is called exactly once per row by the owning thread, with s the
// row sum accumulated in column order (identical rounding to sparse.hpp:104-109 for SELL).
// Epi::NR > 0 enables a fused grid reduction: epi.row adds into acc[0..NR), and epi.fin(tot)
// runs once in the last block.

// Column sources of the SELL kernels: plain int32 indices, or 16-bit codes against a per-slice
// base (Mat::c16). ld() loads the raw entry, dec() turns it into the column.
struct Cols32 {
    const int* ci;
    const int* cbase;  // unused
    int tail0;
    __device__ __forceinline__ int ld(int k) const { return __ldg(ci + k); }
    __device__ __forceinline__ int base(int) const { return 0; }
    __device__ __forceinline__ int dec(int raw, int) const { return raw; }
};
struct Cols16 {
    const unsigned short* c;
    const int* cbase;
    int tail0;
    __device__ __forceinline__ int ld(int k) const { return (int)__ldg(c + k); }
    __device__ __forceinline__ int base(int slice) const { return __ldg(cbase + slice); }
    __device__ __forceinline__ int dec(int raw, int b) const { return raw < 0x8000 ? b + raw : tail0 + (raw - 0x8000); }
};

// SELL-32, thread per row, kSellRows rows per thread: every load of both rows (slice entries,
// epilogue operands) is issued before the first use, doubling the bytes in flight per thread —
// the level-0 kernels are latency-bound otherwise (ncu: 33% DRAM, long-scoreboard stalls).
constexpr int kSellRows = 1;
constexpr int kSellU = 5;  // entries per row loaded up front (5-point rows); wider rows loop

template <class XF, class Epi, class CS = Cols32>
__global__ void __launch_bounds__(kBlock, 8) k_spmv_sell(int rows, const int* __restrict__ rp,
                                                         const int* __restrict__ off, CS cs,
                                                         const double* __restrict__ v, XF xf, Epi epi) {
    pdl_release_early(8);
    constexpr int NR = Epi::NR;
    double acc[NR > 0 ? NR : 1];
#pragma unroll
    for (int r = 0; r < (NR > 0 ? NR : 1); ++r) acc[r] = 0.0;
    // The matrix is constant for the whole solve, so its first slice entries are loaded BEFORE
    // griddepcontrol.wait: under PDL they stream in while the predecessor kernel drains.
    const int n_slices = (rows + 31) >> 5;
    int ix[kSellRows], base[kSellRows], width[kSellRows], len[kSellRows], cb[kSellRows];
#pragma unroll
    for (int q = 0; q < kSellRows; ++q) {
        const int i = (blockIdx.x * kSellRows + q) * kBlock + threadIdx.x;
        const int sl = i >> 5;
        // slice loads depend only on the (warp-broadcast) slice offset; the row length only
        // masks the accumulation, so neither waits on row_ptr
        const int beg = sl < n_slices ? __ldg(off + sl) : 0;
        width[q] = sl < n_slices ? (__ldg(off + sl + 1) - beg) >> 5 : 0;
        cb[q] = sl < n_slices ? cs.base(sl) : 0;
        base[q] = beg + (i & 31);
        len[q] = i < rows ? __ldg(rp + i + 1) - __ldg(rp + i) : 0;
        ix[q] = i;
    }
    int c[kSellRows][kSellU];
    double a[kSellRows][kSellU];
#pragma unroll
    for (int q = 0; q < kSellRows; ++q)
#pragma unroll
        for (int u = 0; u < kSellU; ++u)
            if (u < width[q]) {
                c[q][u] = cs.ld(base[q] + 32 * u);
                a[q][u] = __ldg(v + base[q] + 32 * u);
            }
    pdl_wait();
    // the done flag load overlaps the gathers; nothing is written before it is tested
    const bool skip = epi.skip();
    if constexpr (requires { epi.touch(0); }) {
#pragma unroll
        for (int q = 0; q < kSellRows; ++q)
            if (ix[q] < rows) epi.touch(ix[q]);
    }
    double s[kSellRows];
#pragma unroll
    for (int q = 0; q < kSellRows; ++q) {
        s[q] = 0.0;
#pragma unroll
        for (int u = 0; u < kSellU; ++u)
            if (u < len[q]) s[q] = addd(s[q], mul(a[q][u], xf(cs.dec(c[q][u], cb[q]))));
        for (int k = kSellU; k < len[q]; ++k)  // rows wider than kSellU (body-coupled rows)
            s[q] = addd(s[q], mul(__ldg(v + base[q] + 32 * k), xf(cs.dec(cs.ld(base[q] + 32 * k), cb[q]))));
    }
    if (skip) return;
#pragma unroll
    for (int q = 0; q < kSellRows; ++q)
        if (ix[q] < rows) epi.row(ix[q], s[q], acc);
    pdl_release_late(8);
    if constexpr (NR > 0) {
        block_partial<NR>(acc, epi.slot());
    }
}

// Stencil (DIA-hybrid) SpMV for the 5-point operators (lhs2 / level-0 A, the velocity A and L):
// thread per row, every load coalesced and independent of any index stream — the five band
// values, the mask byte and x[i-S], x[i-1], x[i], x[i+1], x[i+S] all issue at once; only rows
// with extras (body coupling, pinned row) touch the CSR tail. Band slots are summed in column
// order, then the extras (whose columns all exceed i+S), so rounding equals spmv_into.
struct StencilPlan {
    const double* v;            // 5 planes of n
    const unsigned char* mask;  // bits 0-4 slot present, bit 5 has extras, bit 6 second stride
    const int* erp;
    const int* eci;
    const double* ev;
    int S1, S2;
};

template <class XF, class Epi>
__global__ void __launch_bounds__(kBlock, 8) k_spmv_stencil(int rows, StencilPlan P, XF xf, Epi epi) {
    pdl_release_early(8);
    constexpr int NR = Epi::NR;
    double acc[NR > 0 ? NR : 1];
#pragma unroll
    for (int r = 0; r < (NR > 0 ? NR : 1); ++r) acc[r] = 0.0;
    const int i = blockIdx.x * kBlock + threadIdx.x;
    const bool live = i < rows;
    // mask and band values are constant for the solve: loaded before griddepcontrol.wait
    // With a single stride (lhs2) nothing waits on the mask byte: the five band values (stored 0.0
    // where a slot is absent) and the five x gathers (indices clamped into range) all issue at
    // once; the mask only selects which products enter the column-order sum. With two strides
    // (velocity A / L: u and v blocks) the stride comes from the mask.
    const bool one_stride = P.S2 == 0;
    const unsigned m = live ? __ldg(P.mask + i) : 0u;
    double a[5], xv[5];
    if (one_stride) {
#pragma unroll
        for (int q = 0; q < 5; ++q) a[q] = live ? __ldg(P.v + (size_t)q * rows + i) : 0.0;
    } else {
#pragma unroll
        for (int q = 0; q < 5; ++q)
            if (m & (1u << q)) a[q] = __ldg(P.v + (size_t)q * rows + i);
    }
    pdl_wait();
    const bool skip = epi.skip();  // tested after the gathers are issued
    if constexpr (requires { epi.touch(0); }) {
        if (live) epi.touch(i);
    }
    if (one_stride) {
        const int S = P.S1, ic = live ? i : 0;
        const int col[5] = {max(ic - S, 0), max(ic - 1, 0), ic, min(ic + 1, rows - 1), min(ic + S, rows - 1)};
#pragma unroll
        for (int q = 0; q < 5; ++q) xv[q] = xf(col[q]);
    } else {
        const int S = (m & 64u) ? P.S2 : P.S1;
        const int col[5] = {i - S, i - 1, i, i + 1, i + S};
#pragma unroll
        for (int q = 0; q < 5; ++q)
            if (m & (1u << q)) xv[q] = xf(col[q]);
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 5; ++q)
        if (m & (1u << q)) s = addd(s, mul(a[q], xv[q]));
    if (__any_sync(kFull, m & 32u)) {
        if (m & 32u) {
            const int e = __ldg(P.erp + i + 1);
            for (int k = __ldg(P.erp + i); k < e; ++k) s = addd(s, mul(__ldg(P.ev + k), xf(__ldg(P.eci + k))));
        }
    }
    if (skip) return;
    if (live) epi.row(i, s, acc);
    pdl_release_late(8);
    if constexpr (NR > 0) {
        block_partial<NR>(acc, epi.slot());
    }
}

// SELL-32-sigma for the wider Galerkin levels (15-60 entries per row): rows are sorted by length
// (descending) within 512-row windows so a slice's rows have similar lengths, slot i holds
// original row perm[i]. Entries keep their column order, so the sum is still bit-exact with
// spmv_into. The entry loop is software-pipelined: chunk k+1's indices/values are in flight while
// chunk k's x-gathers are consumed.
// Rows longer than 96 entries (listed in long_rows) are handled by the CTAs after the first
// `sblocks`, one warp per row: lanes form the products of 32 consecutive entries in parallel
// (the next 32 already in flight) and every lane adds them in column order from shuffles —
// the same rounding sequence as the thread-per-row sum.
template <class XF>
__device__ __forceinline__ double row_sum_inorder(int row, const int* __restrict__ rp, const int* __restrict__ ci,
                                                  const double* __restrict__ v, XF xf, int lane) {
    const int b = __ldg(rp + row), e = __ldg(rp + row + 1);
    double s = 0.0;
    int k = b + lane;
    double p = k < e ? mul(__ldg(v + k), xf(__ldg(ci + k))) : 0.0;
    for (int k0 = b; k0 < e; k0 += 32) {
        const int kn = k0 + 32 + lane;
        const double pn = kn < e ? mul(__ldg(v + kn), xf(__ldg(ci + kn))) : 0.0;
        const int cnt = min(32, e - k0);
        if (cnt == 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j) s = addd(s, __shfl_sync(kFull, p, j));
        } else {
            for (int j = 0; j < cnt; ++j) s = addd(s, __shfl_sync(kFull, p, j));
        }
        p = pn;
    }
    return s;
}

// kU entries per software-pipeline stage. A matrix with few rows (every row a thread, < ~1000
// threads per SM) cannot hide DRAM latency with more warps, only with more loads in flight per
// thread: those launch the kU = 8 instance (its registers do not matter at that occupancy).
#ifndef IBMGPU_SELLW_WIDE_MINB
#define IBMGPU_SELLW_WIDE_MINB 2
#endif
#ifndef IBMGPU_SELLW_MINB
#define IBMGPU_SELLW_MINB 4
#endif
template <class XF, class Epi, int kU = 4, class CS = Cols32>
__global__ void __launch_bounds__(kBlock, kU == 4 ? IBMGPU_SELLW_MINB : IBMGPU_SELLW_WIDE_MINB) k_spmv_sellw(int rows, const int* __restrict__ rp,
                                                          const int* __restrict__ perm, const int* __restrict__ off,
                                                          CS cs, const double* __restrict__ v,
                                                          XF xf, Epi epi, int sblocks, const int* __restrict__ long_rows,
                                                          int n_long, const int* __restrict__ csr_ci,
                                                          const double* __restrict__ csr_v) {
    pdl_release_early(kU == 4 ? IBMGPU_SELLW_MINB : IBMGPU_SELLW_WIDE_MINB);
    constexpr int NR = Epi::NR;
    constexpr int U = kU;
    double acc[NR > 0 ? NR : 1];
#pragma unroll
    for (int r = 0; r < (NR > 0 ? NR : 1); ++r) acc[r] = 0.0;
    if (blockIdx.x >= sblocks) {
        const int w = (blockIdx.x - sblocks) * (kBlock / 32) + (threadIdx.x >> 5);
        const int lane = threadIdx.x & 31;
        const int row = w < n_long ? __ldg(long_rows + w) : -1;  // plan data: before the wait
        pdl_wait();
        const bool skip = epi.skip();
        if (row >= 0) {
            const double s = row_sum_inorder(row, rp, csr_ci, csr_v, xf, lane);  // CSR arrays, not the slices
            if (skip) return;
            if (lane == 0) epi.row(row, s, acc);
        }
        if (skip) return;
        pdl_release_late(kU == 4 ? IBMGPU_SELLW_MINB : IBMGPU_SELLW_WIDE_MINB);
        if constexpr (NR > 0) block_partial<NR>(acc, epi.slot());
        return;
    }
    const int i = blockIdx.x * kBlock + threadIdx.x;
    const int sl = i >> 5;
    const bool in_slice = sl < ((rows + 31) >> 5);
    const int beg = in_slice ? __ldg(off + sl) : 0;
    const int width = in_slice ? (__ldg(off + sl + 1) - beg) >> 5 : 0;
    const int base = beg + (i & 31);
    const int cb = in_slice ? cs.base(sl) : 0;
    const int row = i < rows ? __ldg(perm + i) : -1;
    const int len = row >= 0 ? __ldg(rp + row + 1) - __ldg(rp + row) : 0;
    int c0[U];
    double a0[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (u < width) {
            c0[u] = cs.ld(base + 32 * u);
            a0[u] = __ldg(v + base + 32 * u);
        }
    pdl_wait();  // everything above is the (constant) matrix
    const bool skip = epi.skip();
    if constexpr (requires { epi.touch(0); }) {
        if (row >= 0) epi.touch(row);
    }
    double s = 0.0;
    for (int k0 = 0; k0 < width; k0 += U) {
        int c1[U];
        double a1[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k0 + U + u < width) {
                c1[u] = cs.ld(base + 32 * (k0 + U + u));
                a1[u] = __ldg(v + base + 32 * (k0 + U + u));
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k0 + u < len) s = addd(s, mul(a0[u], xf(cs.dec(c0[u], cb))));
#pragma unroll
        for (int u = 0; u < U; ++u) {
            c0[u] = c1[u];
            a0[u] = a1[u];
        }
    }
    if (skip) return;
    if (row >= 0) epi.row(row, s, acc);
    pdl_release_late(kU == 4 ? IBMGPU_SELLW_MINB : IBMGPU_SELLW_WIDE_MINB);
    if constexpr (NR > 0) {
        block_partial<NR>(acc, epi.slot());
    }
}

// CSR-adaptive SpMV for irregular / long-row matrices (Galerkin coarse levels: a few aggregate
// rows couple to thousands of body rows). The plan cuts the rows into per-CTA chunks of ~2k
// nonzeros: a chunk is either one long row reduced by the whole CTA, or a run of rows handled by
// `tpr`-thread groups (tpr in 2..32, chosen from the chunk's mean row length). Every reduction
// has a fixed order, so results are deterministic.
// Long rows (> kLongRow entries) are cut into kRowChunk-entry chunks, one CTA each; the last CTA of
// a row to finish (arrival counter) sums the chunk partials in chunk order and runs the epilogue.
constexpr int kLongRow = 1024, kRowChunk = 2048;

struct AdaptPlan {
    const int4* meta;        // {r0, r1, tpr, 0} or, for a long-row chunk, {row, chunk, 0, long-row id}
    const int2* lrow;        // per long row: {partial base, chunk count}
    double* lpart;           // chunk partials
    unsigned* lcnt;          // per long row arrival counters (self-resetting)
};

template <class XF, class Epi>
#ifndef IBMGPU_ADAPT_MINB
#define IBMGPU_ADAPT_MINB 8
#endif
__global__ void __launch_bounds__(kBlock, IBMGPU_ADAPT_MINB) k_spmv_adapt(AdaptPlan pl, const int* __restrict__ rp,
                                                       const int* __restrict__ ci, const double* __restrict__ v,
                                                       XF xf, Epi epi) {
    pdl_release_early(IBMGPU_ADAPT_MINB);
    constexpr int NR = Epi::NR;
    const int4 m = __ldg(pl.meta + blockIdx.x);  // plan and matrix are constant: read before the wait
    double acc[NR > 0 ? NR : 1];
#pragma unroll
    for (int r = 0; r < (NR > 0 ? NR : 1); ++r) acc[r] = 0.0;
    const int tpr = m.z;
    if (tpr == 0) {  // one chunk of a long row, whole CTA
        const int row = m.x, chunk = m.y;
        const int2 lr = __ldg(pl.lrow + m.w);
        const int kb = __ldg(rp + row) + chunk * kRowChunk;
        const int e = min(kb + kRowChunk, __ldg(rp + row + 1));
        pdl_wait();
        const bool skip = epi.skip();
        double s = 0.0;
        int k = kb + threadIdx.x;
        for (; k + 3 * kBlock < e; k += 4 * kBlock) {  // 4 independent gathers in flight per thread
            int c[4];
            double a[4], xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                c[u] = __ldg(ci + k + u * kBlock);
                a[u] = __ldg(v + k + u * kBlock);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) xv[u] = xf(c[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) s = addd(s, mul(a[u], xv[u]));
        }
        for (; k < e; k += kBlock) s = addd(s, mul(__ldg(v + k), xf(__ldg(ci + k))));
        if (skip) return;
        double t[1] = {s};
        block_sum<1>(t);
        if (threadIdx.x == 0) {
            // The row's share of a fused reduction goes to its own partial slot (gridDim.x + long-row
            // id), never into this CTA's block partial: which CTA completes a split row depends on
            // arrival order, so a block slot would make the reduction order (and omega, alpha, ...)
            // run-dependent. The finalize sums the block slots, then the long-row slots, in order.
            double racc[NR > 0 ? NR : 1];
#pragma unroll
            for (int r = 0; r < (NR > 0 ? NR : 1); ++r) racc[r] = 0.0;
            bool done_row = false;
            if (lr.y == 1) {
                epi.row(row, t[0], racc);
                done_row = true;
            } else {
                pl.lpart[lr.x + chunk] = t[0];
                __threadfence();
                if (atomicAdd(pl.lcnt + m.w, 1u) == (unsigned)lr.y - 1) {
                    __threadfence();
                    double tot = 0.0;
                    for (int q = 0; q < lr.y; ++q) tot += __ldcg(pl.lpart + lr.x + q);
                    pl.lcnt[m.w] = 0;
                    epi.row(row, tot, racc);
                    done_row = true;
                }
            }
            if constexpr (NR > 0) {
                if (done_row) {
                    const RedSlot rs = epi.slot();
#pragma unroll
                    for (int r = 0; r < NR; ++r) rs.partials[(size_t)(gridDim.x + m.w) * NR + r] = racc[r];
                }
            }
        }
    } else {
        const int r0 = m.x, r1 = m.y;
        const int lane = threadIdx.x & (tpr - 1), grp = threadIdx.x / tpr, ngrp = kBlock / tpr;
        // the first pass's row bounds and first 4-wide batch are matrix data: issued before the wait
        int c[4];
        double a[4];
        int i = r0 + grp, k = 0, e = 0;
        auto load_batch = [&]() {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k + u * tpr < e) {
                    c[u] = __ldg(ci + k + u * tpr);
                    a[u] = __ldg(v + k + u * tpr);
                }
        };
        if (i < r1) {
            e = __ldg(rp + i + 1);
            k = __ldg(rp + i) + lane;
            load_batch();
        }
        pdl_wait();
        const bool skip = epi.skip();  // tested once the first pass's gathers are in flight
        for (int base = r0; base < r1; base += ngrp) {
            i = base + grp;
            double s = 0.0;
            if (i < r1) {
                if (base != r0) {
                    e = __ldg(rp + i + 1);
                    k = __ldg(rp + i) + lane;
                    load_batch();
                }
                // predicated 4-wide batches: a lane's last (partial) batch issues all its loads at
                // once instead of one dependent index->gather chain per remaining entry. All four
                // gathers issue before the first add, and the next batch's indices/values are
                // requested while they are in flight.
                for (;;) {
                    double xv[4], av[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        xv[u] = k + u * tpr < e ? xf(c[u]) : 0.0;
                        av[u] = a[u];
                    }
                    const int kc = k;
                    k += 4 * tpr;
                    const bool more = k < e;
                    if (more) load_batch();
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (kc + u * tpr < e) s = addd(s, mul(av[u], xv[u]));
                    if (!more) break;
                }
            }
            for (int o = tpr >> 1; o > 0; o >>= 1) s += __shfl_down_sync(kFull, s, o, tpr);
            if (skip) return;
            if (i < r1 && lane == 0) epi.row(i, s, acc);
        }
    }
    pdl_release_late(IBMGPU_ADAPT_MINB);
    if constexpr (NR > 0) {
        block_partial<NR>(acc, epi.slot());
    }
}

// Launch helper: dispatch on the matrix's plan.
// Warp per row with a tree reduction, for the long-row coarse levels (replaces k_spmv_adapt where
// the mean row has >= 48 entries): lanes stride the row four entries at a time with every load of
// a batch issued first (the last, partial batch too), then five shuffle steps. Deterministic (fixed order), not bitwise with spmv_into — the
// same contract as the adaptive kernel. Warps take rows gw, gw + warps, ...
template <class XF, class Epi, int TPR = 32>
__global__ void __launch_bounds__(kBlock, 8) k_spmv_warprow(int rows, const int* __restrict__ rp,
                                                             const int* __restrict__ ci, const double* __restrict__ v,
                                                             XF xf, Epi epi) {
    pdl_release_early(8);
    constexpr int NR = Epi::NR;
    constexpr int G = 32 / TPR;  // rows per warp pass
    double acc[NR > 0 ? NR : 1];
#pragma unroll
    for (int r = 0; r < (NR > 0 ? NR : 1); ++r) acc[r] = 0.0;
    const int lane = threadIdx.x & (TPR - 1), gi = (threadIdx.x & 31) / TPR;
    const int nwr = gridDim.x * (kBlock / 32) * G;  // rows per grid pass
    // warp-uniform pass base: every lane runs every pass (the shuffles need the whole warp)
    int r0 = (blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5)) * G;
    int i = r0 + gi;
    int b = i < rows ? __ldg(rp + i) : 0, e = i < rows ? __ldg(rp + i + 1) : 0;
    pdl_wait();
    const bool skip = epi.skip();
    for (; r0 < rows; r0 += nwr) {
        i = r0 + gi;
        double s = 0.0;
        int k = b + lane;
        for (; k + 3 * TPR < e; k += 4 * TPR) {
            int c[4];
            double a[4], x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) c[u] = __ldg(ci + k + TPR * u), a[u] = __ldg(v + k + TPR * u);
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = xf(c[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) s = addd(s, mul(a[u], x[u]));
        }
        if (k < e) {  // the last (partial) batch: all its loads issued at once
            int c[4];
            double a[4], x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool in = k + TPR * u < e;
                c[u] = in ? __ldg(ci + k + TPR * u) : 0;
                a[u] = in ? __ldg(v + k + TPR * u) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = k + TPR * u < e ? xf(c[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k + TPR * u < e) s = addd(s, mul(a[u], x[u]));
        }
#pragma unroll
        for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_down_sync(kFull, s, o, TPR);
        const int nx = i + nwr;
        b = e = 0;
        if (nx < rows) b = __ldg(rp + nx), e = __ldg(rp + nx + 1);
        if (!skip && lane == 0 && i < rows) epi.row(i, s, acc);
    }
    if (skip) return;
    pdl_release_late(8);
    if constexpr (NR > 0) block_partial<NR>(acc, epi.slot());
}

template <class XF, class Epi>
inline void launch_spmv(Ctx* c, const Mat* A, XF xf, Epi epi, cudaStream_t s) {
    if (A->rows == 0) return;
    int grid = 0;
    const Cols32 c32{A->sell_ci.p, nullptr, 0};
    const Cols16 c16{A->sell_c16.p, A->sell_cbase.p, A->c16_tail0};
    if (A->kind == SPMV_SELL) {
        grid = (A->rows + kSellRows * kBlock - 1) / (kSellRows * kBlock);
        if (A->c16)
            launch_k(c, k_spmv_sell<XF, Epi, Cols16>, grid, kBlock, s, A->rows, A->rp.p, A->sell_off.p, c16,
                     A->sell_v.p, xf, epi);
        else
            launch_k(c, k_spmv_sell<XF, Epi, Cols32>, grid, kBlock, s, A->rows, A->rp.p, A->sell_off.p, c32,
                     A->sell_v.p, xf, epi);
    } else if (A->kind == SPMV_STENCIL) {
        const StencilPlan P{A->st_v.p, A->st_mask.p, A->st_erp.p, A->st_eci.p, A->st_ev.p, A->st_S1, A->st_S2};
        grid = (A->rows + kBlock - 1) / kBlock;
        launch_k(c, k_spmv_stencil<XF, Epi>, grid, kBlock, s, A->rows, P, xf, epi);
    } else if (A->kind == SPMV_SELLW) {
        const int sb = (A->n_short + kBlock - 1) / kBlock;
        grid = sb + (A->n_long + kBlock / 32 - 1) / (kBlock / 32);
        static const int wide_env = [] {  // IBMGPU_SELLW_WIDE=0/1 forces the 4- / 8-entry stage (A/B)
            const char* e = std::getenv("IBMGPU_SELLW_WIDE");
            return e ? std::atoi(e) : -1;
        }();
        // the 8-entry stage while the slots are under 2560 per SM: more loads in flight per thread
        // when the grid is too small to hide latency with warps (C2 L1 320k rows: C2 -2%, S-4M
        // -0.5%; the 1.2M-row S-4M A_1 stays on 4). IBMGPU_SELLW_WIDE_ROWS (A/B): the threshold;
        // 1024 restores the old rule (which also asked for >= 40 entries per row)
        static const int wide_rows = [] {
            const char* e = std::getenv("IBMGPU_SELLW_WIDE_ROWS");
            return e ? std::atoi(e) : 2560;
        }();
        const bool wide = wide_env >= 0 ? wide_env == 1
                                        : (long long)A->n_short < (long long)c->num_sms * wide_rows &&
                                              (wide_rows > 1024 || A->nnz >= 40ll * A->rows);  // few, long rows
        auto go = [&](auto kern, auto cs) {
            launch_k(c, kern, grid, kBlock, s, A->n_short, A->rp.p, A->perm.p, A->sell_off.p, cs, A->sell_v.p, xf,
                     epi, sb, (const int*)A->long_rows.p, A->n_long, (const int*)A->ci.p, (const double*)A->v.p);
        };
        if (A->c16) {
            if (wide)
                go(k_spmv_sellw<XF, Epi, 8, Cols16>, c16);
            else
                go(k_spmv_sellw<XF, Epi, 4, Cols16>, c16);
        } else {
            if (wide)
                go(k_spmv_sellw<XF, Epi, 8, Cols32>, c32);
            else
                go(k_spmv_sellw<XF, Epi, 4, Cols32>, c32);
        }
    } else {
        // warp per row when the mean row has >= 48 entries (S-4M 0.768 -> 0.753 ms per iteration,
        // C2 0.295 -> 0.279; thresholds 32 / 100: C2 0.281 / 0.284). IBMGPU_WARPROW=N sets the bar,
        // 0 keeps every such matrix on k_spmv_adapt
        static const int warprow = [] {
            const char* e = std::getenv("IBMGPU_WARPROW");
            return e ? std::atoi(e) : 48;
        }();
        static const int warprow16 = [] {  // IBMGPU_WARPROW16=N: half-warp rows for means in [N, 48) (A/B)
            const char* e = std::getenv("IBMGPU_WARPROW16");
            return e ? std::atoi(e) : 0;
        }();
        if (warprow > 0 && A->nnz >= (long long)warprow * A->rows) {
            grid = std::max(1, std::min(A->n_blocks, (A->rows + kBlock / 32 - 1) / (kBlock / 32)));
            launch_k(c, k_spmv_warprow<XF, Epi, 32>, grid, kBlock, s, A->rows, A->rp.p, A->ci.p, A->v.p, xf, epi);
            if constexpr (Epi::NR > 0) launch_k(c, k_finalize<Epi>, 1, kFinThreads, s, epi, grid);
            return;
        }
        if (warprow16 > 0 && A->nnz >= (long long)warprow16 * A->rows) {
            grid = std::max(1, std::min(A->n_blocks, (A->rows + kBlock / 16 - 1) / (kBlock / 16)));
            launch_k(c, k_spmv_warprow<XF, Epi, 16>, grid, kBlock, s, A->rows, A->rp.p, A->ci.p, A->v.p, xf, epi);
            if constexpr (Epi::NR > 0) launch_k(c, k_finalize<Epi>, 1, kFinThreads, s, epi, grid);
            return;
        }
        const AdaptPlan pl{A->blk_meta.p, A->lrow.p, A->lpart.p, A->lcnt.p};
        grid = A->n_blocks;
        launch_k(c, k_spmv_adapt<XF, Epi>, grid, kBlock, s, pl, A->rp.p, A->ci.p, A->v.p, xf, epi);
    }
    // adaptive plans: the long rows' reduction slots follow the CTAs' (k_spmv_adapt)
    const int slots = (A->kind == SPMV_SELL || A->kind == SPMV_SELLW || A->kind == SPMV_STENCIL) ? grid
                                                                                                : grid + A->n_lrows;
    if constexpr (Epi::NR > 0) launch_k(c, k_finalize<Epi>, 1, kFinThreads, s, epi, slots);
}

// Number of blocks launch_spmv uses (sizes the reduction partials).
inline int spmv_grid(const Mat* A) {
    if (A->rows == 0) return 0;
    if (A->kind == SPMV_SELL) return (A->rows + kSellRows * kBlock - 1) / (kSellRows * kBlock);
    if (A->kind == SPMV_SELLW)
        return (A->n_short + kBlock - 1) / kBlock + (A->n_long + kBlock / 32 - 1) / (kBlock / 32);
    if (A->kind == SPMV_STENCIL) return (A->rows + kBlock - 1) / kBlock;
    return A->n_blocks + A->n_lrows;  // CTAs + one reduction slot per split long row
}

// Plain epilogue: y_i = s.
struct EpiStore {
    static constexpr int NR = 0;
    double* y;
    __device__ bool skip() const { return false; }
    __device__ void row(int i, double s, double*) const { y[i] = s; }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

// Elementwise kernels over n with an optional fused reduction (same epilogue contract).
template <class Body>
__global__ void __launch_bounds__(kBlock) k_elem(int n, Body body) {
    pdl_release_early(8);
    constexpr int NR = Body::NR;
    pdl_wait();
    if (body.skip()) return;
    double acc[NR > 0 ? NR : 1];
#pragma unroll
    for (int r = 0; r < (NR > 0 ? NR : 1); ++r) acc[r] = 0.0;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) body.row(i, acc);
    pdl_release_late(8);
    if constexpr (NR > 0) block_partial<NR>(acc, body.slot());
}

inline int elem_grid(Ctx* c, long long n) {
    const long long want = (n + kBlock - 1) / kBlock;
    const long long cap = (long long)c->num_sms * 8;
    return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

template <class Body>
inline void launch_elem(Ctx* c, int n, int grid, Body body, cudaStream_t s) {
    launch_k(c, k_elem<Body>, grid, kBlock, s, n, body);
    if constexpr (Body::NR > 0) launch_k(c, k_finalize<Body>, 1, kFinThreads, s, body, grid);
}

}  // namespace ibmgpu
