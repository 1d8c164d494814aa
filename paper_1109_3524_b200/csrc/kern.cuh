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
constexpr unsigned kFull = 0xffffffffu;

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

// ---------------------------------------------------------------- operand gathers
struct XPlain {
    const double* x;
    __device__ __forceinline__ double operator()(int j) const { return __ldg(x + j); }
};
// x_j = (omega d_j) * b_j  — the damped-Jacobi pre-smoothed iterate of amg.hpp:210 computed on the fly
struct XJacobi {
    const double* wd;
    const double* b;
    __device__ __forceinline__ double operator()(int j) const { return mul(__ldg(wd + j), __ldg(b + j)); }
};

// ---------------------------------------------------------------- SpMV kernels
// Row contract: epi.row(i, s) is called exactly once per row by the owning thread, with s the
// row sum accumulated in column order (identical rounding to sparse.hpp:104-109 for SELL).
// Epi::NR > 0 enables a fused grid reduction: epi.row adds into acc[0..NR), and epi.fin(tot)
// runs once in the last block.

template <class XF, class Epi>
__global__ void __launch_bounds__(kBlock) k_spmv_sell(int rows, const int* __restrict__ rp,
                                                      const int* __restrict__ off, const int* __restrict__ ci,
                                                      const double* __restrict__ v, XF xf, Epi epi) {
    constexpr int NR = Epi::NR;
    if (epi.skip()) return;
    double acc[NR > 0 ? NR : 1];
#pragma unroll
    for (int r = 0; r < (NR > 0 ? NR : 1); ++r) acc[r] = 0.0;
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i < rows) {
        const int len = __ldg(rp + i + 1) - __ldg(rp + i);
        const int base = __ldg(off + (i >> 5)) + (i & 31);
        double s = 0.0;
        for (int k0 = 0; k0 < len; k0 += 8) {
            int c[8];
            double a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (k0 + u < len) {
                    c[u] = __ldg(ci + base + 32 * (k0 + u));
                    a[u] = __ldg(v + base + 32 * (k0 + u));
                }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (k0 + u < len) s = addd(s, mul(a[u], xf(c[u])));
        }
        epi.row(i, s, acc);
    }
    if constexpr (NR > 0) {
        if (grid_sum_last<NR>(acc, epi.slot())) epi.fin(acc);
    }
}

template <int TPR, class XF, class Epi>
__global__ void __launch_bounds__(kBlock) k_spmv_vec(int rows, const int* __restrict__ rp,
                                                     const int* __restrict__ ci, const double* __restrict__ v,
                                                     XF xf, Epi epi) {
    constexpr int NR = Epi::NR;
    if (epi.skip()) return;
    double acc[NR > 0 ? NR : 1];
#pragma unroll
    for (int r = 0; r < (NR > 0 ? NR : 1); ++r) acc[r] = 0.0;
    const int g = blockIdx.x * kBlock + threadIdx.x;
    const int i = g / TPR, lane = g % TPR;
    double s = 0.0;
    if (i < rows) {
        const int e = __ldg(rp + i + 1);
        int k = __ldg(rp + i) + lane;
        for (; k + TPR < e; k += 2 * TPR) {
            const int c0 = __ldg(ci + k), c1 = __ldg(ci + k + TPR);
            const double a0 = __ldg(v + k), a1 = __ldg(v + k + TPR);
            s = addd(s, mul(a0, xf(c0)));
            s = addd(s, mul(a1, xf(c1)));
        }
        if (k < e) s = addd(s, mul(__ldg(v + k), xf(__ldg(ci + k))));
    }
#pragma unroll
    for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_down_sync(kFull, s, o, TPR);
    if (i < rows && lane == 0) epi.row(i, s, acc);
    if constexpr (NR > 0) {
        if (grid_sum_last<NR>(acc, epi.slot())) epi.fin(acc);
    }
}

// Launch helper: dispatch on the matrix's plan.
template <class XF, class Epi>
inline void launch_spmv(Ctx* c, const Mat* A, XF xf, Epi epi, cudaStream_t s) {
    if (A->rows == 0) return;
    if (A->kind == SPMV_SELL) {
        const int grid = (A->rows + kBlock - 1) / kBlock;
        k_spmv_sell<<<grid, kBlock, 0, s>>>(A->rows, A->rp.p, A->sell_off.p, A->sell_ci.p, A->sell_v.p, xf, epi);
    } else {
        const long long threads = (long long)A->rows * A->tpr;
        const int grid = (int)((threads + kBlock - 1) / kBlock);
        switch (A->tpr) {
            case 4: k_spmv_vec<4><<<grid, kBlock, 0, s>>>(A->rows, A->rp.p, A->ci.p, A->v.p, xf, epi); break;
            case 8: k_spmv_vec<8><<<grid, kBlock, 0, s>>>(A->rows, A->rp.p, A->ci.p, A->v.p, xf, epi); break;
            case 16: k_spmv_vec<16><<<grid, kBlock, 0, s>>>(A->rows, A->rp.p, A->ci.p, A->v.p, xf, epi); break;
            default: k_spmv_vec<32><<<grid, kBlock, 0, s>>>(A->rows, A->rp.p, A->ci.p, A->v.p, xf, epi); break;
        }
    }
    CK_LAUNCH(c);
}

// Number of blocks launch_spmv uses (sizes the reduction partials).
inline int spmv_grid(const Mat* A) {
    if (A->rows == 0) return 0;
    if (A->kind == SPMV_SELL) return (A->rows + kBlock - 1) / kBlock;
    return (int)(((long long)A->rows * A->tpr + kBlock - 1) / kBlock);
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
    constexpr int NR = Body::NR;
    if (body.skip()) return;
    double acc[NR > 0 ? NR : 1];
#pragma unroll
    for (int r = 0; r < (NR > 0 ? NR : 1); ++r) acc[r] = 0.0;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) body.row(i, acc);
    if constexpr (NR > 0) {
        if (grid_sum_last<NR>(acc, body.slot())) body.fin(acc);
    }
}

inline int elem_grid(Ctx* c, long long n) {
    const long long want = (n + kBlock - 1) / kBlock;
    const long long cap = (long long)c->num_sms * 8;
    return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

template <class Body>
inline void launch_elem(Ctx* c, int n, int grid, Body body, cudaStream_t s) {
    k_elem<<<grid, kBlock, 0, s>>>(n, body);
    CK_LAUNCH(c);
}

}  // namespace ibmgpu
