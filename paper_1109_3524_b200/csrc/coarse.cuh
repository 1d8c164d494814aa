// coarse.cuh — the coarse sub-cycle of the V-cycle as ONE persistent kernel.
//
// Below a size threshold the SA levels are latency-bound: each of their SpMVs moves a few MB
// but costs a full launch plus a dependent-load chain (~8 us), and a V-cycle has 4 per level
// plus the dense coarse solve. The fused kernel runs the whole tail of the cycle —
//   K1(l) K2(l) ... K1(L-1) K2(L-1)  coarse GEMV  K3(L-1) K4(L-1) ... K3(l) K4(l)
// — as phases of a co-resident grid separated by a software grid barrier. Every SpMV phase uses
// the matrix's CSR-adaptive chunk plan (grid-stride over chunks), with the same epilogue
// arithmetic as the standalone kernels (amg.cuh), so results are unchanged up to the
// adaptive kernel's fixed summation order.
#pragma once
#include "kern.cuh"

namespace ibmgpu {

enum PhaseKind : int { PH_JACOBI = 0, PH_STORE = 1, PH_ADD = 2, PH_POST = 3, PH_GEMV = 4 };

struct Phase {
    int kind;
    int n_blocks;   // adaptive chunks (SpMV) or rows (GEMV)
    AdaptPlan pl;
    const int* rp;
    const int* ci;
    const double* v;  // matrix values (GEMV: dense inverse, row-major n x n)
    const double* wd;
    const double* b;
    double* x;    // JACOBI: x out; ADD: x in/out; POST: x in; GEMV: input
    double* out;  // JACOBI: r; STORE: y; POST: out; GEMV: y
};

struct CoarsePlan {
    const Phase* phases;
    int n_phases;
    unsigned* bar_count;
    unsigned* bar_gen;
};

__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vg = gen;
        const unsigned my = *vg;
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            *count = 0;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*vg == my) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// One adaptive chunk of a phase (mirrors k_spmv_adapt), epilogue chosen by kind.
template <int KIND>
__device__ __forceinline__ void coarse_chunk(const Phase& P, int blk) {
    const int4 m = __ldg(P.pl.meta + blk);
    // vectors produced inside this launch are read through L2 (__ldcg): L1 is not coherent
    // across SMs between phases; matrices and omega/D are immutable (__ldg)
    auto gather = [&](int j) -> double {
        if constexpr (KIND == PH_JACOBI) return mul(__ldg(P.wd + j), __ldcg(P.b + j));
        else return __ldcg(P.x + j);
    };
    auto epi = [&](int i, double s) {
        if constexpr (KIND == PH_JACOBI) {
            const double bi = __ldcg(P.b + i);
            P.x[i] = mul(__ldg(P.wd + i), bi);
            P.out[i] = subd(bi, s);
        } else if constexpr (KIND == PH_STORE) {
            P.out[i] = s;
        } else if constexpr (KIND == PH_ADD) {
            P.out[i] = addd(__ldcg(P.out + i), s);  // out aliases the level's x
        } else {
            P.out[i] = addd(__ldcg(P.x + i), mul(__ldg(P.wd + i), subd(__ldcg(P.b + i), s)));
        }
    };
    const int tpr = m.z;
    if (tpr == 0) {
        const int row = m.x, chunk = m.y;
        const int2 lr = __ldg(P.pl.lrow + m.w);
        const int kb = __ldg(P.rp + row) + chunk * kRowChunk;
        const int e = min(kb + kRowChunk, __ldg(P.rp + row + 1));
        double s = 0.0;
        for (int k = kb + threadIdx.x; k < e; k += kBlock) s = addd(s, mul(__ldg(P.v + k), gather(__ldg(P.ci + k))));
        double t[1] = {s};
        block_sum<1>(t);
        if (threadIdx.x == 0) {
            if (lr.y == 1) {
                epi(row, t[0]);
            } else {
                P.pl.lpart[lr.x + chunk] = t[0];
                __threadfence();
                if (atomicAdd(P.pl.lcnt + m.w, 1u) == (unsigned)lr.y - 1) {
                    __threadfence();
                    double tot = 0.0;
                    for (int q = 0; q < lr.y; ++q) tot += __ldcg(P.pl.lpart + lr.x + q);
                    P.pl.lcnt[m.w] = 0;
                    epi(row, tot);
                }
            }
        }
        __syncthreads();  // block_sum's shared buffer is reused by the next chunk
    } else {
        const int r0 = m.x, r1 = m.y;
        const int lane = threadIdx.x & (tpr - 1), grp = threadIdx.x / tpr, ngrp = kBlock / tpr;
        for (int base = r0; base < r1; base += ngrp) {
            const int i = base + grp;
            double s = 0.0;
            if (i < r1)
                for (int k = __ldg(P.rp + i) + lane; k < __ldg(P.rp + i + 1); k += tpr)
                    s = addd(s, mul(__ldg(P.v + k), gather(__ldg(P.ci + k))));
            for (int o = tpr >> 1; o > 0; o >>= 1) s += __shfl_down_sync(kFull, s, o, tpr);
            if (i < r1 && lane == 0) epi(i, s);
        }
    }
}

static __global__ void __launch_bounds__(kBlock) k_coarse_cycle(CoarsePlan cp, const int* done) {
    if (done && flag_set(done)) return;  // uniform: set before this launch
    for (int ph = 0; ph < cp.n_phases; ++ph) {
        const Phase& P = cp.phases[ph];
        if (P.kind == PH_GEMV) {
            const int warps = gridDim.x * (kBlock / 32);
            const int lane = threadIdx.x & 31;
            for (int w = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5); w < P.n_blocks; w += warps) {
                const double* row = P.v + (size_t)w * P.n_blocks;
                double s0 = 0.0, s1 = 0.0;
                int k = lane;
                for (; k + 32 < P.n_blocks; k += 64) {
                    s0 += __ldg(row + k) * __ldcg(P.x + k);
                    s1 += __ldg(row + k + 32) * __ldcg(P.x + k + 32);
                }
                if (k < P.n_blocks) s0 += __ldg(row + k) * __ldcg(P.x + k);
                double s = s0 + s1;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(kFull, s, o);
                if (lane == 0) P.out[w] = s;
            }
        } else {
            for (int blk = blockIdx.x; blk < P.n_blocks; blk += gridDim.x) {
                switch (P.kind) {
                    case PH_JACOBI: coarse_chunk<PH_JACOBI>(P, blk); break;
                    case PH_STORE: coarse_chunk<PH_STORE>(P, blk); break;
                    case PH_ADD: coarse_chunk<PH_ADD>(P, blk); break;
                    default: coarse_chunk<PH_POST>(P, blk); break;
                }
            }
        }
        if (ph + 1 < cp.n_phases) grid_barrier(cp.bar_count, cp.bar_gen);
    }
}

}  // namespace ibmgpu
