// xfer.cu — setup of the level-0 stencil transfers (xfer.cuh): eligibility, aggregate member
// lists and the tentative-prolongator weights t_a = 1/sqrt(|a|) (amg.hpp:153-161).
#include <algorithm>
#include <cstdlib>

#include "amg.cuh"
#include "internal.cuh"

namespace ibmgpu {
namespace {

inline int nblk(long long n) { return (int)((n + 255) / 256); }

// A core row qualifies when it is a band row of the single-stride stencil whose present slots
// stay inside the pressure grid (no wrap across a grid line, no +S into the tail) and whose extras
// are all tail columns.
__global__ void k_xfer_check(int n_core, int S, StencilPlan P, int* bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_core) return;
    const unsigned m = P.mask[i];
    bool ok = (m & 4u) && !(m & 64u);
    if (m & 1u) ok = ok && i >= S;
    if (m & 16u) ok = ok && i + S < n_core;
    if (m & 2u) ok = ok && (i % S) != 0;
    if (m & 8u) ok = ok && (i % S) != S - 1;
    if (ok && (m & 32u))
        for (int k = P.erp[i]; k < P.erp[i + 1]; ++k) ok = ok && P.eci[k] >= n_core;
    if (!ok) atomicAdd(bad, 1);
}

__global__ void k_xfer_count(int n_core, const int* __restrict__ agg, int* __restrict__ size) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_core) atomicAdd(size + agg[i], 1);
}

__global__ void k_xfer_fill(int n_core, const int* __restrict__ agg, const int* __restrict__ mrp,
                            int* __restrict__ cursor, int* __restrict__ mem) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_core) {
        const int a = agg[i];
        mem[mrp[a] + atomicAdd(cursor + a, 1)] = i;
    }
}

// members in ascending row order (fixed summation order) and t_a
__global__ void k_xfer_sort(int n_agg, const int* __restrict__ mrp, int* __restrict__ mem,
                            double* __restrict__ tagg) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n_agg) return;
    const int b = mrp[a], e = mrp[a + 1];
    for (int k = b + 1; k < e; ++k) {
        const int v = mem[k];
        int q = k - 1;
        while (q >= b && mem[q] > v) {
            mem[q + 1] = mem[q];
            --q;
        }
        mem[q + 1] = v;
    }
    tagg[a] = __ddiv_rn(1.0, __dsqrt_rn((double)(e - b)));  // amg.hpp:160
}

// mark the core columns of the tail rows (one warp per tail row)
__global__ void k_xfer_flag(int n, int n_core, const int* __restrict__ rp, const int* __restrict__ ci,
                            unsigned char* mask) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int row = n_core + t;
    if (row >= n) return;
    for (int k = rp[row] + lane; k < rp[row + 1]; k += 32) {
        const int c = ci[k];
        if (c < n_core) mask[c] |= (unsigned char)kXTailCol;  // same value from every writer
    }
}

}  // namespace

bool xfer0_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("IBMGPU_XFER0");
        return !(e && e[0] == '0');
    }();
    return on;
}

void xfer0_setup(Ctx* c, Hier* h) {
    Xfer0& X = h->x0;
    X.on = false;
    if (X.built) {  // buffers are referenced by captured PCG graphs: never rebuilt
        X.on = xfer0_enabled();
        return;
    }
    if (!xfer0_enabled() || h->active_levels() < 1) return;
    if (h->n_phases && h->fuse_from < 1) return;  // level 0 inside the fused coarse cycle
    const Level& lv = *h->levels[0];
    const Mat* A = lv.A;
    if (A->kind != SPMV_STENCIL || A->st_S2 != 0 || A->st_S1 <= 1) return;
    const int S = A->st_S1, n_core = lv.n_core, n = A->rows;
    if (n_core < 2 * S || n_core % S != 0) return;
    const StencilPlan P{A->st_v.p, A->st_mask.p, A->st_erp.p, A->st_eci.p, A->st_ev.p, A->st_S1, A->st_S2};
    DBuf<int> bad(c, 1);
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), c->stream));
    k_xfer_check<<<nblk(n_core), 256, 0, c->stream>>>(n_core, S, P, bad.p);
    CK_LAUNCH(c);
    if (d2h_scalar(c, bad.p) != 0) return;
    const int n_agg = lv.n_agg;
    DBuf<int> size(c, (size_t)n_agg), cursor(c, (size_t)n_agg);
    CK(cudaMemsetAsync(size.p, 0, sizeof(int) * (size_t)n_agg, c->stream));
    CK(cudaMemsetAsync(cursor.p, 0, sizeof(int) * (size_t)n_agg, c->stream));
    k_xfer_count<<<nblk(n_core), 256, 0, c->stream>>>(n_core, lv.agg.p, size.p);
    CK_LAUNCH(c);
    X.mrp.alloc(c, (size_t)n_agg + 1);
    exclusive_scan_total(c, size.p, X.mrp.p, n_agg);
    X.mem.alloc(c, (size_t)n_core);
    k_xfer_fill<<<nblk(n_core), 256, 0, c->stream>>>(n_core, lv.agg.p, X.mrp.p, cursor.p, X.mem.p);
    CK_LAUNCH(c);
    X.tagg.alloc(c, (size_t)n_agg);
    k_xfer_sort<<<nblk(n_agg), 256, 0, c->stream>>>(n_agg, X.mrp.p, X.mem.p, X.tagg.p);
    CK_LAUNCH(c);
    const int n_tail = n - n_core;
    X.r1t.alloc(c, (size_t)std::max(n_tail, 1));
    X.S = S;
    X.NY = n_core / S;
    X.n_ti = (S + kXOut - 1) / kXOut;
    X.tiles = X.n_ti * ((X.NY + kXTJ - 1) / kXTJ);
    X.tail_ctas = (n_tail + kXTailRows - 1) / kXTailRows;
    // core cells that tail rows couple to keep their x for k_xfer_up_tail (mask bit 7 of the
    // hierarchy's private copy of A_0; no SpMV kernel reads that bit)
    if (n_tail > 0) {
        k_xfer_flag<<<nblk((long long)n_tail * 32), 256, 0, c->stream>>>(n, n_core, A->rp.p, A->ci.p, A->st_mask.p);
        CK_LAUNCH(c);
    }
    X.built = X.on = true;
}

}  // namespace ibmgpu
