// dense.cu — coarsest SA level: dense SPD factorisation + explicit inverse, and the GEMV that
// replaces DenseCholesky::solve inside every V-cycle.
//
// Reference: dense.hpp:20-40 (row-major Cholesky, non-positive pivot -> 1e-13*max(|A|,1) shift)
// and :44-56 (forward/back substitution, serial and column-strided). On the device the factor is
// a right-looking blocked Cholesky (64-wide panels), followed by X = L^{-1} (blocked forward
// substitution on the identity) and A^{-1} = X^T X, all built from one tiled FP64 GEMM-update
// kernel. The per-V-cycle coarse solve is then a single bandwidth-bound GEMV over A^{-1}
// (n_c^2 doubles, read once, warp per row) instead of two latency-bound triangular sweeps.
#include <algorithm>

#include "amg.cuh"
#include "internal.cuh"
#include "kern.cuh"

namespace ibmgpu {

namespace {

constexpr int NB = 64;  // panel width

__global__ void k_csr_to_dense(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                               const double* __restrict__ v, double* __restrict__ A) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) A[(size_t)i * n + ci[k]] = v[k];
}

// Unblocked Cholesky of the diagonal block [kb, kb+nb) (trailing updates already applied).
// Column j: d = a_jj - sum_k l_jk^2 ; d <= 0 -> shift ; l_ij = (a_ij - sum_k l_ik l_jk) / d.
__global__ void k_potrf_diag(int n, int kb, int nb, double shift, double* __restrict__ A) {
    __shared__ double blk[NB][NB + 1];
    const int t = threadIdx.x;
    for (int e = t; e < nb * nb; e += blockDim.x) {
        const int i = e / nb, j = e % nb;
        blk[i][j] = A[(size_t)(kb + i) * n + kb + j];
    }
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
        if (t == 0) {
            double d = blk[j][j];
            for (int k = 0; k < j; ++k) d -= blk[j][k] * blk[j][k];
            if (d <= 0.0) d = shift;
            blk[j][j] = sqrt(d);
        }
        __syncthreads();
        for (int i = j + 1 + t; i < nb; i += blockDim.x) {
            double s = blk[i][j];
            for (int k = 0; k < j; ++k) s -= blk[i][k] * blk[j][k];
            blk[i][j] = s / blk[j][j];
        }
        __syncthreads();
    }
    for (int e = t; e < nb * nb; e += blockDim.x) {
        const int i = e / nb, j = e % nb;
        A[(size_t)(kb + i) * n + kb + j] = j <= i ? blk[i][j] : 0.0;
    }
}

// Panel rows i >= kb+nb: L[i, kb:kb+nb] = A[i, kb:kb+nb] L_kk^{-T} (row-wise forward substitution).
__global__ void k_trsm_panel(int n, int kb, int nb, double* __restrict__ A) {
    __shared__ double Lkk[NB][NB + 1];
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) Lkk[e / nb][e % nb] = A[(size_t)(kb + e / nb) * n + kb + e % nb];
    __syncthreads();
    const int i = kb + nb + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double row[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j)
        if (j < nb) row[j] = A[(size_t)i * n + kb + j];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        if (j < nb) {
            double s = row[j];
            for (int k = 0; k < j; ++k) s -= row[k] * Lkk[j][k];
            row[j] = s / Lkk[j][j];
        }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
        if (j < nb) A[(size_t)i * n + kb + j] = row[j];
}

// Tiled FP64 GEMM update: C[i][j] = beta*C[i][j] + alpha * sum_k opA(i,k) opB(k,j), i<m, j<nn.
// opA(i,k) = TA ? A[k*lda+i] : A[i*lda+k];  opB(k,j) = TB ? B[j*ldb+k] : B[k*ldb+j].
// LOWER: skip tiles strictly above the diagonal (C symmetric / lower-triangular targets).
template <bool TA, bool TB, bool LOWER>
__global__ void __launch_bounds__(256) k_gemm(int m, int nn, int kk, double alpha, const double* __restrict__ A,
                                              int lda, const double* __restrict__ B, int ldb, double beta,
                                              double* __restrict__ C, int ldc) {
    constexpr int BM = 64, BN = 64, BK = 16;
    const int bi = blockIdx.y * BM, bj = blockIdx.x * BN;
    if (LOWER && bj > bi + BM - 1) return;
    __shared__ double As[BK][BM + 1];
    __shared__ double Bs[BK][BN + 1];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    double acc[4][4] = {};
    for (int k0 = 0; k0 < kk; k0 += BK) {
        for (int e = threadIdx.x; e < BM * BK; e += 256) {
            int i, k;
            if (TA) {
                i = e % BM, k = e / BM;
            } else {
                k = e % BK, i = e / BK;
            }
            const int gi = bi + i, gk = k0 + k;
            double val = 0.0;
            if (gi < m && gk < kk) val = TA ? A[(size_t)gk * lda + gi] : A[(size_t)gi * lda + gk];
            As[k][i] = val;
        }
        for (int e = threadIdx.x; e < BN * BK; e += 256) {
            int j, k;
            if (TB) {
                k = e % BK, j = e / BK;
            } else {
                j = e % BN, k = e / BN;
            }
            const int gj = bj + j, gk = k0 + k;
            double val = 0.0;
            if (gj < nn && gk < kk) val = TB ? B[(size_t)gj * ldb + gk] : B[(size_t)gk * ldb + gj];
            Bs[k][j] = val;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            double a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = As[k][ty + 16 * u];
#pragma unroll
            for (int u = 0; u < 4; ++u) b[u] = Bs[k][tx + 16 * u];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int w = 0; w < 4; ++w) acc[u][w] += a[u] * b[w];
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int gi = bi + ty + 16 * u, gj = bj + tx + 16 * w;
            if (gi < m && gj < nn) {
                double* p = C + (size_t)gi * ldc + gj;
                *p = (beta == 0.0 ? 0.0 : beta * *p) + alpha * acc[u][w];
            }
        }
}

template <bool TA, bool TB, bool LOWER>
void gemm(Ctx* c, int m, int nn, int kk, double alpha, const double* A, int lda, const double* B, int ldb,
          double beta, double* C, int ldc) {
    if (m <= 0 || nn <= 0) return;
    dim3 grid((nn + 63) / 64, (m + 63) / 64);
    k_gemm<TA, TB, LOWER><<<grid, 256, 0, c->stream>>>(m, nn, kk, alpha, A, lda, B, ldb, beta, C, ldc);
    CK_LAUNCH(c);
}

__global__ void k_identity(int n, double* X) {
    const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (size_t)n * n) return;
    X[e] = (e / n == e % n) ? 1.0 : 0.0;
}

// Block-row forward substitution: X[kb+r][j] = (X[kb+r][j] - sum_t L[kb+r][kb+t] X[kb+t][j]) / L[kb+r][kb+r]
__global__ void k_trsm_rows(int n, int kb, int nb, int ncols, const double* __restrict__ L, double* __restrict__ X) {
    __shared__ double Lkk[NB][NB + 1];
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) Lkk[e / nb][e % nb] = L[(size_t)(kb + e / nb) * n + kb + e % nb];
    __syncthreads();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ncols) return;
    double col[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r)
        if (r < nb) col[r] = X[(size_t)(kb + r) * n + j];
#pragma unroll
    for (int r = 0; r < NB; ++r) {
        if (r < nb) {
            double s = col[r];
            for (int t = 0; t < r; ++t) s -= Lkk[r][t] * col[t];
            col[r] = s / Lkk[r][r];
        }
    }
#pragma unroll
    for (int r = 0; r < NB; ++r)
        if (r < nb) X[(size_t)(kb + r) * n + j] = col[r];
}

__global__ void k_symmetrize_lower(int n, double* A) {
    const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (size_t)n * n) return;
    const int i = (int)(e / n), j = (int)(e % n);
    if (j > i) A[e] = A[(size_t)j * n + i];
}

// warp per row GEMV y = A x (A row-major n x n); x staged through shared memory in chunks.
__global__ void __launch_bounds__(256) k_gemv(int n, const double* __restrict__ A, const double* __restrict__ x,
                                              double* __restrict__ y, const int* done) {
    if (done && flag_set(done)) return;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n) return;
    const double* row = A + (size_t)warp * n;
    double s0 = 0.0, s1 = 0.0;
    int k = lane;
    for (; k + 32 < n; k += 64) {
        s0 += __ldg(row + k) * __ldg(x + k);
        s1 += __ldg(row + k + 32) * __ldg(x + k + 32);
    }
    if (k < n) s0 += __ldg(row + k) * __ldg(x + k);
    double s = s0 + s1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(kFull, s, o);
    if (lane == 0) y[warp] = s;
}

// ---- packed symmetric inverse: lower-triangle 64x64 tiles, tile (I,J), J <= I, at I(I+1)/2+J
constexpr int TS = kSymvTile;
constexpr int TP = TS + 1;  // stored row pitch of a packed tile: the pad keeps row and column reads
                            // of the smem copy bank-conflict free, and lets one bulk copy land it

__global__ void k_pack_tiles(int n, const double* __restrict__ full, double* __restrict__ tiles) {
    const int t = blockIdx.x;
    int I = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    while (I * (I + 1) / 2 > t) --I;
    const int J = t - I * (I + 1) / 2;
    double* dst = tiles + (size_t)t * TS * TP;
    for (int e = threadIdx.x; e < TS * TP; e += blockDim.x) {
        const int rr = e / TP, cl = e % TP;
        const int r = I * TS + rr, cc = J * TS + cl;
        dst[e] = (cl < TS && r < n && cc < n) ? full[(size_t)r * n + cc] : 0.0;
    }
}

// one CTA per tile: row sums A_IJ x_J and (off-diagonal tiles) column sums A_IJ^T x_I, each in a
// fixed order, from one read of the tile. The tile (33 KB, constant) arrives by one TMA bulk copy
// (cp.async.bulk + mbarrier transaction count) issued before griddepcontrol.wait, so under PDL it
// streams in while the predecessor drains and no thread spends registers staging it.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(128) k_symv_tiles(int n, int nt, const double* __restrict__ tiles,
                                                    const double* __restrict__ x, double* __restrict__ prow,
                                                    double* __restrict__ pcol, const int* done) {
    pdl_release_early(6);
    __shared__ alignas(128) double A[TS][TP];
    __shared__ double xi[TS], xj[TS];
    __shared__ alignas(8) unsigned long long bar;
    constexpr unsigned kBytes = TS * TP * sizeof(double);
    const int t = blockIdx.x;
    int I = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    while (I * (I + 1) / 2 > t) --I;
    const int J = t - I * (I + 1) / 2;
    const unsigned bar_a = smem_u32(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double* src = tiles + (size_t)t * TS * TP;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"(kBytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(&A[0][0])),
                     "l"(src), "r"(kBytes), "r"(bar_a)
                     : "memory");
    }
    pdl_wait();
    const bool skip = done && flag_set(done);  // x is read regardless: one round trip
    if (threadIdx.x < TS) {
        const int gi = I * TS + threadIdx.x, gj = J * TS + threadIdx.x;
        xi[threadIdx.x] = gi < n ? x[gi] : 0.0;
        xj[threadIdx.x] = gj < n ? x[gj] : 0.0;
    }
    unsigned landed = 0;  // the copy must land before the CTA may exit, even when skipping
    while (!landed)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(landed)
                     : "r"(bar_a), "r"(0u)
                     : "memory");
    __syncthreads();
    if (skip) return;
    if (threadIdx.x < TS) {
        const int r = threadIdx.x;
        double s = 0.0;
        for (int k = 0; k < TS; ++k) s += A[r][k] * xj[k];
        prow[(size_t)t * TS + r] = s;
    } else if (I != J) {
        const int cc = threadIdx.x - TS;
        double s = 0.0;
        for (int k = 0; k < TS; ++k) s += A[k][cc] * xi[k];
        pcol[(size_t)t * TS + cc] = s;
    }
    pdl_release_late(6);
}

// y_I = sum_{J<=I} prow[(I,J)] + sum_{K>I} pcol[(K,I)]: the nt partials of tile row I are split
// over kCombG thread groups (group g takes terms g, g + kCombG, ...), then the groups' sums are
// added in group order — a fixed order, and kCombG times more loads in flight than one thread
// per row (C2's 5931^2 folded operator: 93 partials per row, 19 -> ~5 us).
constexpr int kCombG = 8;
__global__ void __launch_bounds__(TS* kCombG) k_symv_combine(int n, int nt, const double* __restrict__ prow,
                                                             const double* __restrict__ pcol, double* __restrict__ y,
                                                             const int* done) {
    __shared__ double part[kCombG][TS];
    pdl_release_early(8);
    pdl_wait();
    const int I = blockIdx.x, r = threadIdx.x % TS, g = threadIdx.x / TS;
    double s = 0.0;
    for (int t = g; t < nt; t += kCombG) {
        const size_t k = t <= I ? ((size_t)I * (I + 1) / 2 + t) : ((size_t)t * (t + 1) / 2 + I);
        s += (t <= I ? prow : pcol)[k * TS + r];
    }
    part[g][r] = s;
    const bool skip = done && flag_set(done);  // tested after the partial loads
    __syncthreads();
    if (g == 0 && !skip) {
        double tot = part[0][r];
#pragma unroll
        for (int q = 1; q < kCombG; ++q) tot += part[q][r];
        const int gi = I * TS + r;
        if (gi < n) y[gi] = tot;
    }
    pdl_release_late(8);
}

}  // namespace

void pack_symmetric_tiles(Ctx* c, int n, const double* full, double* tiles) {
    const int nt = (n + TS - 1) / TS;
    const int ntiles = nt * (nt + 1) / 2;
    if (ntiles == 0) return;
    k_pack_tiles<<<ntiles, 256, 0, c->stream>>>(n, full, tiles);
    CK_LAUNCH(c);
}

size_t packed_tiles_doubles(int n) {
    const size_t nt = (size_t)(n + TS - 1) / TS;
    return nt * (nt + 1) / 2 * TS * TP;
}
size_t packed_partials_doubles(int n) {
    const size_t nt = (size_t)(n + TS - 1) / TS;
    return nt * (nt + 1) / 2 * TS;
}

void launch_symv_packed(Ctx* c, int n, const double* tiles, const double* x, double* y, double* prow, double* pcol,
                        const int* done, cudaStream_t s) {
    const int nt = (n + TS - 1) / TS;
    const int ntiles = nt * (nt + 1) / 2;
    if (ntiles == 0) return;
    launch_k(c, k_symv_tiles, ntiles, 128, s, n, nt, tiles, x, prow, pcol, done);
    launch_k(c, k_symv_combine, nt, TS * kCombG, s, n, nt, (const double*)prow, (const double*)pcol, y, done);
}

void dense_spd_inverse(Ctx* c, const Mat* Ac, double* inv) {
    const int n = Ac->rows;
    if (n == 0) return;
    DBuf<double> L(c, (size_t)n * n);
    CK(cudaMemsetAsync(L.p, 0, sizeof(double) * (size_t)n * n, c->stream));
    k_csr_to_dense<<<(n + 255) / 256, 256, 0, c->stream>>>(n, Ac->rp.p, Ac->ci.p, Ac->v.p, L.p);
    CK_LAUNCH(c);
    const double shift = 1e-13 * std::max(max_abs(c, Ac), 1.0);  // dense.hpp:27
    for (int kb = 0; kb < n; kb += NB) {
        const int nb = std::min(NB, n - kb);
        k_potrf_diag<<<1, 256, 0, c->stream>>>(n, kb, nb, shift, L.p);
        CK_LAUNCH(c);
        const int below = n - kb - nb;
        if (below > 0) {
            k_trsm_panel<<<(below + 127) / 128, 128, 0, c->stream>>>(n, kb, nb, L.p);
            CK_LAUNCH(c);
            // trailing lower update A22 -= L21 L21^T
            double* L21 = L.p + (size_t)(kb + nb) * n + kb;
            double* A22 = L.p + (size_t)(kb + nb) * n + kb + nb;
            gemm<false, true, true>(c, below, below, nb, -1.0, L21, n, L21, n, 1.0, A22, n);
        }
    }
    // zero the strict upper triangle left from the input
    {
        // X = L^{-1}: start from I, block forward substitution (right-looking)
        DBuf<double> X(c, (size_t)n * n);
        const size_t nn = (size_t)n * n;
        k_identity<<<(unsigned)((nn + 255) / 256), 256, 0, c->stream>>>(n, X.p);
        CK_LAUNCH(c);
        for (int kb = 0; kb < n; kb += NB) {
            const int nb = std::min(NB, n - kb);
            const int ncols = kb + nb;  // X is lower triangular: columns > kb+nb-1 stay zero
            k_trsm_rows<<<(ncols + 127) / 128, 128, 0, c->stream>>>(n, kb, nb, ncols, L.p, X.p);
            CK_LAUNCH(c);
            const int below = n - kb - nb;
            if (below > 0) {
                // X[kb+nb:, :ncols] -= L[kb+nb:, kb:kb+nb] X[kb:kb+nb, :ncols]
                gemm<false, false, false>(c, below, ncols, nb, -1.0, L.p + (size_t)(kb + nb) * n + kb, n,
                                          X.p + (size_t)kb * n, n, 1.0, X.p + (size_t)(kb + nb) * n, n);
            }
        }
        // inv = X^T X (lower half computed, then mirrored)
        gemm<true, false, true>(c, n, n, n, 1.0, X.p, n, X.p, n, 0.0, inv, n);
        k_symmetrize_lower<<<(unsigned)((nn + 255) / 256), 256, 0, c->stream>>>(n, inv);
        CK_LAUNCH(c);
    }
}

void launch_dense_gemv(Ctx* c, int n, const double* Ainv, const double* x, double* y, const int* done,
                       cudaStream_t s) {
    if (n == 0) return;
    const long long threads = (long long)n * 32;
    k_gemv<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(n, Ainv, x, y, done);
    CK_LAUNCH(c);
}

}  // namespace ibmgpu
