// Dense folding of the smallest SA levels into the coarse operator.
//
// The V(1,1) cycle below level l is a fixed linear map of the level's right-hand side. With the
// damped-Jacobi smoother W = diag(omega / a_ii) (amg.hpp:204-233), the cycle at level l is
//
//     M_l = 2 W - W A W + B^T M_{l+1} B,      B = P^T (I - A W)      (A symmetric, W diagonal)
//
// and M_L = A_c^{-1} at the coarsest level (dense.hpp:20-40). The last levels of a hierarchy are
// tiny (a few thousand rows, mostly the identity tail of body rows) and cost ~5 us of launch and
// latency per SpMV, four SpMVs per level per cycle. Folding them into one dense symmetric operator
// replaces those launches with a slightly larger packed SYMV (dense.cu). It is the same operator,
// with different rounding. Levels are folded from the bottom while the dense dimension grows by
// at most kFoldGrowth per level and stays under kFoldMax. IBMGPU_FOLD=0 turns it off.
// Structure, aggregates and the level matrices are untouched: only the V-cycle stops earlier.
#include <algorithm>
#include <cstdlib>

#include "amg.cuh"

namespace ibmgpu {
namespace {

constexpr int kFoldMax = 8192;
constexpr double kFoldGrowth = 1.8;

// out[r, :] = sum over row r of S of S[r,k] X[k, :]   (X row-major with ncols columns), fixed order
__global__ void __launch_bounds__(256) k_rowcomb(int ncols, const int* __restrict__ rp, const int* __restrict__ ci,
                                                 const double* __restrict__ v, const double* __restrict__ X,
                                                 double* __restrict__ out) {
    const int r = blockIdx.x;
    const int b = rp[r], e = rp[r + 1];
    for (int j = threadIdx.x; j < ncols; j += blockDim.x) {
        double s = 0.0;
        int k = b;
        for (; k + 3 < e; k += 4) {
            const double x0 = X[(size_t)ci[k] * ncols + j], x1 = X[(size_t)ci[k + 1] * ncols + j];
            const double x2 = X[(size_t)ci[k + 2] * ncols + j], x3 = X[(size_t)ci[k + 3] * ncols + j];
            s = fma(v[k], x0, s);
            s = fma(v[k + 1], x1, s);
            s = fma(v[k + 2], x2, s);
            s = fma(v[k + 3], x3, s);
        }
        for (; k < e; ++k) s = fma(v[k], X[(size_t)ci[k] * ncols + j], s);
        out[(size_t)r * ncols + j] = s;
    }
}

// dst (cols x rows) = src (rows x cols)^T, 32x32 tiles through shared memory
__global__ void k_transpose_dense(int rows, int cols, const double* __restrict__ src, double* __restrict__ dst) {
    __shared__ double t[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int r = by + y, cc = bx + threadIdx.x;
        if (r < rows && cc < cols) t[y][threadIdx.x] = src[(size_t)r * cols + cc];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int r = bx + y, cc = by + threadIdx.x;  // dst row = src column
        if (r < cols && cc < rows) dst[(size_t)r * rows + cc] = t[threadIdx.x][y];
    }
}

// M += 2 W - W A W   (thread per row: each thread writes only its own row)
__global__ void k_fold_smoother(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                const double* __restrict__ v, const double* __restrict__ wd, double* __restrict__ M) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double wi = wd[i];
    double* row = M + (size_t)i * n;
    for (int k = rp[i]; k < rp[i + 1]; ++k) row[ci[k]] -= wi * v[k] * wd[ci[k]];
    row[i] += 2.0 * wi;
}

// The packed SYMV reads off-diagonal tiles from the lower triangle only, diagonal 64x64 tiles in
// full: make those exactly symmetric.
__global__ void k_sym_diag_tiles(int n, int ts, double* __restrict__ M) {
    const int base = blockIdx.x * ts;
    for (int t = threadIdx.x; t < ts * ts; t += blockDim.x) {
        const int r = t / ts, k = t % ts;
        if (r <= k || base + r >= n) continue;
        double* a = M + (size_t)(base + r) * n + base + k;
        double* b = M + (size_t)(base + k) * n + base + r;
        const double m = 0.5 * (*a + *b);
        *a = m;
        *b = m;
    }
}

}  // namespace

void fold_tail(Ctx* c, Hier* h, int tile) {
    const char* ev = std::getenv("IBMGPU_FOLD");
    if ((ev && std::atoi(ev) == 0) || std::getenv("IBMGPU_FUSE_ROWS")) return;
    const int L = (int)h->levels.size();
    int nf = 0, dim = h->n_c;
    while (L - nf - 1 >= 1) {  // level 0 always stays sparse
        const int n = h->levels[L - nf - 1]->A->rows;
        if (n > kFoldMax || n > kFoldGrowth * dim) break;
        ++nf;
        dim = n;
    }
    if (nf == 0) return;
    cudaStream_t s = c->stream;
    const double* Mcur = h->coarse_inv.p;
    int m = h->n_c;
    DBuf<double> Mown;
    for (int l = L - 1; l >= L - nf; --l) {
        Level& lv = *h->levels[l];
        const int n = lv.A->rows;
        // B = P^T (I - A W), held as B^T (n x m) so both products below read rows
        Mat* PtA = spmm_rows(c, lv.Pt, 0, lv.Pt->rows, lv.A);
        Mat* PtAW = scale(c, PtA, 2, 0.0, lv.wd.p);
        delete PtA;
        Mat* B = add(c, 1.0, lv.Pt, -1.0, PtAW);
        delete PtAW;
        Mat* Bt = transpose(c, B);
        delete B;
        DBuf<double> Gt(c, (size_t)n * m), G(c, (size_t)m * n);
        k_rowcomb<<<n, 256, 0, s>>>(m, Bt->rp.p, Bt->ci.p, Bt->v.p, Mcur, Gt.p);  // (M_{l+1} B)^T
        CK_LAUNCH(c);
        k_transpose_dense<<<dim3((m + 31) / 32, (n + 31) / 32), dim3(32, 8), 0, s>>>(n, m, Gt.p, G.p);
        CK_LAUNCH(c);
        DBuf<double> Mn(c, (size_t)n * n);
        k_rowcomb<<<n, 256, 0, s>>>(n, Bt->rp.p, Bt->ci.p, Bt->v.p, G.p, Mn.p);  // B^T M_{l+1} B
        CK_LAUNCH(c);
        k_fold_smoother<<<(n + 255) / 256, 256, 0, s>>>(n, lv.A->rp.p, lv.A->ci.p, lv.A->v.p, lv.wd.p, Mn.p);
        CK_LAUNCH(c);
        delete Bt;
        Mown = std::move(Mn);
        Mcur = Mown.p;
        m = n;
    }
    k_sym_diag_tiles<<<(m + tile - 1) / tile, 256, 0, s>>>(m, tile, Mown.p);
    CK_LAUNCH(c);
    h->n_fold = nf;
    h->n_dense = m;
    h->dense = std::move(Mown);
}

}  // namespace ibmgpu
