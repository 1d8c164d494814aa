// csr.cu — device CSR container, SpMV plan construction and the plain SpMV entry.
//
// Reference: SparseMatrix (sparse.hpp:27-222). The device keeps the exact reference CSR
// (int32 row_ptr/col_idx, f64 values) for every structural operation, plus — for matrices
// whose rows are short (the 5-point lhs2/A/L blocks: 99.3% of lhs2 rows have 5 entries) — a
// SELL-32 copy laid out column-major per 32-row slice so that a warp's 32 rows load 128 B of
// column indices and 256 B of values per step, fully coalesced. Thread-per-row accumulation in
// column order with explicit non-FMA arithmetic reproduces spmv_into (sparse.hpp:101-110)
// bit for bit. Long-row matrices (Galerkin coarse levels, 50-233 entries per row) use a
// CSR-vector kernel with 4..32 threads per row.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>

#include "internal.cuh"
#include "kern.cuh"

namespace ibmgpu {

Mat* mat_new(Ctx* c, int rows, int cols, int nnz) {
    auto* m = new Mat();
    m->rows = rows;
    m->cols = cols;
    m->nnz = nnz;
    m->rp.alloc(c, (size_t)rows + 1);
    m->ci.alloc(c, (size_t)nnz);
    m->v.alloc(c, (size_t)nnz);
    return m;
}

void exclusive_scan_total(Ctx* c, const int* in, int* out, int n) {
    // out[0..n] with out[n] = sum(in[0..n))
    CK(cudaMemsetAsync(out, 0, sizeof(int), c->stream));
    if (n == 0) return;
    size_t tmp = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out + 1, n, c->stream));
    DBuf<char> t(c, tmp);
    CK(cub::DeviceScan::InclusiveSum(t.p, tmp, in, out + 1, n, c->stream));
    c->pdl_fence = 1;  // library kernels write too (CK_LAUNCH)
}

long long exclusive_scan_total64(Ctx* c, const long long* in, long long* out, int n) {
    CK(cudaMemsetAsync(out, 0, sizeof(long long), c->stream));
    if (n == 0) return 0;
    size_t tmp = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out + 1, n, c->stream));
    DBuf<char> t(c, tmp);
    CK(cub::DeviceScan::InclusiveSum(t.p, tmp, in, out + 1, n, c->stream));
    c->pdl_fence = 1;  // library kernels write too (CK_LAUNCH)
    return d2h_scalar(c, out + n);
}

namespace {

__global__ void k_slice_width(int rows, const int* __restrict__ rp, int* __restrict__ width_elems,
                              int* __restrict__ max_row) {
    const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int n_slices = (rows + 31) >> 5;
    if (s >= n_slices) return;
    const int i = s * 32 + lane;
    int len = i < rows ? rp[i + 1] - rp[i] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_down_sync(kFull, len, o));
    if (lane == 0) {
        width_elems[s] = 32 * len;
        atomicMax(max_row, len);
    }
}

__global__ void k_sell_fill(int rows, const int* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ v, const int* __restrict__ off, const int* __restrict__ perm,
                            int* __restrict__ sci, double* __restrict__ sv) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n_slices = (rows + 31) >> 5;
    if (i >= n_slices * 32) return;
    const int s = i >> 5, lane = i & 31;
    const int width = (off[s + 1] - off[s]) >> 5;
    const int row = i < rows ? (perm ? perm[i] : i) : -1;
    const int b = row >= 0 ? rp[row] : 0;
    const int len = row >= 0 ? rp[row + 1] - b : 0;
    for (int k = 0; k < width; ++k) {
        const int dst = off[s] + 32 * k + lane;
        if (k < len) {
            sci[dst] = ci[b + k];
            sv[dst] = v[b + k];
        } else {
            sci[dst] = 0;
            sv[dst] = 0.0;
        }
    }
}

// ---- 16-bit column codes for SELL / SELL-sigma slices (Mat::c16): one warp per slice; the
// slice base is the smallest column below tail0 among its real entries; every entry must land
// in [base, base + 0x8000) or in the top region [tail0, tail0 + 0x8000), else *fail is set.
__global__ void k_c16_build(int n_slices, int n_slots, const int* __restrict__ rp, const int* __restrict__ perm,
                            const int* __restrict__ off, const int* __restrict__ sci, int tail0,
                            unsigned short* __restrict__ code, int* __restrict__ cbase, int* __restrict__ fail) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= n_slices) return;
    const int slot = w * 32 + lane;
    const int row = slot < n_slots ? (perm ? perm[slot] : slot) : -1;
    const int len = row >= 0 ? rp[row + 1] - rp[row] : 0;
    const int o = off[w], width = (off[w + 1] - o) >> 5;
    int mn = INT_MAX;
    for (int k = 0; k < len; ++k) {
        const int col = sci[o + 32 * k + lane];
        if (col < tail0) mn = min(mn, col);
    }
    for (int d = 16; d > 0; d >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, d));
    const int base = mn == INT_MAX ? 0 : mn;
    if (lane == 0) cbase[w] = base;
    for (int k = 0; k < width; ++k) {
        unsigned short cd = 0;
        if (k < len) {
            const int col = sci[o + 32 * k + lane];
            if (col - base >= 0 && col - base < 0x8000)
                cd = (unsigned short)(col - base);
            else if (col >= tail0 && col - tail0 < 0x8000)
                cd = (unsigned short)(0x8000 + (col - tail0));
            else
                *fail = 1;
        }
        code[o + 32 * k + lane] = cd;
    }
}

// Replace the slices' int32 columns by 16-bit codes when every entry fits (see Mat::c16).
void try_c16(Ctx* c, Mat* m, int n_slots) {
    // Off by default since the level-0 transfers (xfer.cuh) no longer stream P_0 / P_0^T, the
    // matrices that fit best: A/B with them gone, S-4M 0.780 vs 0.779 ms, C2 0.313 vs 0.309 ms
    // (the decode costs more than the index bytes save on the remaining levels). IBMGPU_C16=1 on.
    static const bool off_env = [] {
        const char* e = std::getenv("IBMGPU_C16");
        return !(e && e[0] == '1');
    }();
    if (off_env || m->sell_ci.n == 0) return;
    const int n_slices = (n_slots + 31) / 32;
    const int tail0 = m->cols > 0x8000 ? m->cols - 0x8000 : 0;
    DBuf<unsigned short> code(c, m->sell_ci.n);
    DBuf<int> base(c, (size_t)std::max(n_slices, 1)), fail(c, 1);
    CK(cudaMemsetAsync(fail.p, 0, sizeof(int), c->stream));
    k_c16_build<<<(n_slices * 32 + 255) / 256, 256, 0, c->stream>>>(n_slices, n_slots, m->rp.p,
                                                                    m->kind == SPMV_SELLW ? m->perm.p : nullptr,
                                                                    m->sell_off.p, m->sell_ci.p, tail0, code.p,
                                                                    base.p, fail.p);
    CK_LAUNCH(c);
    if (d2h_scalar(c, fail.p)) return;
    m->sell_c16 = std::move(code);
    m->sell_cbase = std::move(base);
    m->c16_tail0 = tail0;
    m->c16 = true;
    m->sell_ci.release();
}

// ---- stencil (DIA-hybrid) plan: classify each row against the band {i-S,i-1,i,i+1,i+S}
__device__ bool band_match(int i, int b, int e, const int* __restrict__ ci, int S, unsigned& mask, int& ext) {
    const int col[5] = {i - S, i - 1, i, i + 1, i + S};
    mask = 0;
    int q = 0;
    for (int k = b; k < e; ++k) {
        const int c = ci[k];
        if (c > i + S) {
            ext = k;
            return true;
        }
        while (q < 5 && col[q] < c) ++q;
        if (q < 5 && col[q] == c) {
            mask |= 1u << q;
            ++q;
        } else {
            return false;
        }
    }
    ext = e;
    return true;
}

__global__ void k_stencil_classify(int rows, const int* __restrict__ rp, const int* __restrict__ ci, int S1, int S2,
                                   unsigned char* __restrict__ mask, int* __restrict__ estart,
                                   int* __restrict__ ecount) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const int b = rp[i], e = rp[i + 1];
    unsigned m = 0;
    int ext = b;
    if (band_match(i, b, e, ci, S1, m, ext)) {
    } else if (S2 > 1 && band_match(i, b, e, ci, S2, m, ext)) {
        m |= 64u;
    } else {
        m = 0;  // generic row: every entry goes to the CSR tail
        ext = b;
    }
    if (e > ext) m |= 32u;
    mask[i] = static_cast<unsigned char>(m);
    estart[i] = ext;
    ecount[i] = e - ext;
}

__global__ void k_stencil_fill(int rows, const int* __restrict__ rp, const int* __restrict__ ci,
                               const double* __restrict__ v, int S1, int S2, const unsigned char* __restrict__ mask,
                               const int* __restrict__ estart, const int* __restrict__ erp, double* __restrict__ sv,
                               int* __restrict__ eci, double* __restrict__ ev) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const unsigned m = mask[i];
    const int S = (m & 64u) ? S2 : S1;
    const int col[5] = {i - S, i - 1, i, i + 1, i + S};
    const int b = rp[i], ext = estart[i];
    int k = b;
    for (int q = 0; q < 5; ++q) {
        double val = 0.0;
        if (m & (1u << q)) {
            while (k < ext && ci[k] != col[q]) ++k;
            val = v[k++];
        }
        sv[(size_t)q * rows + i] = val;
    }
    const int o = erp[i];
    for (int kk = ext; kk < rp[i + 1]; ++kk) {
        eci[o + kk - ext] = ci[kk];
        ev[o + kk - ext] = v[kk];
    }
}

// two most frequent positive offsets > 1 among sampled rows (grid strides of the 5-point blocks)
void detect_strides(Ctx* c, const Mat* m, int& S1, int& S2) {
    S1 = S2 = 0;
    std::vector<std::pair<int, int>> hist;  // (offset, count)
    const int win = std::min(m->rows, 2048);
    for (const double f : {0.0, 0.5, 0.8}) {
        const int r0 = std::min(m->rows - win, static_cast<int>(f * m->rows));
        std::vector<int> rp(static_cast<size_t>(win) + 1);
        d2h(c, rp.data(), m->rp.p + r0, rp.size());
        sync(c);
        const int n = rp[win] - rp[0];
        std::vector<int> ci(static_cast<size_t>(std::max(n, 1)));
        d2h(c, ci.data(), m->ci.p + rp[0], (size_t)n);
        sync(c);
        for (int r = 0; r < win; ++r)
            for (int k = rp[r] - rp[0]; k < rp[r + 1] - rp[0]; ++k) {
                const int off = ci[k] - (r0 + r);
                if (off <= 1) continue;
                auto it = std::find_if(hist.begin(), hist.end(), [&](auto& p) { return p.first == off; });
                if (it == hist.end()) hist.push_back({off, 1});
                else ++it->second;
            }
    }
    std::sort(hist.begin(), hist.end(), [](auto& a, auto& b) { return a.second > b.second; });
    const int thresh = win / 8;  // a stride must appear in >= 1/8 of one window's rows
    if (hist.size() > 0 && hist[0].second >= thresh) S1 = hist[0].first;
    if (hist.size() > 1 && hist[1].second >= thresh) S2 = hist[1].first;
}

// Build the stencil plan if >= 90% of the nonzeros sit in the band; returns true on success.
bool try_stencil(Ctx* c, Mat* m) {
    if (m->rows != m->cols || m->rows < 4096) return false;
    int S1, S2;
    detect_strides(c, m, S1, S2);
    if (S1 <= 1) return false;
    const int n = m->rows;
    DBuf<unsigned char> mask(c, (size_t)n);
    DBuf<int> estart(c, (size_t)n), ecount(c, (size_t)n), erp(c, (size_t)n + 1);
    k_stencil_classify<<<(n + 255) / 256, 256, 0, c->stream>>>(n, m->rp.p, m->ci.p, S1, S2, mask.p, estart.p, ecount.p);
    CK_LAUNCH(c);
    exclusive_scan_total(c, ecount.p, erp.p, n);
    const int n_ext = d2h_scalar(c, erp.p + n);
    if (n_ext > m->nnz / 10) return false;
    m->st_S1 = S1;
    m->st_S2 = S2;
    m->st_v.alloc(c, (size_t)5 * n);
    m->st_eci.alloc(c, (size_t)std::max(n_ext, 1));
    m->st_ev.alloc(c, (size_t)std::max(n_ext, 1));
    k_stencil_fill<<<(n + 255) / 256, 256, 0, c->stream>>>(n, m->rp.p, m->ci.p, m->v.p, S1, S2, mask.p, estart.p, erp.p,
                                                           m->st_v.p, m->st_eci.p, m->st_ev.p);
    CK_LAUNCH(c);
    m->st_mask = std::move(mask);
    m->st_erp = std::move(erp);
    m->kind = SPMV_STENCIL;
    sync(c);
    return true;
}

__global__ void k_diag(int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                       double* __restrict__ d) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int lo = rp[i], hi = rp[i + 1];
    const int e = hi;
    while (lo < hi) {  // lower_bound (sparse.hpp:96)
        const int mid = (lo + hi) >> 1;
        if (ci[mid] < i)
            lo = mid + 1;
        else
            hi = mid;
    }
    d[i] = (lo < e && ci[lo] == i) ? v[lo] : 0.0;
}

__global__ void k_max_abs(int n, const double* __restrict__ v, unsigned long long* out) {
    double m = 0.0;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) m = fmax(m, fabs(v[k]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(kFull, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

}  // namespace

void mat_plan(Ctx* c, Mat* m) {
    m->planned = true;
    if (m->rows == 0) return;
    const int n_slices = (m->rows + 31) / 32;
    DBuf<int> width(c, n_slices), mx(c, 1);
    CK(cudaMemsetAsync(mx.p, 0, sizeof(int), c->stream));
    k_slice_width<<<(n_slices * 32 + 255) / 256, 256, 0, c->stream>>>(m->rows, m->rp.p, width.p, mx.p);
    CK_LAUNCH(c);
    m->max_row = d2h_scalar(c, mx.p);
    const double avg = m->rows ? double(m->nnz) / m->rows : 0.0;
    if (avg <= 12.0 && !std::getenv("IBMGPU_NO_STENCIL") && try_stencil(c, m)) return;
    // Thread-per-row kernels pay one dependent load chain per row: on a small matrix (one short
    // wave) a single long row sets the kernel time (S-4M L6 P^T: 1-entry rows plus a few of 86,
    // 16 us). There, rows longer than max(16, 4 x mean) go to the warp-per-row path instead.
    const bool small = m->rows < 65536;
    const int kWide = small ? std::max(16, 4 * static_cast<int>(std::ceil(avg))) : 96;
    if (avg <= 12.0 && m->max_row <= 48 && (!small || m->max_row <= kWide)) {
        m->kind = SPMV_SELL;
        m->sell_off.alloc(c, (size_t)n_slices + 1);
        exclusive_scan_total(c, width.p, m->sell_off.p, n_slices);
        const int total = d2h_scalar(c, m->sell_off.p + n_slices);
        m->sell_ci.alloc(c, (size_t)total);
        m->sell_v.alloc(c, (size_t)total);
        k_sell_fill<<<(n_slices * 32 + 255) / 256, 256, 0, c->stream>>>(m->rows, m->rp.p, m->ci.p, m->v.p,
                                                                        m->sell_off.p, nullptr, m->sell_ci.p,
                                                                        m->sell_v.p);
        CK_LAUNCH(c);
        try_c16(c, m, m->rows);
        return;
    }
    std::vector<int> rp(static_cast<size_t>(m->rows) + 1);
    d2h(c, rp.data(), m->rp.p, rp.size());
    sync(c);
    // thread-per-row SELL-sigma for the rows of <= 96 entries; the few longer rows (the body
    // tail of the Galerkin levels: force unknowns couple to many aggregates) get a warp each with
    // an in-order sum, so one long row no longer sends the whole level to the adaptive kernel
    {
        constexpr int kSigma = 512;
        std::vector<int> shortrows, longrows;
        long long long_nnz = 0;
        for (int i = 0; i < m->rows; ++i) {
            const int l = rp[i + 1] - rp[i];
            if (l <= kWide) {
                shortrows.push_back(i);
            } else {
                longrows.push_back(i);
                long_nnz += l;
            }
        }
        const int ns = static_cast<int>(shortrows.size());
        // (every row > 96 on its own warp — i.e. no CSR-adaptive at all — measured 1.69 vs 1.01 ms
        // per S-4M iteration: the in-order add chain is too long for the 150-2000-entry coarse rows)
        const bool few_long = longrows.size() * 20 <= (size_t)m->rows && long_nnz * 3 <= (long long)m->nnz;
        // (SELL-sigma for the 150-entry S-4M level-3 rows measured no faster than adaptive)
        // thread per row needs rows to fill the machine: a 22k-row, 33-entry level (C2 L3 P) has
        // 7% of the thread slots busy and ran 19 us as SELL-sigma vs 14 us on the adaptive kernel
        const bool enough_rows = m->rows >= 65536 || avg <= 8.0;
        if (few_long && ns > 0 && enough_rows) {
            // SELL-32-sigma: sort short rows by length within 512-slot windows; accept if padding <= 25%
            std::vector<int> perm(shortrows);
            // windows are independent: sort them on all host threads (same result as serial)
            const int n_win = (ns + kSigma - 1) / kSigma;
#pragma omp parallel for schedule(static) if (n_win >= 64)
            for (int wi = 0; wi < n_win; ++wi) {
                const int w0 = wi * kSigma, w1 = std::min(ns, w0 + kSigma);
                std::stable_sort(perm.begin() + w0, perm.begin() + w1,
                                 [&](int a, int b) { return rp[a + 1] - rp[a] > rp[b + 1] - rp[b]; });
            }
            const int ss = (ns + 31) / 32;
            std::vector<int> off(static_cast<size_t>(ss) + 1, 0);
            long long total = 0;
            for (int sl = 0; sl < ss; ++sl) {
                int w = 0;
                for (int i = sl * 32; i < std::min(ns, sl * 32 + 32); ++i)
                    w = std::max(w, rp[perm[i] + 1] - rp[perm[i]]);
                total += 32ll * w;
                off[sl + 1] = static_cast<int>(total);
            }
            if (total <= (long long)(1.25 * (m->nnz - long_nnz)) + 32 * 64 && total < (1ll << 31)) {
                m->kind = SPMV_SELLW;
                m->n_short = ns;
                m->n_long = static_cast<int>(longrows.size());
                m->perm.alloc(c, perm.size());
                h2d(c, m->perm.p, perm.data(), perm.size());
                m->long_rows.alloc(c, std::max<size_t>(longrows.size(), 1));
                h2d(c, m->long_rows.p, longrows.data(), longrows.size());
                m->sell_off.alloc(c, off.size());
                h2d(c, m->sell_off.p, off.data(), off.size());
                m->sell_ci.alloc(c, (size_t)std::max(total, 1ll));
                m->sell_v.alloc(c, (size_t)std::max(total, 1ll));
                k_sell_fill<<<(ss * 32 + 255) / 256, 256, 0, c->stream>>>(ns, m->rp.p, m->ci.p, m->v.p, m->sell_off.p,
                                                                          m->perm.p, m->sell_ci.p, m->sell_v.p);
                CK_LAUNCH(c);
                try_c16(c, m, ns);
                sync(c);
                return;
            }
        }
    }
    m->kind = SPMV_VECTOR;
    plan_adaptive_from(c, m, rp);
}

void mat_plan_adaptive(Ctx* c, Mat* m) {
    if (m->n_blocks > 0 || m->rows == 0) return;
    std::vector<int> rp(static_cast<size_t>(m->rows) + 1);
    d2h(c, rp.data(), m->rp.p, rp.size());
    sync(c);
    plan_adaptive_from(c, m, rp);
}

// CSR-adaptive chunks (kern.cuh k_spmv_adapt / coarse.cuh), planned on the host from row_ptr
void plan_adaptive_from(Ctx* c, Mat* m, const std::vector<int>& rp) {
    const double avg = m->rows ? double(m->nnz) / m->rows : 0.0;
    {
        // ~2k nonzeros per CTA, but small matrices use smaller chunks so the grid still fills every
        // SM (>= 4 CTAs each; 8 and 2 measured slower): these levels are latency-bound
        const int kChunkNnz = std::clamp(static_cast<int>(m->nnz / std::max(1, c->num_sms * 4)), 512, 2048);
        // rows much longer than the mean never share a CTA with short rows
        const int kOwnCta = std::max(128, static_cast<int>(4.0 * avg));
        std::vector<int4> meta;
        std::vector<int2> lrow;
        int parts = 0;
        int r = 0;
        while (r < m->rows) {
            const int len = rp[r + 1] - rp[r];
            if (len > kOwnCta) {  // long row: one CTA per kRowChunk entries (at least one)
                const int nch = (len + kRowChunk - 1) / kRowChunk;
                const int lid = static_cast<int>(lrow.size());
                lrow.push_back(make_int2(parts, nch));
                for (int q = 0; q < nch; ++q) meta.push_back(make_int4(r, q, 0, lid));
                parts += nch;
                ++r;
                continue;
            }
            int r1 = r, nz = 0;
            while (r1 < m->rows) {
                const int l = rp[r1 + 1] - rp[r1];
                if (l > kOwnCta || (r1 > r && (nz + l > kChunkNnz || r1 - r >= 256))) break;
                nz += l;
                ++r1;
            }
            const double mean = double(nz) / (r1 - r);
            static const int epl = [] {  // target entries per lane (IBMGPU_ADAPT_EPL, A/B)
                const char* e = std::getenv("IBMGPU_ADAPT_EPL");
                return e ? std::max(1, std::atoi(e)) : 8;  // 8: S-4M -0.3%, C2 -0.8% vs 4
            }();
            int tpr = 2;
            while (tpr < 32 && tpr * epl < mean) tpr *= 2;
            // keep at least a few rows per group for short-row chunks
            while (tpr > 2 && (r1 - r) > (kBlock / tpr) * 8) tpr /= 2;
            // whole passes only: a chunk of 17 rows on 8 groups costs 3 latency-bound passes, 16 cost 2
            const int ngrp = kBlock / tpr;
            if (r1 - r > ngrp && (r1 - r) % ngrp) r1 = r + ((r1 - r) / ngrp) * ngrp;
            meta.push_back(make_int4(r, r1, tpr, 0));
            r = r1;
        }
        m->n_blocks = static_cast<int>(meta.size());
        m->n_lrows = static_cast<int>(lrow.size());
        m->blk_meta.alloc(c, meta.size());
        h2d(c, m->blk_meta.p, meta.data(), meta.size());
        m->lrow.alloc(c, std::max<size_t>(lrow.size(), 1));
        h2d(c, m->lrow.p, lrow.data(), lrow.size());
        m->lpart.alloc(c, (size_t)std::max(parts, 1));
        m->lcnt.alloc(c, std::max<size_t>(lrow.size(), 1));
        CK(cudaMemsetAsync(m->lcnt.p, 0, sizeof(unsigned) * std::max<size_t>(lrow.size(), 1), c->stream));
        sync(c);
    }
}

Mat* mat_upload(Ctx* c, int rows, int cols, int nnz, const int* rp, const int* ci, const double* v) {
    require(rows >= 0 && cols >= 0 && nnz >= 0, "csr_upload: negative dimension");
    require(rp[0] == 0 && rp[rows] == nnz, "csr_upload: row_ptr inconsistent with nnz");
    Mat* m = mat_new(c, rows, cols, nnz);
    h2d(c, m->rp.p, rp, (size_t)rows + 1);
    h2d(c, m->ci.p, ci, (size_t)nnz);
    h2d(c, m->v.p, v, (size_t)nnz);
    mat_plan(c, m);
    return m;
}

void mat_download(Ctx* c, const Mat* m, int* rp, int* ci, double* v) {
    d2h(c, rp, m->rp.p, (size_t)m->rows + 1);
    if (ci) d2h(c, ci, m->ci.p, (size_t)m->nnz);
    if (v) d2h(c, v, m->v.p, (size_t)m->nnz);
    sync(c);
}

void spmv(Ctx* c, Mat* A, const double* x, double* y) {
    if (!A->planned) mat_plan(c, A);
    launch_spmv(c, A, XPlain{x}, EpiStore{y}, c->stream);
}

void diag_of(Ctx* c, const Mat* A, double* d) {
    const int n = A->rows < A->cols ? A->rows : A->cols;
    if (n == 0) return;
    k_diag<<<(n + 255) / 256, 256, 0, c->stream>>>(n, A->rp.p, A->ci.p, A->v.p, d);
    CK_LAUNCH(c);
}

double max_abs(Ctx* c, const Mat* A) {
    if (A->nnz == 0) return 0.0;
    DBuf<unsigned long long> out(c, 1);
    CK(cudaMemsetAsync(out.p, 0, sizeof(unsigned long long), c->stream));
    k_max_abs<<<elem_grid(c, A->nnz), 256, 0, c->stream>>>(A->nnz, A->v.p, out.p);
    CK_LAUNCH(c);
    const unsigned long long bits = d2h_scalar(c, out.p);
    double r;
    memcpy(&r, &bits, sizeof(r));
    return r;
}

}  // namespace ibmgpu
