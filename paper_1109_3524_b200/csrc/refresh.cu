// refresh.cu — refresh_body_operators (operators.hpp:445-450) for a moving body, re-assembling
// only what the body touches. Bit-exact with the full assembly (coupled_system in body.cu):
//
//   Q    = [G  E^T]                       concat_cols, as before (operators.hpp:394-404)
//   Q^T  = [G^T ; E]                       G^T is cached; Q^T's rows are G^T's rows then E's
//                                          (transpose of a column concat = row concat)
//   raw  = Q^T B^N Q                       (operators.hpp:408-417)
//     pressure-pressure block  G^T B^N G   invariant: cached from the first full assembly
//     pressure rows, body cols G^T B^N E^T only rows in a band around the body are non-empty;
//                                          Gustavson accumulates column n_p+b of row i over
//                                          k in (G^T B^N)[i,:] in k order, the same sequence
//                                          triple(G^T_band, B^N, E^T) forms
//     body rows                E B^N Q     triple(Q^T body rows, B^N, Q)
//   lhs2 = pin(sym(raw), 0)                sym of an entry is 0.5 raw_ij + 0.5 raw_ji with exact
//                                          zeros dropped (add_sparse); the body-involving entries
//                                          only need the body-involving raw entries, so
//                                          sym(Bx) of the body part Bx equals those entries of
//                                          sym(raw); pin drops row/column 0 outside (0,0)
//   lhs2 = merge(Lpp, pin'(sym(Bx)))       pressure rows: cached Lpp row (cols < n_p) followed by
//                                          the body columns; body rows: sym(Bx) rows
// The pressure block being bitwise invariant under body motion is measured in SURVEY.md App. A
// (probe6) and checked on every moving step by tests/test_gpu_parity_steps.py against the
// reference's own lhs2.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "kern.cuh"
#include "refresh.cuh"
#include "small_rows.cuh"

namespace ibmgpu {

Mat* concat_rows(Ctx* c, std::vector<Mat*>& parts, int rows, int cols);  // sparse_ops.cu

namespace {

inline int nblk(long long n, int b = 256) { return (int)((n + b - 1) / b); }

// rows [r0, r1) of A (entries copied)
__global__ void k_slice_rp(int rows, const int* __restrict__ rp, int r0, int* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= rows) out[i] = rp[r0 + i] - rp[r0];
}

// entries of rows [0, rows) with column < colmax (count, then fill)
__global__ void k_block_lt(int rows, int colmax, const int* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ v, int* __restrict__ cnt, const int* __restrict__ orp,
                           int* __restrict__ oci, double* __restrict__ ov) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    int n = 0;
    const int o = orp ? orp[i] : 0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int col = ci[k];
        if (col >= colmax) break;  // columns increase along the row
        if (oci) {
            oci[o + n] = col;
            ov[o + n] = v[k];
        }
        ++n;
    }
    if (cnt) cnt[i] = n;
}

// vertical concatenation [A ; B] with exact zeros dropped (Q^T = transpose of the zero-free Q)
__global__ void k_vcat(int ra, int rb, const int* __restrict__ arp, const int* __restrict__ aci,
                       const double* __restrict__ av, const int* __restrict__ brp, const int* __restrict__ bci,
                       const double* __restrict__ bv, int* __restrict__ cnt, const int* __restrict__ orp,
                       int* __restrict__ oci, double* __restrict__ ov) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ra + rb) return;
    const bool top = i < ra;
    const int r = top ? i : i - ra;
    const int* rp = top ? arp : brp;
    const int* ci = top ? aci : bci;
    const double* v = top ? av : bv;
    int n = 0;
    const int o = orp ? orp[i] : 0;
    for (int k = rp[r]; k < rp[r + 1]; ++k)
        if (v[k] != 0.0) {
            if (oci) {
                oci[o + n] = ci[k];
                ov[o + n] = v[k];
            }
            ++n;
        }
    if (cnt) cnt[i] = n;
}

// lhs2 row i: Lpp row (i < n_p; already pinned) then sym(Bx) row i without the pin row/column
__global__ void k_merge(int n, int n_p, int pin, const int* __restrict__ lrp, const int* __restrict__ lci,
                        const double* __restrict__ lv, const int* __restrict__ srp, const int* __restrict__ sci,
                        const double* __restrict__ sv, int* __restrict__ cnt, const int* __restrict__ orp,
                        int* __restrict__ oci, double* __restrict__ ov) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int m = 0;
    const int o = orp ? orp[i] : 0;
    if (i < n_p)
        for (int k = lrp[i]; k < lrp[i + 1]; ++k) {
            if (oci) {
                oci[o + m] = lci[k];
                ov[o + m] = lv[k];
            }
            ++m;
        }
    if (i != pin)
        for (int k = srp[i]; k < srp[i + 1]; ++k) {
            const int col = sci[k];
            if (col == pin) continue;
            IBM_DCHECK(i >= n_p || col >= n_p);  // the cached pressure block holds every pressure column
            if (oci) {
                oci[o + m] = col;
                ov[o + m] = sv[k];
            }
            ++m;
        }
    if (cnt) cnt[i] = m;
}

// pressure columns (< n_p) present in the body rows of raw
__global__ void k_mark_cols(int nnz, int n_p, const int* __restrict__ ci, int* __restrict__ flag) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nnz && ci[k] < n_p) flag[ci[k]] = 1;
}
__global__ void k_flag_index(int n, const int* __restrict__ flag, const int* __restrict__ pos, int* __restrict__ idx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) idx[pos[i]] = i;
}
// rows idx[0..m) of A
__global__ void k_gather_cnt(int m, const int* __restrict__ idx, const int* __restrict__ rp, int* __restrict__ cnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < m) cnt[r] = rp[idx[r] + 1] - rp[idx[r]];
}
__global__ void k_gather_fill(int m, const int* __restrict__ idx, const int* __restrict__ rp, const int* __restrict__ ci,
                              const double* __restrict__ v, const int* __restrict__ orp, int* __restrict__ oci,
                              double* __restrict__ ov) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const int s = rp[idx[r]], n = rp[idx[r] + 1] - s, o = orp[r];
    for (int k = 0; k < n; ++k) {
        oci[o + k] = ci[s + k];
        ov[o + k] = v[s + k];
    }
}
// Bx (n x n): pressure rows idx[r] hold Xpb row r shifted to columns n_p + b; rows [n_p, n) hold
// Xb's rows; every other row is empty (pos: exclusive scan of the row flags)
__global__ void k_body_part2(int n, int n_p, const int* __restrict__ flag, const int* __restrict__ pos,
                             const int* __restrict__ prp, const int* __restrict__ pci, const double* __restrict__ pv,
                             const int* __restrict__ brp, const int* __restrict__ bci, const double* __restrict__ bv,
                             int* __restrict__ cnt, const int* __restrict__ orp, int* __restrict__ oci,
                             double* __restrict__ ov) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int n_out = 0;
    const int o = orp ? orp[i] : 0;
    const int* rp = nullptr;
    const int* ci = nullptr;
    const double* v = nullptr;
    int r = 0, shift = 0;
    if (i >= n_p) {
        rp = brp, ci = bci, v = bv, r = i - n_p;
    } else if (flag[i]) {
        rp = prp, ci = pci, v = pv, r = pos[i], shift = n_p;
    }
    if (rp)
        for (int k = rp[r]; k < rp[r + 1]; ++k) {
            if (oci) {
                oci[o + n_out] = shift + ci[k];
                ov[o + n_out] = v[k];
            }
            ++n_out;
        }
    if (cnt) cnt[i] = n_out;
}

// Two-pass (count, scan, fill) construction of a rows x cols matrix from a row kernel.
template <class Launch>
Mat* build_rows(Ctx* c, int rows, int cols, Launch&& launch) {
    DBuf<int> cnt(c, (size_t)rows + 1);
    Mat* m = mat_new(c, rows, cols, 0);
    if (rows) {
        launch(cnt.p, (const int*)nullptr, (int*)nullptr, (double*)nullptr);
        CK_LAUNCH(c);
    }
    exclusive_scan_total(c, cnt.p, m->rp.p, rows);
    m->nnz = rows ? d2h_scalar(c, m->rp.p + rows) : 0;
    m->ci.alloc(c, (size_t)std::max(m->nnz, 1));
    m->v.alloc(c, (size_t)std::max(m->nnz, 1));
    if (rows && m->nnz) {
        launch((int*)nullptr, (const int*)m->rp.p, m->ci.p, m->v.p);
        CK_LAUNCH(c);
    }
    return m;
}

// ---- small triple products D = (A B) C, one warp per row of A (the body strips of the refresh)
// Gustavson per stage exactly as spmm_rows (sparse.hpp:226-268): products in A-row order then
// B-row order, each column summed from 0.0 in that order, columns sorted, cancelled entries kept.
// Products of a row are staged in shared memory, stably ranked by column (O(n^2) in the warp —
// rows here have at most kSmallCap products), and each column's run is summed by one lane.
__global__ void __launch_bounds__(kSmallWarps * 32)
    k_triple_small(int rows, const int* __restrict__ arp, const int* __restrict__ aci, const double* __restrict__ av,
                   const int* __restrict__ brp, const int* __restrict__ bci, const double* __restrict__ bv,
                   const int* __restrict__ crp, const int* __restrict__ cci, const double* __restrict__ cv,
                   int* __restrict__ cnt, const int* __restrict__ orp, int* __restrict__ oci, double* __restrict__ ov) {
    __shared__ SmallRow ws[kSmallWarps];
    __shared__ int tci[kSmallWarps][kSmallCap];
    __shared__ double tv[kSmallWarps][kSmallCap];
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    SmallRow& w = ws[wi];
    for (int i = blockIdx.x * kSmallWarps + wi; i < rows; i += gridDim.x * kSmallWarps) {
        // stage 1: T = A(i,:) B
        int n = small_expand(w, aci, av, arp[i], arp[i + 1], brp, bci, bv, lane);
        int u = small_reduce(w, n, lane);
        for (int q = lane; q < u; q += 32) {
            tci[wi][q] = w.scol[q];
            tv[wi][q] = w.sval[q];
        }
        __syncwarp();
        // stage 2: D(i,:) = T C
        n = small_expand(w, tci[wi], tv[wi], 0, u, crp, cci, cv, lane);
        u = small_reduce(w, n, lane);
        if (cnt) {
            if (lane == 0) cnt[i] = u;
        } else {
            const int o = orp[i];
            for (int q = lane; q < u; q += 32) {
                oci[o + q] = w.scol[q];
                ov[o + q] = w.sval[q];
            }
        }
        __syncwarp();
    }
}

// products per row of A*B (stage 1) and the stage-2 bound sum over A row of (B row len * max C row)
__global__ void k_small_bound(int rows, const int* __restrict__ arp, const int* __restrict__ aci,
                              const int* __restrict__ brp, const int* __restrict__ bci, const int* __restrict__ crp,
                              int* __restrict__ over) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    long long p1 = 0, p2 = 0;
    for (int k = arp[i]; k < arp[i + 1]; ++k) {
        const int kk = aci[k];
        p1 += brp[kk + 1] - brp[kk];
        for (int t = brp[kk]; t < brp[kk + 1]; ++t) p2 += crp[bci[t] + 1] - crp[bci[t]];
    }
    if (p1 > kSmallCap || p2 > kSmallCap) *over = 1;
}

}  // namespace

// (A B) C with one warp per row when every row stays under kSmallCap products per stage;
// otherwise the general sliced product. Bit-exact with triple_product either way.
Mat* triple_small(Ctx* c, const Mat* A, const Mat* B, const Mat* Cm) {
    require(A->cols == B->rows && B->cols == Cm->rows, "sliced_triple_product: dimension mismatch");
    const int rows = A->rows;
    if (rows > 0) {
        DBuf<int> over(c, 1);
        CK(cudaMemsetAsync(over.p, 0, sizeof(int), c->stream));
        k_small_bound<<<nblk(rows), 256, 0, c->stream>>>(rows, A->rp.p, A->ci.p, B->rp.p, B->ci.p, Cm->rp.p, over.p);
        CK_LAUNCH(c);
        if (d2h_scalar(c, over.p)) return triple_product(c, A, B, Cm, std::max(1, rows), nullptr, nullptr);
    }
    const int grid = std::max(1, std::min(nblk(rows, kSmallWarps), c->num_sms * 8));
    return build_rows(c, rows, Cm->cols, [&](int* cnt, const int* orp, int* oci, double* ov) {
        k_triple_small<<<grid, kSmallWarps * 32, 0, c->stream>>>(rows, A->rp.p, A->ci.p, A->v.p, B->rp.p, B->ci.p,
                                                                B->v.p, Cm->rp.p, Cm->ci.p, Cm->v.p, cnt, orp, oci, ov);
    });
}

Mat* row_slice(Ctx* c, const Mat* A, int r0, int r1) {
    r0 = std::clamp(r0, 0, A->rows);
    r1 = std::clamp(r1, r0, A->rows);
    const int rows = r1 - r0;
    int k[2] = {0, 0};
    d2h(c, k, A->rp.p + r0, 1);
    d2h(c, k + 1, A->rp.p + r1, 1);
    sync(c);
    Mat* m = mat_new(c, rows, A->cols, k[1] - k[0]);
    k_slice_rp<<<nblk(rows + 1), 256, 0, c->stream>>>(rows, A->rp.p, r0, m->rp.p);
    CK_LAUNCH(c);
    d2d(c, m->ci.p, A->ci.p + k[0], (size_t)(k[1] - k[0]));
    d2d(c, m->v.p, A->v.p + k[0], (size_t)(k[1] - k[0]));
    return m;
}

Mat* block_lt(Ctx* c, const Mat* A, int rows, int colmax) {
    return build_rows(c, rows, A->cols, [&](int* cnt, const int* orp, int* oci, double* ov) {
        k_block_lt<<<nblk(rows), 256, 0, c->stream>>>(rows, colmax, A->rp.p, A->ci.p, A->v.p, cnt, orp, oci, ov);
    });
}

Mat* vcat(Ctx* c, const Mat* A, const Mat* B) {
    require(A->cols == B->cols, "vcat: column mismatch");
    const int rows = A->rows + B->rows;
    return build_rows(c, rows, A->cols, [&](int* cnt, const int* orp, int* oci, double* ov) {
        k_vcat<<<nblk(rows), 256, 0, c->stream>>>(A->rows, B->rows, A->rp.p, A->ci.p, A->v.p, B->rp.p, B->ci.p,
                                                  B->v.p, cnt, orp, oci, ov);
    });
}

bool mat_equal(Ctx* c, const Mat* A, const Mat* B) {
    if (A->rows != B->rows || A->cols != B->cols || A->nnz != B->nnz) return false;
    std::vector<int> ra(A->rows + 1), rb(B->rows + 1), ca(A->nnz), cb(B->nnz);
    std::vector<double> va(A->nnz), vb(B->nnz);
    mat_download(c, A, ra.data(), ca.data(), va.data());
    mat_download(c, B, rb.data(), cb.data(), vb.data());
    return ra == rb && ca == cb && std::memcmp(va.data(), vb.data(), sizeof(double) * va.size()) == 0;
}

bool pattern_symmetric(Ctx* c, const Mat* A) {
    if (A->rows != A->cols) return false;
    Mat* T = transpose(c, A);
    std::vector<int> ra(A->rows + 1), rt(A->rows + 1), ca(A->nnz), ct(A->nnz);
    mat_download(c, A, ra.data(), ca.data(), nullptr);
    mat_download(c, T, rt.data(), ct.data(), nullptr);
    delete T;
    return ra == rt && ca == ct;
}

bool RefreshCache::init(Ctx* c, const Mat* G, const Mat* BN, const Mat* lhs2, int n_p_, int pin_, int n_order_) {
    if (!pattern_symmetric(c, BN)) return false;
    n_p = n_p_;
    pin = pin_;
    n_order = n_order_;
    delete GT;
    delete Lpp;
    GT = transpose(c, G);
    Lpp = block_lt(c, lhs2, n_p, n_p);
    return true;
}

RefreshCache::~RefreshCache() {
    delete GT;
    delete Lpp;
}

void coupled_refresh(Ctx* c, const RefreshCache& rc, const Mat* G, const Mat* E, const Mat* BN, Mat** Q, Mat** QT,
                     Mat** lhs2) {
    const int n_p = rc.n_p, n_b2 = E->rows, n = n_p + n_b2;
    static const bool prof = std::getenv("IBMGPU_SETUP_PROFILE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!prof) return;
        sync(c);
        const auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[refresh]   %-12s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    };
    {
        Mat* Et0 = transpose(c, E);
        *Q = concat_cols(c, G, Et0);  // drops exact zeros, as the reference's triplets do
        delete Et0;
    }
    *QT = vcat(c, rc.GT, E);
    lap("Q, QT");
    // body rows of raw: (Q^T body rows) B^N Q, in Gustavson order exactly as the full product
    Mat* QTb = row_slice(c, *QT, n_p, n);
    Mat* Xb = triple_small(c, QTb, BN, *Q);
    Mat* Et = transpose(c, QTb);  // the E^T block of Q (zero-free)
    delete QTb;
    lap("Xb");
    // pressure rows with body coupling: raw is structurally symmetric (B^N's pattern is, checked
    // at init), so they are exactly the pressure columns of raw's body rows. Their body columns
    // are G^T B^N E^T on those rows: Gustavson accumulates column n_p + b of row i over k in
    // (G^T B^N)[i,:] in k order, the sequence triple(G^T rows, B^N, E^T) forms.
    DBuf<int> flag(c, (size_t)n_p), pos(c, (size_t)n_p + 1);
    CK(cudaMemsetAsync(flag.p, 0, sizeof(int) * (size_t)n_p, c->stream));
    if (Xb->nnz) {
        k_mark_cols<<<nblk(Xb->nnz), 256, 0, c->stream>>>(Xb->nnz, n_p, Xb->ci.p, flag.p);
        CK_LAUNCH(c);
    }
    exclusive_scan_total(c, flag.p, pos.p, n_p);
    const int m = d2h_scalar(c, pos.p + n_p);
    DBuf<int> idx(c, (size_t)std::max(m, 1));
    k_flag_index<<<nblk(n_p), 256, 0, c->stream>>>(n_p, flag.p, pos.p, idx.p);
    CK_LAUNCH(c);
    const Mat* GT = rc.GT;
    Mat* GTs = build_rows(c, m, GT->cols, [&](int* cnt, const int* orp, int* oci, double* ov) {
        if (cnt)
            k_gather_cnt<<<nblk(m), 256, 0, c->stream>>>(m, idx.p, GT->rp.p, cnt);
        else
            k_gather_fill<<<nblk(m), 256, 0, c->stream>>>(m, idx.p, GT->rp.p, GT->ci.p, GT->v.p, orp, oci, ov);
    });
    Mat* Xpb = triple_small(c, GTs, BN, Et);
    delete GTs;
    delete Et;
    lap("Xpb");
    Mat* Bx = build_rows(c, n, n, [&](int* cnt, const int* orp, int* oci, double* ov) {
        k_body_part2<<<nblk(n), 256, 0, c->stream>>>(n, n_p, flag.p, pos.p, Xpb->rp.p, Xpb->ci.p, Xpb->v.p, Xb->rp.p,
                                                     Xb->ci.p, Xb->v.p, cnt, orp, oci, ov);
    });
    delete Xpb;
    delete Xb;
    lap("Bx");
    Mat* S = symmetrized(c, Bx);
    delete Bx;
    lap("sym");
    const Mat* L = rc.Lpp;
    *lhs2 = build_rows(c, n, n, [&](int* cnt, const int* orp, int* oci, double* ov) {
        k_merge<<<nblk(n), 256, 0, c->stream>>>(n, n_p, rc.pin, L->rp.p, L->ci.p, L->v.p, S->rp.p, S->ci.p, S->v.p, cnt,
                                                orp, oci, ov);
    });
    delete S;
    lap("merge");
}

}  // namespace ibmgpu
