// sparse_ops.cu — structural sparse operations on the device, bit-exact with the reference.
//
//   transpose       sparse.hpp:120-138  stable radix sort of column keys (rows stay increasing)
//   spmm_rows       sparse.hpp:226-268  expand-sort-compress: products are emitted in Gustavson
//                                        traversal order (A-row entry, then B-row entry), stably
//                                        sorted by (row, col), then summed sequentially from 0.0 —
//                                        identical rounding to the reference's acc[c] += a*b;
//                                        cancelled entries are kept
//   triple_product  sparse.hpp:282-314  row slices of A, intermediate discarded per slice
//   add             sparse.hpp:317-329  row merge; (0+a*A)+b*B; exact zeros dropped (from_triplets)
//   symmetrized     sparse.hpp:351-353, pin (operators.hpp:381-392), concat (operators.hpp:394-404)
//   from_triplets   sparse.hpp:36-67
// All products/sums use explicit round-to-nearest intrinsics (no FMA contraction).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"
#include "kern.cuh"

namespace ibmgpu {

namespace {

constexpr long long kProductBudget = 1ll << 27;  // products per ESC chunk (~4.3 GB of sort buffers)

__global__ void k_row_of(int rows, const int* __restrict__ rp, int* __restrict__ row_of) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) row_of[k] = i;
}

__global__ void k_iota(int n, int* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

__global__ void k_count_cols(int nnz, const int* __restrict__ ci, int* __restrict__ cnt) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nnz) atomicAdd(cnt + ci[k], 1);
}

__global__ void k_transpose_fill(int nnz, const int* __restrict__ perm, const int* __restrict__ row_of,
                                 const double* __restrict__ v, int* __restrict__ tci, double* __restrict__ tv) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nnz) return;
    const int k = perm[p];
    tci[p] = row_of[k];
    tv[p] = v[k];
}

// products contributed by each A entry in rows [r0, r1)
__global__ void k_prod_count(int k0, int k1, const int* __restrict__ aci, const int* __restrict__ brp,
                             long long* __restrict__ cnt) {
    const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= k1) return;
    const int j = aci[k];
    cnt[k - k0] = brp[j + 1] - brp[j];
}

__global__ void k_expand(int r0, int k0, int k1, const int* __restrict__ arow_of, const int* __restrict__ aci,
                         const double* __restrict__ av, const int* __restrict__ brp, const int* __restrict__ bci,
                         const double* __restrict__ bv, const long long* __restrict__ pos, long long pos0,
                         unsigned long long* __restrict__ keys, double* __restrict__ vals) {
    const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= k1) return;
    const int j = aci[k];
    const double a = av[k];
    const unsigned long long rowkey = (unsigned long long)(arow_of[k] - r0) << 32;
    long long p = pos[k - k0] - pos0;
    for (int kb = brp[j]; kb < brp[j + 1]; ++kb, ++p) {
        keys[p] = rowkey | (unsigned)bci[kb];
        vals[p] = mul(a, bv[kb]);
    }
}

__global__ void k_heads(long long n, const unsigned long long* __restrict__ keys, int* __restrict__ head) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    head[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1 : 0;
}

__global__ void k_seg_start(long long n, const int* __restrict__ head, const int* __restrict__ uid,
                            long long* __restrict__ start) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    if (head[p]) start[uid[p]] = p;
}

// sequential in-order segment sums: acc = 0.0; acc += p_1; acc += p_2; ...
__global__ void k_seg_sum(int n_unique, long long n, const long long* __restrict__ start,
                          const unsigned long long* __restrict__ keys, const double* __restrict__ vals,
                          int* __restrict__ ci, double* __restrict__ v, int* __restrict__ rowcnt) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n_unique) return;
    const long long b = start[u], e = u + 1 < n_unique ? start[u + 1] : n;
    double s = 0.0;
    for (long long p = b; p < e; ++p) s = addd(s, vals[p]);
    ci[u] = (int)(keys[b] & 0xffffffffu);
    v[u] = s;
    atomicAdd(rowcnt + (int)(keys[b] >> 32), 1);
}

__global__ void k_shift_rp(int rows, const int* __restrict__ src, int add, int* __restrict__ dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= rows) dst[i] = src[i] + add;
}

// ---- add / pin / concat: thread-per-row two-pass (count, fill)
__global__ void k_add_rows(int rows, double a, const int* __restrict__ arp, const int* __restrict__ aci,
                           const double* __restrict__ av, double b, const int* __restrict__ brp,
                           const int* __restrict__ bci, const double* __restrict__ bv, int* __restrict__ cnt,
                           const int* __restrict__ orp, int* __restrict__ oci, double* __restrict__ ov) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    int ka = arp[i], ea = arp[i + 1], kb = brp[i], eb = brp[i + 1];
    int n = 0, o = orp ? orp[i] : 0;
    while (ka < ea || kb < eb) {
        const int ca = ka < ea ? aci[ka] : INT_MAX;
        const int cb = kb < eb ? bci[kb] : INT_MAX;
        const int col = ca < cb ? ca : cb;
        double s = 0.0;
        if (ca == col) s = addd(s, mul(a, av[ka++]));
        if (cb == col) s = addd(s, mul(b, bv[kb++]));
        if (s != 0.0) {
            if (oci) {
                oci[o + n] = col;
                ov[o + n] = s;
            }
            ++n;
        }
    }
    if (cnt) cnt[i] = n;
}

__global__ void k_pin_rows(int rows, int pin, const int* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ v, int* __restrict__ cnt, const int* __restrict__ orp,
                           int* __restrict__ oci, double* __restrict__ ov) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    int n = 0;
    const int o = orp ? orp[i] : 0;
    if (i == pin) {
        if (oci) {
            oci[o] = pin;
            ov[o] = 1.0;
        }
        n = 1;
    } else {
        bool placed = false;  // (pin,pin) only lives in row pin
        (void)placed;
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int c = ci[k];
            if (c == pin || v[k] == 0.0) continue;
            if (oci) {
                oci[o + n] = c;
                ov[o + n] = v[k];
            }
            ++n;
        }
    }
    if (cnt) cnt[i] = n;
}

__global__ void k_concat_rows(int rows, int gcols, const int* __restrict__ grp, const int* __restrict__ gci,
                              const double* __restrict__ gv, const int* __restrict__ erp, const int* __restrict__ eci,
                              const double* __restrict__ ev, int* __restrict__ cnt, const int* __restrict__ orp,
                              int* __restrict__ oci, double* __restrict__ ov) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    int n = 0;
    const int o = orp ? orp[i] : 0;
    for (int k = grp[i]; k < grp[i + 1]; ++k)
        if (gv[k] != 0.0) {
            if (oci) {
                oci[o + n] = gci[k];
                ov[o + n] = gv[k];
            }
            ++n;
        }
    if (erp)
        for (int k = erp[i]; k < erp[i + 1]; ++k)
            if (ev[k] != 0.0) {
                if (oci) {
                    oci[o + n] = gcols + eci[k];
                    ov[o + n] = ev[k];
                }
                ++n;
            }
    if (cnt) cnt[i] = n;
}

__global__ void k_scale(int rows, int mode, double a, const int* __restrict__ rp, const int* __restrict__ ci,
                        const double* __restrict__ d, double* __restrict__ v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const double f = mode == 0 ? a : mode == 1 ? d[i] : d[ci[k]];
        v[k] = mul(v[k], f);
    }
}

__global__ void k_tail_rows(int rows, int n_core, int n_agg, const int* __restrict__ prp, int* __restrict__ cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    cnt[i] = i < n_core ? prp[i + 1] - prp[i] : 1;
}

__global__ void k_tail_fill(int rows, int n_core, int n_agg, const int* __restrict__ prp, const int* __restrict__ pci,
                            const double* __restrict__ pv, const int* __restrict__ orp, int* __restrict__ oci,
                            double* __restrict__ ov) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const int o = orp[i];
    if (i < n_core) {
        for (int k = prp[i]; k < prp[i + 1]; ++k) {
            oci[o + k - prp[i]] = pci[k];
            ov[o + k - prp[i]] = pv[k];
        }
    } else {
        oci[o] = n_agg + (i - n_core);
        ov[o] = 1.0;
    }
}

__global__ void k_sym_check(int rows, double thr, const int* __restrict__ arp, const int* __restrict__ aci,
                            const double* __restrict__ av, const int* __restrict__ brp, const int* __restrict__ bci,
                            const double* __restrict__ bv, int* __restrict__ bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    int ka = arp[i], ea = arp[i + 1], kb = brp[i], eb = brp[i + 1];
    while (ka < ea || kb < eb) {
        const int ca = ka < ea ? aci[ka] : INT_MAX, cb = kb < eb ? bci[kb] : INT_MAX;
        double va = 0.0, vb = 0.0;
        if (ca <= cb) va = av[ka++];
        if (cb <= ca) vb = bv[kb++];
        if (fabs(va - vb) > thr) {
            atomicExch(bad, 1);
            return;
        }
    }
}

__global__ void k_trip_check(size_t n, int rows, int cols, const int* __restrict__ r, const int* __restrict__ c,
                             int* __restrict__ bad) {
    const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n && (r[k] < 0 || r[k] >= rows || c[k] < 0 || c[k] >= cols)) atomicExch(bad, 1);
}

__global__ void k_trip_keys(size_t n, const int* __restrict__ r, const int* __restrict__ c,
                            unsigned long long* __restrict__ keys) {
    const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) keys[k] = ((unsigned long long)(unsigned)r[k] << 32) | (unsigned)c[k];
}

// compress sorted (key, val) into CSR entries, dropping exact-zero sums (from_triplets semantics)
__global__ void k_seg_sum_drop(int n_unique, long long n, const long long* __restrict__ start,
                               const unsigned long long* __restrict__ keys, const double* __restrict__ vals,
                               int* __restrict__ keep, int* __restrict__ col, double* __restrict__ sum) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n_unique) return;
    const long long b = start[u], e = u + 1 < n_unique ? start[u + 1] : n;
    double s = 0.0;
    for (long long p = b; p < e; ++p) s = addd(s, vals[p]);
    keep[u] = s != 0.0;
    col[u] = (int)(keys[b] & 0xffffffffu);
    sum[u] = s;
}

__global__ void k_compact_keep(int n_unique, const long long* __restrict__ start, const unsigned long long* __restrict__ keys,
                               const int* __restrict__ keep, const int* __restrict__ kpos, const int* __restrict__ col,
                               const double* __restrict__ sum, int* __restrict__ oci, double* __restrict__ ov,
                               int* __restrict__ rowcnt) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n_unique || !keep[u]) return;
    oci[kpos[u]] = col[u];
    ov[kpos[u]] = sum[u];
    atomicAdd(rowcnt + (int)(keys[start[u]] >> 32), 1);
}

__global__ void k_diag_fill(int n, const double* __restrict__ d, int* __restrict__ cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) cnt[i] = d[i] != 0.0;
}
__global__ void k_diag_write(int n, const double* __restrict__ d, const int* __restrict__ rp, int* __restrict__ ci,
                             double* __restrict__ v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && d[i] != 0.0) {
        ci[rp[i]] = i;
        v[rp[i]] = d[i];
    }
}

inline int blocks(long long n, int b = 256) { return (int)((n + b - 1) / b); }

int bits_for(long long n) {
    int b = 1;
    while ((1ll << b) < n) ++b;
    return b;
}

// Sort (keys, vals) stably by key; results in *_out.
void sort_pairs(Ctx* c, unsigned long long* kin, unsigned long long* kout, double* vin, double* vout, long long n,
                int end_bit) {
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, n, 0, end_bit, c->stream));
    DBuf<char> t(c, tmp);
    CK(cub::DeviceRadixSort::SortPairs(t.p, tmp, kin, kout, vin, vout, n, 0, end_bit, c->stream));
}

// Segment bookkeeping over sorted keys: returns number of unique keys; fills start[u].
int segments(Ctx* c, const unsigned long long* keys, long long n, DBuf<long long>& start) {
    DBuf<int> head(c, (size_t)n), uid(c, (size_t)n + 1);
    k_heads<<<blocks(n), 256, 0, c->stream>>>(n, keys, head.p);
    CK_LAUNCH(c);
    // exclusive scan of heads gives uid+1 at each head position; use inclusive then subtract
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, head.p, uid.p, (int)n, c->stream));
    DBuf<char> t(c, tmp);
    CK(cub::DeviceScan::ExclusiveSum(t.p, tmp, head.p, uid.p, (int)n, c->stream));
    const int last_uid = d2h_scalar(c, uid.p + n - 1);
    const int last_head = d2h_scalar(c, head.p + n - 1);
    const int n_unique = last_uid + last_head;
    start.alloc(c, (size_t)n_unique);
    k_seg_start<<<blocks(n), 256, 0, c->stream>>>(n, head.p, uid.p, start.p);
    CK_LAUNCH(c);
    return n_unique;
}

// Concatenate row-slice pieces into one matrix.
Mat* concat_rows(Ctx* c, std::vector<Mat*>& parts, int rows, int cols) {
    long long total = 0;
    for (auto* p : parts) total += p->nnz;
    require(total < (1ll << 31), "sparse: result exceeds int32 nonzero indexing");
    Mat* m = mat_new(c, rows, cols, (int)total);
    int r = 0, off = 0;
    CK(cudaMemsetAsync(m->rp.p, 0, sizeof(int), c->stream));
    for (auto* p : parts) {
        k_shift_rp<<<blocks(p->rows + 1), 256, 0, c->stream>>>(p->rows, p->rp.p, off, m->rp.p + r);
        CK_LAUNCH(c);
        d2d(c, m->ci.p + off, p->ci.p, (size_t)p->nnz);
        d2d(c, m->v.p + off, p->v.p, (size_t)p->nnz);
        r += p->rows;
        off += p->nnz;
        delete p;
    }
    parts.clear();
    return m;
}

// ESC product of A rows [r0, r1) (entries [k0, k1)) with B; all products fit in one chunk.
Mat* esc_chunk(Ctx* c, const Mat* A, const int* arow_of, int r0, int r1, const Mat* B) {
    const int k0 = d2h_scalar(c, A->rp.p + r0), k1 = d2h_scalar(c, A->rp.p + r1);
    const int rows = r1 - r0;
    const int na = k1 - k0;
    DBuf<long long> cnt(c, (size_t)na + 1), pos(c, (size_t)na + 1);
    long long n = 0;
    if (na > 0) {
        k_prod_count<<<blocks(na), 256, 0, c->stream>>>(k0, k1, A->ci.p, B->rp.p, cnt.p);
        CK_LAUNCH(c);
        n = exclusive_scan_total64(c, cnt.p, pos.p, na);
    }
    Mat* out = mat_new(c, rows, B->cols, 0);
    CK(cudaMemsetAsync(out->rp.p, 0, sizeof(int) * ((size_t)rows + 1), c->stream));
    if (n == 0) {
        out->nnz = 0;
        return out;
    }
    DBuf<unsigned long long> kin(c, (size_t)n), kout(c, (size_t)n);
    DBuf<double> vin(c, (size_t)n), vout(c, (size_t)n);
    k_expand<<<blocks(na), 256, 0, c->stream>>>(r0, k0, k1, arow_of, A->ci.p, A->v.p, B->rp.p, B->ci.p, B->v.p,
                                                 pos.p, 0, kin.p, vin.p);
    CK_LAUNCH(c);
    if (std::getenv("IBMGPU_SETUP_PROFILE")) {
        sync(c);
        const auto t0 = std::chrono::steady_clock::now();
        sort_pairs(c, kin.p, kout.p, vin.p, vout.p, n, 32 + bits_for(rows + 1));
        sync(c);
        std::fprintf(stderr, "[esc] rows %d products %lld sort %.3f ms\n", rows, n,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    } else {
        sort_pairs(c, kin.p, kout.p, vin.p, vout.p, n, 32 + bits_for(rows + 1));
    }
    kin.release();
    vin.release();
    DBuf<long long> start;
    const int nu = segments(c, kout.p, n, start);
    DBuf<int> rowcnt(c, (size_t)rows);
    CK(cudaMemsetAsync(rowcnt.p, 0, sizeof(int) * rows, c->stream));
    out->ci.alloc(c, (size_t)nu);
    out->v.alloc(c, (size_t)nu);
    out->nnz = nu;
    k_seg_sum<<<blocks(nu), 256, 0, c->stream>>>(nu, n, start.p, kout.p, vout.p, out->ci.p, out->v.p, rowcnt.p);
    CK_LAUNCH(c);
    exclusive_scan_total(c, rowcnt.p, out->rp.p, rows);
    return out;
}

__global__ void k_row_products(int rows, const int* __restrict__ arp, const int* __restrict__ aci,
                               const int* __restrict__ brp, long long* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    long long s = 0;
    for (int k = arp[i]; k < arp[i + 1]; ++k) s += brp[aci[k] + 1] - brp[aci[k]];
    out[i] = s;
}

__global__ void k_chunk_bounds(int rows, const long long* __restrict__ pref, long long budget, int n_chunks,
                               int* __restrict__ bounds) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > n_chunks) return;
    if (t == n_chunks) {
        bounds[t] = rows;
        return;
    }
    // first row whose prefix (products before it) >= t * budget
    long long target = (long long)t * budget;
    int lo = 0, hi = rows;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (pref[mid] < target)
            lo = mid + 1;
        else
            hi = mid;
    }
    bounds[t] = lo;
}

// SpMV plans are built lazily (spmv / solver setup), not for every intermediate product.
Mat* finish_plan(Ctx*, Mat* m) { return m; }

}  // namespace

Mat* transpose(Ctx* c, const Mat* A) {
    Mat* t = mat_new(c, A->cols, A->rows, A->nnz);
    DBuf<int> cnt(c, (size_t)A->cols + 1);
    CK(cudaMemsetAsync(cnt.p, 0, sizeof(int) * ((size_t)A->cols + 1), c->stream));
    if (A->nnz > 0) {
        k_count_cols<<<blocks(A->nnz), 256, 0, c->stream>>>(A->nnz, A->ci.p, cnt.p);
        CK_LAUNCH(c);
    }
    exclusive_scan_total(c, cnt.p, t->rp.p, A->cols);
    if (A->nnz > 0) {
        DBuf<int> row_of(c, A->nnz), idx(c, A->nnz), kout(c, A->nnz), perm(c, A->nnz);
        k_row_of<<<blocks(A->rows), 256, 0, c->stream>>>(A->rows, A->rp.p, row_of.p);
        CK_LAUNCH(c);
        k_iota<<<blocks(A->nnz), 256, 0, c->stream>>>(A->nnz, idx.p);
        CK_LAUNCH(c);
        size_t tmp = 0;
        const int eb = bits_for((long long)A->cols + 1);
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, A->ci.p, kout.p, idx.p, perm.p, A->nnz, 0, eb, c->stream));
        DBuf<char> tt(c, tmp);
        CK(cub::DeviceRadixSort::SortPairs(tt.p, tmp, A->ci.p, kout.p, idx.p, perm.p, A->nnz, 0, eb, c->stream));
        k_transpose_fill<<<blocks(A->nnz), 256, 0, c->stream>>>(A->nnz, perm.p, row_of.p, A->v.p, t->ci.p, t->v.p);
        CK_LAUNCH(c);
    }
    return finish_plan(c, t);
}

Mat* spmm_rows(Ctx* c, const Mat* A, int r0, int r1, const Mat* B) {
    require(A->cols == B->rows, "spmm: dimension mismatch");
    const int rows = r1 - r0;
    DBuf<int> row_of(c, (size_t)std::max(A->nnz, 1));
    if (A->nnz) {
        k_row_of<<<blocks(A->rows), 256, 0, c->stream>>>(A->rows, A->rp.p, row_of.p);
        CK_LAUNCH(c);
    }
    // per-row product counts -> chunking under the product budget
    DBuf<long long> rprod(c, (size_t)rows + 1), pref(c, (size_t)rows + 1);
    long long total = 0;
    if (rows > 0) {
        k_row_products<<<blocks(rows), 256, 0, c->stream>>>(rows, A->rp.p + r0, A->ci.p, B->rp.p, rprod.p);
        CK_LAUNCH(c);
        total = exclusive_scan_total64(c, rprod.p, pref.p, rows);
    }
    std::vector<int> bounds = {0, rows};
    if (total > kProductBudget) {
        const int n_chunks = (int)((total + kProductBudget - 1) / kProductBudget);
        DBuf<int> b(c, (size_t)n_chunks + 1);
        k_chunk_bounds<<<blocks(n_chunks + 1), 256, 0, c->stream>>>(rows, pref.p, kProductBudget, n_chunks, b.p);
        CK_LAUNCH(c);
        bounds.assign((size_t)n_chunks + 1, 0);
        d2h(c, bounds.data(), b.p, (size_t)n_chunks + 1);
        sync(c);
        bounds.erase(std::unique(bounds.begin(), bounds.end()), bounds.end());
        // a single row larger than the budget still forms its own chunk
    }
    std::vector<Mat*> parts;
    for (size_t t = 0; t + 1 < bounds.size(); ++t)
        parts.push_back(esc_chunk(c, A, row_of.p, r0 + bounds[t], r0 + bounds[t + 1], B));
    Mat* out = parts.size() == 1 ? parts[0] : concat_rows(c, parts, rows, B->cols);
    if (parts.size() == 1) parts.clear();
    return finish_plan(c, out);
}

Mat* triple_product(Ctx* c, const Mat* A, const Mat* B, const Mat* C, int slice, long long* peak, int* slices) {
    require(A->cols == B->rows && B->cols == C->rows, "sliced_triple_product: dimension mismatch");
    require(slice >= 1, "sliced_triple_product: slice size must be >= 1");
    std::vector<Mat*> parts;
    long long pk = 0;
    int ns = 0;
    for (int r0 = 0; r0 < A->rows; r0 += slice) {
        const int r1 = std::min(A->rows, r0 + slice);
        Mat* t = spmm_rows(c, A, r0, r1, B);
        pk = std::max<long long>(pk, t->nnz);
        ++ns;
        parts.push_back(spmm_rows(c, t, 0, t->rows, C));
        delete t;
    }
    if (peak) *peak = pk;
    if (slices) *slices = ns;
    if (A->rows == 0) {
        Mat* m = mat_new(c, 0, C->cols, 0);
        CK(cudaMemsetAsync(m->rp.p, 0, sizeof(int), c->stream));
        return finish_plan(c, m);
    }
    if (parts.size() == 1) {
        Mat* m = parts[0];
        return m;
    }
    return finish_plan(c, concat_rows(c, parts, A->rows, C->cols));
}

Mat* add(Ctx* c, double a, const Mat* A, double b, const Mat* B) {
    require(A->rows == B->rows && A->cols == B->cols, "add_sparse: dimension mismatch");
    const int rows = A->rows;
    DBuf<int> cnt(c, (size_t)rows + 1);
    Mat* m = mat_new(c, rows, A->cols, 0);
    if (rows) {
        k_add_rows<<<blocks(rows), 256, 0, c->stream>>>(rows, a, A->rp.p, A->ci.p, A->v.p, b, B->rp.p, B->ci.p, B->v.p,
                                                        cnt.p, nullptr, nullptr, nullptr);
        CK_LAUNCH(c);
    }
    exclusive_scan_total(c, cnt.p, m->rp.p, rows);
    m->nnz = d2h_scalar(c, m->rp.p + rows);
    m->ci.alloc(c, (size_t)m->nnz);
    m->v.alloc(c, (size_t)m->nnz);
    if (rows) {
        k_add_rows<<<blocks(rows), 256, 0, c->stream>>>(rows, a, A->rp.p, A->ci.p, A->v.p, b, B->rp.p, B->ci.p, B->v.p,
                                                        nullptr, m->rp.p, m->ci.p, m->v.p);
        CK_LAUNCH(c);
    }
    return finish_plan(c, m);
}

Mat* symmetrized(Ctx* c, const Mat* A) {
    Mat* At = transpose(c, A);
    Mat* S = add(c, 0.5, A, 0.5, At);
    delete At;
    return S;
}

Mat* pin(Ctx* c, const Mat* A, int p) {
    require(A->rows == A->cols && p >= 0 && p < A->rows, "pin_row_col: bad pin index");
    const int rows = A->rows;
    DBuf<int> cnt(c, (size_t)rows + 1);
    Mat* m = mat_new(c, rows, A->cols, 0);
    k_pin_rows<<<blocks(rows), 256, 0, c->stream>>>(rows, p, A->rp.p, A->ci.p, A->v.p, cnt.p, nullptr, nullptr, nullptr);
    CK_LAUNCH(c);
    exclusive_scan_total(c, cnt.p, m->rp.p, rows);
    m->nnz = d2h_scalar(c, m->rp.p + rows);
    m->ci.alloc(c, (size_t)m->nnz);
    m->v.alloc(c, (size_t)m->nnz);
    k_pin_rows<<<blocks(rows), 256, 0, c->stream>>>(rows, p, A->rp.p, A->ci.p, A->v.p, nullptr, m->rp.p, m->ci.p, m->v.p);
    CK_LAUNCH(c);
    return finish_plan(c, m);
}

Mat* concat_cols(Ctx* c, const Mat* G, const Mat* Et) {
    require(Et == nullptr || Et->rows == G->rows, "concat_cols: row mismatch");
    const int rows = G->rows;
    const int cols = G->cols + (Et ? Et->cols : 0);
    DBuf<int> cnt(c, (size_t)rows + 1);
    Mat* m = mat_new(c, rows, cols, 0);
    const int* erp = Et ? Et->rp.p : nullptr;
    const int* eci = Et ? Et->ci.p : nullptr;
    const double* ev = Et ? Et->v.p : nullptr;
    if (rows) {
        k_concat_rows<<<blocks(rows), 256, 0, c->stream>>>(rows, G->cols, G->rp.p, G->ci.p, G->v.p, erp, eci, ev, cnt.p,
                                                           nullptr, nullptr, nullptr);
        CK_LAUNCH(c);
    }
    exclusive_scan_total(c, cnt.p, m->rp.p, rows);
    m->nnz = d2h_scalar(c, m->rp.p + rows);
    m->ci.alloc(c, (size_t)m->nnz);
    m->v.alloc(c, (size_t)m->nnz);
    if (rows) {
        k_concat_rows<<<blocks(rows), 256, 0, c->stream>>>(rows, G->cols, G->rp.p, G->ci.p, G->v.p, erp, eci, ev,
                                                           nullptr, m->rp.p, m->ci.p, m->v.p);
        CK_LAUNCH(c);
    }
    return finish_plan(c, m);
}

Mat* scale(Ctx* c, const Mat* A, int mode, double a, const double* d_dev) {
    Mat* m = mat_new(c, A->rows, A->cols, A->nnz);
    d2d(c, m->rp.p, A->rp.p, (size_t)A->rows + 1);
    d2d(c, m->ci.p, A->ci.p, (size_t)A->nnz);
    d2d(c, m->v.p, A->v.p, (size_t)A->nnz);
    if (A->rows) {
        k_scale<<<blocks(A->rows), 256, 0, c->stream>>>(A->rows, mode, a, m->rp.p, m->ci.p, d_dev, m->v.p);
        CK_LAUNCH(c);
    }
    return finish_plan(c, m);
}

Mat* identity_tail_append(Ctx* c, const Mat* Pc, int n_core, int n_agg, int tail) {
    const int rows = n_core + tail;
    DBuf<int> cnt(c, (size_t)rows + 1);
    Mat* m = mat_new(c, rows, n_agg + tail, 0);
    k_tail_rows<<<blocks(rows), 256, 0, c->stream>>>(rows, n_core, n_agg, Pc->rp.p, cnt.p);
    CK_LAUNCH(c);
    exclusive_scan_total(c, cnt.p, m->rp.p, rows);
    m->nnz = d2h_scalar(c, m->rp.p + rows);
    m->ci.alloc(c, (size_t)m->nnz);
    m->v.alloc(c, (size_t)m->nnz);
    k_tail_fill<<<blocks(rows), 256, 0, c->stream>>>(rows, n_core, n_agg, Pc->rp.p, Pc->ci.p, Pc->v.p, m->rp.p,
                                                     m->ci.p, m->v.p);
    CK_LAUNCH(c);
    return finish_plan(c, m);
}

bool is_symmetric(Ctx* c, const Mat* A, double tol) {
    if (A->rows != A->cols) return false;
    Mat* At = transpose(c, A);
    const double scale = std::max(max_abs(c, A), 1e-300);
    DBuf<int> bad(c, 1);
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), c->stream));
    if (A->rows) {
        k_sym_check<<<blocks(A->rows), 256, 0, c->stream>>>(A->rows, tol * scale, A->rp.p, A->ci.p, A->v.p, At->rp.p,
                                                            At->ci.p, At->v.p, bad.p);
        CK_LAUNCH(c);
    }
    const int b = d2h_scalar(c, bad.p);
    delete At;
    return b == 0;
}

Mat* from_triplets(Ctx* c, int rows, int cols, size_t n, const int* r, const int* cc, const double* v) {
    DBuf<int> bad(c, 1);
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), c->stream));
    if (n) {
        k_trip_check<<<blocks((long long)n), 256, 0, c->stream>>>(n, rows, cols, r, cc, bad.p);
        CK_LAUNCH(c);
    }
    require(d2h_scalar(c, bad.p) == 0, "sparse: triplet index out of range");
    Mat* m = mat_new(c, rows, cols, 0);
    CK(cudaMemsetAsync(m->rp.p, 0, sizeof(int) * ((size_t)rows + 1), c->stream));
    if (n == 0) return finish_plan(c, m);
    DBuf<unsigned long long> kin(c, n), kout(c, n);
    DBuf<double> vin(c, n), vout(c, n);
    k_trip_keys<<<blocks((long long)n), 256, 0, c->stream>>>(n, r, cc, kin.p);
    CK_LAUNCH(c);
    d2d(c, vin.p, v, n);
    sort_pairs(c, kin.p, kout.p, vin.p, vout.p, (long long)n, 32 + bits_for((long long)rows + 1));
    DBuf<long long> start;
    const int nu = segments(c, kout.p, (long long)n, start);
    DBuf<int> keep(c, (size_t)nu), kpos(c, (size_t)nu + 1), col(c, (size_t)nu), rowcnt(c, (size_t)rows);
    DBuf<double> sum(c, (size_t)nu);
    k_seg_sum_drop<<<blocks(nu), 256, 0, c->stream>>>(nu, (long long)n, start.p, kout.p, vout.p, keep.p, col.p, sum.p);
    CK_LAUNCH(c);
    exclusive_scan_total(c, keep.p, kpos.p, nu);
    m->nnz = d2h_scalar(c, kpos.p + nu);
    m->ci.alloc(c, (size_t)m->nnz);
    m->v.alloc(c, (size_t)m->nnz);
    CK(cudaMemsetAsync(rowcnt.p, 0, sizeof(int) * (size_t)rows, c->stream));
    k_compact_keep<<<blocks(nu), 256, 0, c->stream>>>(nu, start.p, kout.p, keep.p, kpos.p, col.p, sum.p, m->ci.p,
                                                      m->v.p, rowcnt.p);
    CK_LAUNCH(c);
    exclusive_scan_total(c, rowcnt.p, m->rp.p, rows);
    return finish_plan(c, m);
}

Mat* diag_matrix(Ctx* c, int n, const double* d) {
    DBuf<int> cnt(c, (size_t)n + 1);
    Mat* m = mat_new(c, n, n, 0);
    if (n) {
        k_diag_fill<<<blocks(n), 256, 0, c->stream>>>(n, d, cnt.p);
        CK_LAUNCH(c);
    }
    exclusive_scan_total(c, cnt.p, m->rp.p, n);
    m->nnz = d2h_scalar(c, m->rp.p + n);
    m->ci.alloc(c, (size_t)m->nnz);
    m->v.alloc(c, (size_t)m->nnz);
    if (n) {
        k_diag_write<<<blocks(n), 256, 0, c->stream>>>(n, d, m->rp.p, m->ci.p, m->v.p);
        CK_LAUNCH(c);
    }
    return finish_plan(c, m);
}

}  // namespace ibmgpu
