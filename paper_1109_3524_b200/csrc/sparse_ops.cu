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
#include <climits>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"
#include "kern.cuh"

namespace ibmgpu {

namespace {

constexpr long long kProductBudget = 1ll << 25;  // products per ESC chunk (~1.1 GB of sort buffers)

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
    // thread per segment; segments longer than 64 products (the coarse body-tail entries sum
    // thousands) are summed by the whole warp: 32 products in flight per load, added in order
    // from shuffles — the same rounding sequence, without a serial load chain
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool valid = u < n_unique;
    long long b = 0, e = 0;
    if (valid) b = start[u], e = u + 1 < n_unique ? start[u + 1] : n;
    const bool is_long = valid && e - b > 64;
    double s = 0.0;
    if (valid && !is_long)
        for (long long p = b; p < e; ++p) s = addd(s, vals[p]);
    for (unsigned longs = __ballot_sync(kFull, is_long); longs; longs &= longs - 1) {
        const int l = __ffs(longs) - 1;
        const long long lb = __shfl_sync(kFull, b, l), le = __shfl_sync(kFull, e, l);
        double acc = 0.0;
        double x = lb + lane < le ? vals[lb + lane] : 0.0;
        for (long long p0 = lb; p0 < le; p0 += 32) {
            const double xn = p0 + 32 + lane < le ? vals[p0 + 32 + lane] : 0.0;
            const int cnt = (int)min(32ll, le - p0);
            for (int j = 0; j < cnt; ++j) acc = addd(acc, __shfl_sync(kFull, x, j));
            x = xn;
        }
        if (lane == l) s = acc;
    }
    if (!valid) return;
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
    } else {  // (pin, pin) only lives in row pin
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
    c->pdl_fence = 1;
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
    c->pdl_fence = 1;
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

// ---------------------------------------------------------------- hash SpGEMM (warp per row)
// spmm_rows (sparse.hpp:226-268) with one warp per output row and the row's accumulator as an
// open-addressing hash table in shared memory — instead of sorting every product. Products are
// formed 32 at a time in Gustavson order (A-row entry, then B-row entry); lanes whose products hit
// the same column are grouped with __match_any_sync and the group's first lane adds them to the
// table entry in lane (= Gustavson) order, so each column's sum is 0.0 + p1 + p2 + ... exactly as
// the reference accumulates it. Columns are then sorted (bitonic, in shared memory). Symbolic
// pass: unique counts per row; a row over 3/4 of the symbolic table sends the product to ESC.
constexpr int kHashSym = 4096, kSymWarps = 8;
constexpr int kHashU = 4;  // product batches whose loads are issued together

__device__ __forceinline__ unsigned hslot(int c, int mask) { return ((unsigned)c * 2654435761u) & (unsigned)mask; }

// The 32 A entries of one chunk: B-row start, product offsets (inclusive scan), A value.
struct HashChunk {
    int off[33];
    int bs[32];
    double a[32];
};

// next row for this warp from a global counter (lane 0 takes it, the warp shares it)
__device__ __forceinline__ int next_row(unsigned* next, int lane) {
    unsigned r = 0;
    if (lane == 0) r = atomicAdd(next, 1u);
    return static_cast<int>(__shfl_sync(kFull, r, 0));
}

__device__ __forceinline__ int chunk_load(HashChunk& ch, int c0, int e, const int* __restrict__ aci,
                                          const double* __restrict__ av, const int* __restrict__ brp, int lane,
                                          bool values) {
    const int kk = c0 + lane;
    int bs = 0, bl = 0;
    double a = 0.0;
    if (kk < e) {
        const int k = __ldg(aci + kk);
        bs = __ldg(brp + k);
        bl = __ldg(brp + k + 1) - bs;
        if (values) a = __ldg(av + kk);
    }
    int inc = bl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += t;
    }
    ch.off[lane + 1] = inc;
    if (lane == 0) ch.off[0] = 0;
    ch.bs[lane] = bs;
    if (values) ch.a[lane] = a;
    __syncwarp();
    return __shfl_sync(kFull, inc, 31);
}

__device__ __forceinline__ int chunk_owner(const HashChunk& ch, int q) {  // largest o with off[o] <= q
    int lo = 0, hi = 31;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ch.off[mid] <= q)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(kSymWarps * 32) k_hash_symbolic(int r0, int rows, const int* __restrict__ arp,
                                                                  const int* __restrict__ aci,
                                                                  const int* __restrict__ brp,
                                                                  const int* __restrict__ bci, int* __restrict__ cnt,
                                                                  int* __restrict__ maxcnt,
                                                                  const long long* __restrict__ rprod,
                                                                  long long limit, unsigned* __restrict__ next) {
    extern __shared__ int hsm[];
    __shared__ HashChunk chunks[kSymWarps];
    __shared__ int counter[kSymWarps];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int* keys = hsm + w * kHashSym;
    HashChunk& ch = chunks[w];
    for (;;) {
        const int row = next_row(next, lane);  // rows handed out one at a time: no CTA-wave tail
        if (row >= rows) break;
        if (rprod[row] > limit) continue;  // long row: counted by the ESC pass
        for (int t = lane; t < kHashSym; t += 32) keys[t] = -1;
        if (lane == 0) counter[w] = 0;
        __syncwarp();
        const int i = r0 + row, b = __ldg(arp + i), e = __ldg(arp + i + 1);
        for (int c0 = b; c0 < e; c0 += 32) {
            if (*(volatile int*)(counter + w) > kHashSym * 3 / 4) break;  // overflow: ESC takes over
            const int total = chunk_load(ch, c0, e, aci, nullptr, brp, lane, false);
            for (int q0 = 0; q0 < total; q0 += 32 * kHashU) {
                if (*(volatile int*)(counter + w) > kHashSym * 3 / 4) break;
                int cols[kHashU];  // kHashU independent column loads in flight per lane
#pragma unroll
                for (int u = 0; u < kHashU; ++u) {
                    const int q = q0 + u * 32 + lane;
                    cols[u] = -1;
                    if (q < total) {
                        const int o = chunk_owner(ch, q);
                        cols[u] = __ldg(bci + ch.bs[o] + (q - ch.off[o]));
                    }
                }
#pragma unroll
                for (int u = 0; u < kHashU; ++u) {
                    const int col = cols[u];
                    if (col < 0) continue;
                    unsigned h = hslot(col, kHashSym - 1);
                    for (int probe = 0; probe < kHashSym; ++probe) {
                        const int prev = atomicCAS(keys + h, -1, col);
                        if (prev == -1) {
                            atomicAdd(counter + w, 1);
                            break;
                        }
                        if (prev == col) break;
                        h = (h + 1) & (kHashSym - 1);
                    }
                }
            }
            __syncwarp();
        }
        __syncwarp();
        if (lane == 0) {
            cnt[row] = counter[w];
            atomicMax(maxcnt, counter[w]);
        }
        __syncwarp();
    }
}

__global__ void k_hash_numeric(int r0, int rows, const int* __restrict__ arp, const int* __restrict__ aci,
                               const double* __restrict__ av, const int* __restrict__ brp,
                               const int* __restrict__ bci, const double* __restrict__ bv,
                               const int* __restrict__ crp, int* __restrict__ cci, double* __restrict__ cv,
                               int slots, const long long* __restrict__ rprod, long long limit,
                               unsigned* __restrict__ next) {
    extern __shared__ double hsd[];
    const int nw = blockDim.x >> 5;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* vals = hsd + (size_t)w * slots;
    int* keys = reinterpret_cast<int*>(hsd + (size_t)nw * slots) + (size_t)w * slots;
    HashChunk* chunks = reinterpret_cast<HashChunk*>(reinterpret_cast<int*>(hsd + (size_t)nw * slots) + (size_t)nw * slots);
    double* prod = reinterpret_cast<double*>(chunks + nw) + w * 32;
    HashChunk& ch = chunks[w];
    const int mask = slots - 1;
    for (;;) {
        const int row = next_row(next, lane);
        if (row >= rows) break;
        if (rprod[row] > limit) continue;
        for (int t = lane; t < slots; t += 32) {
            keys[t] = -1;
            vals[t] = 0.0;
        }
        __syncwarp();
        const int i = r0 + row, b = __ldg(arp + i), e = __ldg(arp + i + 1);
        for (int c0 = b; c0 < e; c0 += 32) {
            const int total = chunk_load(ch, c0, e, aci, av, brp, lane, true);
            for (int q0 = 0; q0 < total; q0 += 32 * kHashU) {
                // kHashU batches of 32 products loaded at once (independent loads in flight),
                // then accumulated batch by batch: Gustavson order is kept
                int cols[kHashU];
                double ps[kHashU];
#pragma unroll
                for (int u = 0; u < kHashU; ++u) {
                    const int q = q0 + u * 32 + lane;
                    cols[u] = -1;
                    ps[u] = 0.0;
                    if (q < total) {
                        const int o = chunk_owner(ch, q);
                        const int jj = ch.bs[o] + (q - ch.off[o]);
                        cols[u] = __ldg(bci + jj);
                        ps[u] = mul(ch.a[o], __ldg(bv + jj));
                    }
                }
#pragma unroll
                for (int u = 0; u < kHashU; ++u) {
                    if (q0 + u * 32 >= total) break;  // warp-uniform
                    const int col = cols[u];
                    prod[lane] = ps[u];
                    const unsigned grp = __match_any_sync(kFull, col);
                    __syncwarp();
                    if (col >= 0 && lane == __ffs(grp) - 1) {
                        unsigned h = hslot(col, mask);
                        int probes = 0;
                        for (;;) {  // find or claim the column's slot (other leaders hold other columns)
                            const int prev = atomicCAS(keys + h, -1, col);
                            if (prev == -1 || prev == col) break;
                            h = (h + 1) & mask;
                            IBM_DCHECK(++probes < slots);  // table never full
                        }
                        double acc = vals[h];
                        for (unsigned m = grp; m; m &= m - 1) acc = addd(acc, prod[__ffs(m) - 1]);
                        vals[h] = acc;
                    }
                    __syncwarp();
                }
            }
            __syncwarp();
        }
        // compact the occupied slots to the front (in slot order; positions never pass a read)
        int n_u = 0;
        for (int base = 0; base < slots; base += 32) {
            const int t = base + lane;
            const int k = keys[t];
            const double v = vals[t];
            const unsigned has = __ballot_sync(kFull, k != -1);
            __syncwarp();
            if (k != -1) {
                const int pos = n_u + __popc(has & ((1u << lane) - 1));
                keys[pos] = k;
                vals[pos] = v;
            }
            n_u += __popc(has);
            __syncwarp();
        }
        int n2 = 1;
        while (n2 < n_u) n2 <<= 1;
        for (int t = n_u + lane; t < n2; t += 32) keys[t] = INT_MAX;
        __syncwarp();
        for (int k = 2; k <= n2; k <<= 1)  // bitonic sort by column (columns are unique)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int t = lane; t < n2; t += 32) {
                    const int u = t ^ j;
                    if (u > t) {
                        const int kt = keys[t], ku = keys[u];
                        if ((kt > ku) == ((t & k) == 0)) {
                            keys[t] = ku;
                            keys[u] = kt;
                            const double vt = vals[t];
                            vals[t] = vals[u];
                            vals[u] = vt;
                        }
                    }
                }
                __syncwarp();
            }
        const int o0 = crp[row];
        IBM_DCHECK(o0 + n_u == crp[row + 1]);  // symbolic count == numeric count
        for (int t = lane; t < n_u; t += 32) {
            IBM_DCHECK(keys[t] >= 0 && (t == 0 || keys[t - 1] < keys[t]));  // unique, sorted columns
            cci[o0 + t] = keys[t];
            cv[o0 + t] = vals[t];
        }
        __syncwarp();
    }
}

__global__ void k_long_flags(int n, const long long* __restrict__ rprod, long long limit, int* __restrict__ flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = rprod[i] > limit;
}
__global__ void k_long_rows(int n, const int* __restrict__ flag, const int* __restrict__ pos, int r0,
                            const int* __restrict__ arp, int* __restrict__ idx, int* __restrict__ len) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) {
        idx[pos[i]] = i;
        len[pos[i]] = arp[r0 + i + 1] - arp[r0 + i];
    }
}
__global__ void k_gather_rows(int nl, const int* __restrict__ idx, int r0, const int* __restrict__ arp,
                              const int* __restrict__ aci, const double* __restrict__ av,
                              const int* __restrict__ lrp, int* __restrict__ lci, double* __restrict__ lv) {
    const int r = blockIdx.x;
    if (r >= nl) return;
    const int src = arp[r0 + idx[r]], n = lrp[r + 1] - lrp[r];
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        lci[lrp[r] + k] = aci[src + k];
        lv[lrp[r] + k] = av[src + k];
    }
}
__global__ void k_long_counts(int nl, const int* __restrict__ idx, const int* __restrict__ crp_long,
                              int* __restrict__ cnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nl) cnt[idx[r]] = crp_long[r + 1] - crp_long[r];
}
__global__ void k_place_rows(int nl, const int* __restrict__ idx, const int* __restrict__ lrp,
                             const int* __restrict__ lci, const double* __restrict__ lv, const int* __restrict__ crp,
                             int* __restrict__ cci, double* __restrict__ cv) {
    const int r = blockIdx.x;
    if (r >= nl) return;
    const int dst = crp[idx[r]], src = lrp[r], n = lrp[r + 1] - lrp[r];
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        cci[dst + k] = lci[src + k];
        cv[dst + k] = lv[src + k];
    }
}

// ---------------------------------------------------------------- dense-accumulator SpGEMM
// spmm_rows for products with a narrow output (<= kDenseCols columns) and long rows — the coarse
// Galerkin products, whose long rows (tens of thousands of products) serialised a hash warp. One
// CTA per output row (rows handed out from a counter); the row's accumulator is a dense array of
// the output width in shared memory plus a bitmap of touched columns. Products are formed 256 at a
// time in Gustavson order (A-row entry, then B-row entry); the 8 warps add their 32 products in
// warp order, each warp grouping equal columns with __match_any_sync and adding a group in lane
// order — every column receives 0.0 + p1 + p2 + ... in Gustavson order, as the reference. The
// bitmap then yields the columns already sorted (no sort). Symbolic pass: the bitmap only.
constexpr int kDenseCols = 12288, kDenseThreads = 256, kDenseChunk = 256;

struct DenseChunk {
    int off[kDenseChunk + 1];  // inclusive product offsets of the chunk's A entries
    int bs[kDenseChunk];       // B-row start of each A entry
    double a[kDenseChunk];
};

// Wider outputs (up to kDenseWideMax columns): `win` gives each row a window [base, base + ncols)
// holding all its columns (the rows of P^T A on coarse levels are spatially local). A row whose
// span exceeds the window uses this CTA's full-width accumulator and bitmap in global memory
// (gacc / gbits, zero between rows like the shared ones) — same order of additions either way.
struct DenseWide {
    const int* lo;   // per row: first column (window base); nullptr: no windows
    const int* hi;   // per row: last column
    int full;        // output width
    double* gacc;    // per CTA: full doubles (numeric)
    unsigned* gbits; // per CTA: (full + 31) / 32 words
};

template <bool kNumeric>
__global__ void __launch_bounds__(kDenseThreads) k_dense_rows(int r0, int rows, int ncols, const int* __restrict__ arp,
                                                             const int* __restrict__ aci, const double* __restrict__ av,
                                                             const int* __restrict__ brp, const int* __restrict__ bci,
                                                             const double* __restrict__ bv, int* __restrict__ cnt,
                                                             const int* __restrict__ crp, int* __restrict__ cci,
                                                             double* __restrict__ cv, unsigned* __restrict__ next,
                                                             DenseWide win) {
    extern __shared__ double dsm[];
    double* const sacc = dsm;  // ncols (numeric only)
    unsigned* const sbits = reinterpret_cast<unsigned*>(kNumeric ? dsm + ncols : dsm);
    __shared__ DenseChunk ch;
    __shared__ int s_row, s_total, s_scan[kDenseThreads + 1];
    __shared__ double s_prod[kDenseThreads / 32][32];
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    for (int k = t; k < ((ncols + 31) >> 5); k += kDenseThreads) sbits[k] = 0u;
    if (kNumeric)
        for (int k = t; k < ncols; k += kDenseThreads) sacc[k] = 0.0;
    __syncthreads();
    for (;;) {
        if (t == 0) s_row = (int)atomicAdd(next, 1u);
        __syncthreads();
        const int row = s_row;
        if (row >= rows) break;
        // this row's accumulator: the shared window, or the CTA's full-width global one
        int base = 0, width = ncols;
        double* acc = sacc;
        unsigned* bits = sbits;
        if (win.lo) {
            const int lo = win.lo[row], hi = win.hi[row];
            if (hi - lo < ncols) {
                base = lo;
            } else {
                width = win.full;
                bits = win.gbits + (size_t)blockIdx.x * ((win.full + 31) >> 5);
                if (kNumeric) acc = win.gacc + (size_t)blockIdx.x * win.full;
            }
        }
        const int nwords = (width + 31) >> 5;
        const int i = r0 + row, b = arp[i], e = arp[i + 1];
        for (int c0 = b; c0 < e; c0 += kDenseChunk) {
            // chunk of A entries: B-row starts, lengths -> inclusive offsets (block scan)
            const int kk = c0 + t;
            int len = 0;
            if (kk < e) {
                const int k = aci[kk];
                ch.bs[t] = brp[k];
                len = brp[k + 1] - ch.bs[t];
                if (kNumeric) ch.a[t] = av[kk];
            }
            s_scan[t + 1] = len;
            if (t == 0) s_scan[0] = 0;
            __syncthreads();
            for (int d = 1; d < kDenseThreads; d <<= 1) {  // Hillis-Steele inclusive scan
                const int v = t + 1 >= d + 1 ? s_scan[t + 1 - d] : 0;
                __syncthreads();
                s_scan[t + 1] += v;
                __syncthreads();
            }
            ch.off[t + 1] = s_scan[t + 1];
            if (t == 0) {
                ch.off[0] = 0;
                s_total = s_scan[kDenseThreads];
            }
            __syncthreads();
            const int total = s_total, na = min(kDenseChunk, e - c0);
            for (int q0 = 0; q0 < total; q0 += kDenseThreads) {
                const int q = q0 + t;
                int col = -1;
                double p = 0.0;
                if (q < total) {
                    int lo = 0, hi = na - 1;  // largest o with off[o] <= q
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (ch.off[mid] <= q)
                            lo = mid;
                        else
                            hi = mid - 1;
                    }
                    const int jj = ch.bs[lo] + (q - ch.off[lo]);
                    col = bci[jj] - base;
                    if (kNumeric) p = mul(ch.a[lo], bv[jj]);
                }
                if (!kNumeric) {
                    if (col >= 0) atomicOr(bits + (col >> 5), 1u << (col & 31));
                } else {
                    const unsigned grp = __match_any_sync(kFull, col);
                    const bool leader = col >= 0 && lane == __ffs(grp) - 1;
                    s_prod[w][lane] = p;
                    __syncwarp();
                    // warps add in warp order: Gustavson order across the 256 products
                    for (int ww = 0; ww < kDenseThreads / 32; ++ww) {
                        if (w == ww && leader) {
                            double a_ = acc[col];
                            for (unsigned m = grp; m; m &= m - 1) a_ = addd(a_, s_prod[w][__ffs(m) - 1]);
                            acc[col] = a_;
                            atomicOr(bits + (col >> 5), 1u << (col & 31));  // leaders may share a word
                        }
                        __syncthreads();
                    }
                }
            }
            __syncthreads();
        }
        // columns in order from the bitmap: per-thread word ranges, block prefix of popcounts
        const int per = (nwords + kDenseThreads - 1) / kDenseThreads;
        const int w0 = min(nwords, t * per), w1 = min(nwords, w0 + per);
        int mine = 0;
        for (int k = w0; k < w1; ++k) mine += __popc(bits[k]);
        s_scan[t + 1] = mine;
        if (t == 0) s_scan[0] = 0;
        __syncthreads();
        for (int d = 1; d < kDenseThreads; d <<= 1) {
            const int v = t + 1 >= d + 1 ? s_scan[t + 1 - d] : 0;
            __syncthreads();
            s_scan[t + 1] += v;
            __syncthreads();
        }
        if (!kNumeric) {
            if (t == 0) cnt[row] = s_scan[kDenseThreads];
            for (int k = w0; k < w1; ++k) bits[k] = 0u;
        } else {
            int o = crp[row] + s_scan[t];
            for (int k = w0; k < w1; ++k) {
                unsigned m = bits[k];
                while (m) {
                    const int col = (k << 5) + __ffs(m) - 1;
                    m &= m - 1;
                    cci[o] = col + base;
                    cv[o] = acc[col];
                    acc[col] = 0.0;
                    ++o;
                }
                bits[k] = 0u;
            }
        }
        __syncthreads();
    }
}

// first and last output column of each row: the first / last column of the B rows its A entries
// select (B rows are sorted)
__global__ void k_row_span(int r0, int rows, const int* __restrict__ arp, const int* __restrict__ aci,
                           const int* __restrict__ brp, const int* __restrict__ bci, int* __restrict__ lo,
                           int* __restrict__ hi, int width, unsigned* __restrict__ nwide) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    int a = INT_MAX, z = -1;
    for (int k = arp[r0 + r]; k < arp[r0 + r + 1]; ++k) {
        const int j = aci[k], s0 = brp[j], s1 = brp[j + 1];
        if (s1 > s0) a = min(a, bci[s0]), z = max(z, bci[s1 - 1]);
    }
    if (z < 0) a = z = 0;
    lo[r] = a;
    hi[r] = z;
    if (z - a >= width) atomicAdd(nwide, 1u);
}

constexpr int kDenseWideMax = 131072;  // widest output the windowed path takes (1 MB per CTA scratch)

// spmm_rows by the dense-accumulator kernels; nullptr when the output is too wide
Mat* spmm_dense(Ctx* c, const Mat* A, int r0, int r1, const Mat* B) {
    const int rows = r1 - r0, full = B->cols;
    if (rows <= 0 || full > kDenseWideMax || full <= 0) return nullptr;
    const bool windowed = full > kDenseCols;
    const int ncols = windowed ? kDenseCols : full;  // shared accumulator width
    DenseWide win{nullptr, nullptr, full, nullptr, nullptr};
    DBuf<int> lo, hi;
    if (windowed) {
        lo.alloc(c, (size_t)rows), hi.alloc(c, (size_t)rows);
        DBuf<unsigned> nwide(c, 1);
        CK(cudaMemsetAsync(nwide.p, 0, sizeof(unsigned), c->stream));
        k_row_span<<<(rows + 255) / 256, 256, 0, c->stream>>>(r0, rows, A->rp.p, A->ci.p, B->rp.p, B->ci.p, lo.p, hi.p,
                                                              ncols, nwide.p);
        CK_LAUNCH(c);
        // rows that overflow the window run at global-memory speed: worth it while they are few
        if ((long long)d2h_scalar(c, nwide.p) * 8 > rows) return nullptr;
        win.lo = lo.p, win.hi = hi.p;
    }
    const int nwords = (ncols + 31) / 32;
    const size_t sym_smem = sizeof(unsigned) * (size_t)nwords;
    const size_t num_smem = sizeof(double) * (size_t)ncols + sizeof(unsigned) * (size_t)nwords;
    IBM_SMEM_OPTIN(c, k_dense_rows<false>);
    IBM_SMEM_OPTIN(c, k_dense_rows<true>);
    int occ_s = 0, occ_n = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, k_dense_rows<false>, kDenseThreads, sym_smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_n, k_dense_rows<true>, kDenseThreads, num_smem));
    const int gs = std::max(1, std::min(rows, c->num_sms * std::max(occ_s, 1)));
    const int gn = std::max(1, std::min(rows, c->num_sms * std::max(occ_n, 1)));
    DBuf<unsigned> next(c, 2);
    CK(cudaMemsetAsync(next.p, 0, 2 * sizeof(unsigned), c->stream));
    DBuf<int> cnt(c, (size_t)rows + 1);
    if (windowed) {  // per-CTA full-width accumulators for the rows wider than the window: the
                     // context's zero scratch (the kernels clear what they touch)
        const size_t fw = (size_t)(full + 31) / 32;
        const size_t acc_b = sizeof(double) * (size_t)full * gn;
        char* z = static_cast<char*>(zero_scratch(c, acc_b + sizeof(unsigned) * fw * (size_t)std::max(gs, gn)));
        win.gacc = reinterpret_cast<double*>(z);
        win.gbits = reinterpret_cast<unsigned*>(z + acc_b);
    }
    k_dense_rows<false><<<gs, kDenseThreads, sym_smem, c->stream>>>(r0, rows, ncols, A->rp.p, A->ci.p, A->v.p, B->rp.p,
                                                                     B->ci.p, B->v.p, cnt.p, nullptr, nullptr, nullptr,
                                                                     next.p, win);
    CK_LAUNCH(c);
    Mat* m = mat_new(c, rows, full, 0);
    exclusive_scan_total(c, cnt.p, m->rp.p, rows);
    m->nnz = d2h_scalar(c, m->rp.p + rows);
    m->ci.alloc(c, (size_t)std::max(m->nnz, 1));
    m->v.alloc(c, (size_t)std::max(m->nnz, 1));
    k_dense_rows<true><<<gn, kDenseThreads, num_smem, c->stream>>>(r0, rows, ncols, A->rp.p, A->ci.p, A->v.p, B->rp.p,
                                                                    B->ci.p, B->v.p, nullptr, m->rp.p, m->ci.p, m->v.p,
                                                                    next.p + 1, win);
    CK_LAUNCH(c);
    return m;
}

Mat* esc_rows(Ctx* c, const Mat* A, int r0, int r1, const Mat* B);

// Hash path for rows [r0, r1) of A*B (rprod: products per row). Rows of more than
// kHashMaxProducts products — the few body-tail rows of the coarse Galerkin products reach
// millions — are gathered into a side matrix and go through ESC, which spreads them over the
// whole GPU; their results are placed back. nullptr if a short row's column count overflows.
constexpr long long kHashMaxProducts = 1 << 17;
Mat* spmm_hash(Ctx* c, const Mat* A, int r0, int r1, const Mat* B, const long long* rprod) {
    const int rows = r1 - r0;
    if (rows <= 0 || A->nnz == 0) return nullptr;
    const bool prof = std::getenv("IBMGPU_SETUP_PROFILE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what, long long extra) {
        if (!prof) return;
        sync(c);
        const auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[hash] rows %d %-9s %8.3f ms (%lld)\n", rows, what,
                     std::chrono::duration<double, std::milli>(t1 - t0).count(), extra);
        t0 = t1;
    };
    const long long limit = kHashMaxProducts;
    DBuf<int> cnt(c, (size_t)rows), mx(c, 1);
    CK(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (size_t)rows, c->stream));
    CK(cudaMemsetAsync(mx.p, 0, sizeof(int), c->stream));
    // long rows -> side matrix -> ESC
    DBuf<int> flag(c, (size_t)rows), pos(c, (size_t)rows + 1);
    k_long_flags<<<blocks(rows), 256, 0, c->stream>>>(rows, rprod, limit, flag.p);
    CK_LAUNCH(c);
    exclusive_scan_total(c, flag.p, pos.p, rows);
    const int nl = d2h_scalar(c, pos.p + rows);
    DBuf<int> lidx;
    Mat* Cl = nullptr;
    if (nl > 0) {
        lidx.alloc(c, (size_t)nl);
        DBuf<int> llen(c, (size_t)nl);
        k_long_rows<<<blocks(rows), 256, 0, c->stream>>>(rows, flag.p, pos.p, r0, A->rp.p, lidx.p, llen.p);
        CK_LAUNCH(c);
        Mat* Al = mat_new(c, nl, A->cols, 0);
        exclusive_scan_total(c, llen.p, Al->rp.p, nl);
        Al->nnz = d2h_scalar(c, Al->rp.p + nl);
        Al->ci.alloc(c, (size_t)std::max(Al->nnz, 1));
        Al->v.alloc(c, (size_t)std::max(Al->nnz, 1));
        k_gather_rows<<<nl, 256, 0, c->stream>>>(nl, lidx.p, r0, A->rp.p, A->ci.p, A->v.p, Al->rp.p, Al->ci.p,
                                                  Al->v.p);
        CK_LAUNCH(c);
        Cl = esc_rows(c, Al, 0, nl, B);
        delete Al;
        k_long_counts<<<blocks(nl), 256, 0, c->stream>>>(nl, lidx.p, Cl->rp.p, cnt.p);
        CK_LAUNCH(c);
    }
    lap("long/ESC", nl);
    std::unique_ptr<Mat> hold(Cl);
    const size_t sym_smem = sizeof(int) * (size_t)kSymWarps * kHashSym;
    IBM_SMEM_OPTIN(c, k_hash_symbolic);
    int sym_occ = 0;  // persistent grid: every CTA resident, rows handed out dynamically
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&sym_occ, k_hash_symbolic, kSymWarps * 32, sym_smem));
    const int sgrid = std::min((rows + kSymWarps - 1) / kSymWarps, c->num_sms * std::max(sym_occ, 1));
    DBuf<unsigned> next(c, 2);
    CK(cudaMemsetAsync(next.p, 0, 2 * sizeof(unsigned), c->stream));
    k_hash_symbolic<<<sgrid, kSymWarps * 32, sym_smem, c->stream>>>(r0, rows, A->rp.p, A->ci.p, B->rp.p, B->ci.p,
                                                                      cnt.p, mx.p, rprod, limit, next.p);
    CK_LAUNCH(c);
    const int maxc = d2h_scalar(c, mx.p);
    lap("symbolic", maxc);
    if (maxc > kHashSym * 3 / 4) return nullptr;
    int slots = 64;
    while (slots < 2 * maxc) slots <<= 1;
    const size_t per_warp = (size_t)slots * (sizeof(double) + sizeof(int)) + sizeof(HashChunk) + 32 * sizeof(double);
    const int nw = (int)std::max<size_t>(1, std::min<size_t>(8, (200u << 10) / per_warp));
    const size_t smem = per_warp * nw;
    Mat* m = mat_new(c, rows, B->cols, 0);
    exclusive_scan_total(c, cnt.p, m->rp.p, rows);
    m->nnz = d2h_scalar(c, m->rp.p + rows);
    m->ci.alloc(c, (size_t)std::max(m->nnz, 1));
    m->v.alloc(c, (size_t)std::max(m->nnz, 1));
    IBM_SMEM_OPTIN(c, k_hash_numeric);
    int num_occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&num_occ, k_hash_numeric, nw * 32, smem));
    const int ngrid = std::min((rows + nw - 1) / nw, c->num_sms * std::max(num_occ, 1));
    k_hash_numeric<<<ngrid, nw * 32, smem, c->stream>>>(r0, rows, A->rp.p, A->ci.p, A->v.p, B->rp.p, B->ci.p, B->v.p,
                                                        m->rp.p, m->ci.p, m->v.p, slots, rprod, limit, next.p + 1);
    CK_LAUNCH(c);
    if (nl > 0) {
        k_place_rows<<<nl, 256, 0, c->stream>>>(nl, lidx.p, Cl->rp.p, Cl->ci.p, Cl->v.p, m->rp.p, m->ci.p, m->v.p);
        CK_LAUNCH(c);
    }
    lap("numeric", slots);
    return m;
}

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
        c->pdl_fence = 1;
        k_transpose_fill<<<blocks(A->nnz), 256, 0, c->stream>>>(A->nnz, perm.p, row_of.p, A->v.p, t->ci.p, t->v.p);
        CK_LAUNCH(c);
    }
    return finish_plan(c, t);
}

Mat* spmm_rows(Ctx* c, const Mat* A, int r0, int r1, const Mat* B) {
    require(A->cols == B->rows, "spmm: dimension mismatch");
    if (r1 > r0 && A->nnz > 0 && !std::getenv("IBMGPU_ESC_ONLY")) {
        DBuf<long long> rprod(c, (size_t)(r1 - r0)), pref(c, (size_t)(r1 - r0) + 1);
        k_row_products<<<blocks(r1 - r0), 256, 0, c->stream>>>(r1 - r0, A->rp.p + r0, A->ci.p, B->rp.p, rprod.p);
        CK_LAUNCH(c);
        // a warp per row pays off only when rows carry at least a batch of products: the lhs2
        // assembly (4-8 products per row) stays on ESC (2.7 vs 5.1 ms per flapping refresh)
        const long long total = exclusive_scan_total64(c, rprod.p, pref.p, r1 - r0);
        // narrow outputs with long rows (coarse Galerkin products): a CTA per row, dense accumulator
        static const bool dense_on = [] {
            const char* e = std::getenv("IBMGPU_DENSE_SPGEMM");  // IBMGPU_DENSE_SPGEMM=0: hash only
            return !(e && e[0] == '0');
        }();
        // (windowed, wider outputs: only for rows of >= 1024 products — the level-2 P^T A of a
        // moving body; at ~300 products per row a CTA per row loses to the hash warps)
        if (dense_on && total >= 256ll * (r1 - r0) &&
            (B->cols <= kDenseCols || (B->cols <= kDenseWideMax && total >= 1024ll * (r1 - r0))))
            if (Mat* d = spmm_dense(c, A, r0, r1, B)) return finish_plan(c, d);
        if (total >= 32ll * (r1 - r0))
            if (Mat* h = spmm_hash(c, A, r0, r1, B, rprod.p)) return finish_plan(c, h);
    }
    return esc_rows(c, A, r0, r1, B);
}

namespace {
Mat* esc_rows(Ctx* c, const Mat* A, int r0, int r1, const Mat* B) {
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
}  // namespace

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

namespace {
// symmetrized() for a structurally symmetric A without forming A^T: entry (i, j) pairs with (j, i),
// found by binary search in row j; the sum is (0 + 0.5 a_ij) + 0.5 a_ji with exact zeros dropped,
// exactly what add_sparse(0.5, A, 0.5, A^T) computes (sparse.hpp:317-329, 351-353). An entry
// without a partner sets *asym and the caller takes the transpose path.
__global__ void k_sym_pairs(int rows, const int* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ v, int* __restrict__ cnt, const int* __restrict__ orp,
                            int* __restrict__ oci, double* __restrict__ ov, int* __restrict__ asym) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    int n = 0;
    const int o = orp ? orp[i] : 0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = ci[k];
        int lo = rp[j], hi = rp[j + 1];
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (ci[mid] < i)
                lo = mid + 1;
            else
                hi = mid;
        }
        if (lo == rp[j + 1] || ci[lo] != i) {
            *asym = 1;
            return;
        }
        const double s = addd(addd(0.0, mul(0.5, v[k])), mul(0.5, v[lo]));
        if (s != 0.0) {
            if (oci) {
                oci[o + n] = j;
                ov[o + n] = s;
            }
            ++n;
        }
    }
    if (cnt) cnt[i] = n;
}
}  // namespace

Mat* symmetrized(Ctx* c, const Mat* A) {
    if (A->rows == A->cols && A->rows > 0) {
        const int rows = A->rows;
        DBuf<int> cnt(c, (size_t)rows + 1), asym(c, 1);
        CK(cudaMemsetAsync(asym.p, 0, sizeof(int), c->stream));
        k_sym_pairs<<<blocks(rows), 256, 0, c->stream>>>(rows, A->rp.p, A->ci.p, A->v.p, cnt.p, nullptr, nullptr,
                                                         nullptr, asym.p);
        CK_LAUNCH(c);
        if (!d2h_scalar(c, asym.p)) {
            Mat* m = mat_new(c, rows, rows, 0);
            exclusive_scan_total(c, cnt.p, m->rp.p, rows);
            m->nnz = d2h_scalar(c, m->rp.p + rows);
            m->ci.alloc(c, (size_t)std::max(m->nnz, 1));
            m->v.alloc(c, (size_t)std::max(m->nnz, 1));
            k_sym_pairs<<<blocks(rows), 256, 0, c->stream>>>(rows, A->rp.p, A->ci.p, A->v.p, nullptr, m->rp.p,
                                                             m->ci.p, m->v.p, asym.p);
            CK_LAUNCH(c);
            return finish_plan(c, m);
        }
    }
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
