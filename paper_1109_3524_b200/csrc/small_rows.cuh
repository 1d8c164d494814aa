// small_rows.cuh — warp-per-row Gustavson for rows with few products (refresh.cu, amg_setup.cu).
// Products of a row are staged in shared memory in Gustavson order (A-row entry, then B-row
// entry), stably ranked by column (O(n^2) inside the warp; rows have at most kSmallCap products)
// and each column's run is summed by one lane from 0.0 in that order — the rounding of the
// reference's acc[c] += a*b (sparse.hpp:226-268), cancelled entries kept.
#pragma once
#include "kern.cuh"

namespace ibmgpu {
namespace {

constexpr int kSmallCap = 256, kSmallWarps = 4;

struct SmallRow {
    int col[kSmallCap];
    double val[kSmallCap];
    int scol[kSmallCap];
    double sval[kSmallCap];
};

// products of row entries (cols ci[b..e), values v) with the rows of M into w.col/val (n returned)
__device__ __forceinline__ int small_expand(SmallRow& w, const int* ci, const double* v, int b, int e, const int* __restrict__ mrp,
                            const int* __restrict__ mci, const double* __restrict__ mv, int lane) {
    int n = 0;
    for (int k = b; k < e; ++k) {  // A-row order
        const int kk = ci[k];
        const double a = v[k];
        const int s = mrp[kk], len = mrp[kk + 1] - s;
        IBM_DCHECK(n + len <= kSmallCap);
        for (int t = lane; t < len; t += 32) {  // B-row order
            w.col[n + t] = mci[s + t];
            w.val[n + t] = mul(a, mv[s + t]);
        }
        n += len;
    }
    __syncwarp();
    return n;
}

// stable rank by column, then one lane per column run sums it from 0.0; result (sorted by
// column) left in scol/sval[0..u), u returned
__device__ __forceinline__ int small_reduce(SmallRow& w, int n, int lane) {
    for (int s = lane; s < n; s += 32) {
        const int c = w.col[s];
        int r = 0;
        for (int t = 0; t < n; ++t) {
            const int ct = w.col[t];
            r += (ct < c) || (ct == c && t < s);
        }
        w.scol[r] = c;
        w.sval[r] = w.val[s];
    }
    __syncwarp();
    // heads of runs, compacted in order: u-th head at position w.col[u] (reuse col as head list)
    int u = 0;
    for (int base = 0; base < n; base += 32) {
        const int s = base + lane;
        const bool head = s < n && (s == 0 || w.scol[s] != w.scol[s - 1]);
        const unsigned m = __ballot_sync(0xffffffffu, head);
        if (head) w.col[u + __popc(m & ((1u << lane) - 1))] = s;
        u += __popc(m);
    }
    __syncwarp();
    for (int q = lane; q < u; q += 32) {
        const int s0 = w.col[q], s1 = q + 1 < u ? w.col[q + 1] : n;
        double acc = 0.0;
        for (int s = s0; s < s1; ++s) acc = addd(acc, w.sval[s]);
        w.val[q] = acc;  // value of the q-th unique column
    }
    __syncwarp();
    for (int q = lane; q < u; q += 32) w.col[q] = w.scol[w.col[q]];
    __syncwarp();
    for (int q = lane; q < u; q += 32) {
        w.scol[q] = w.col[q];
        w.sval[q] = w.val[q];
    }
    __syncwarp();
    return u;
}


}  // namespace
}  // namespace ibmgpu
