// amg_setup.cu — build_sa_hierarchy (amg.hpp:127-194) entirely on the device.
//
// Per level (identical semantics and rounding to the reference):
//   strength graph       amg.hpp:110-123  |a_ij| >= theta_l sqrt|a_ii a_jj| on the core block
//   aggregation          amg.hpp:79-107   exact replica of the sequential 3-pass greedy:
//                                          pass 1 is the lexicographically-first independent set of
//                                          the conflict relation N[i] ∩ N[s] ≠ ∅ (N[x] = {x} ∪ out(x)),
//                                          resolved by a persistent dependency-driven kernel (a node
//                                          decides once every lower conflicting node has decided) on
//                                          large levels, by the chunked sequential loop on small ones;
//                                          pass 2 follows "first already-assigned neighbour in column
//                                          order" chains by pointer jumping; pass 3 numbers leftovers
//   spectral radius      amg.hpp:58-75    10 power iterations, LCG start vector by jump-ahead
//   prolongator          amg.hpp:153-183  P_tent, DA*P_tent (ESC SpGEMM), add, identity tail, P^T
//   Galerkin             amg.hpp:188      sliced_triple_product(P^T, A, P) on the device
//   coarse               amg.hpp:191-192  dense SPD inverse (dense.cu)
#include <cub/cub.cuh>

#include <atomic>
#include <future>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>

#include "amg.cuh"
#include "internal.cuh"
#include "kern.cuh"
#include "small_rows.cuh"

namespace ibmgpu {

namespace {

inline int blocks(long long n, int b = 256) { return (int)((n + b - 1) / b); }

// ---------------------------------------------------------------- strength graph
__global__ void k_strength(int n_core, double theta, const int* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ v, const double* __restrict__ diag, int* __restrict__ cnt,
                           const int* __restrict__ orp, int* __restrict__ oci) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_core) return;
    int n = 0;
    const int o = orp ? orp[i] : 0;
    const double di = diag[i];
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = ci[k];
        if (j == i || j >= n_core) continue;
        const double bound = mul(theta, __dsqrt_rn(fabs(mul(di, diag[j]))));
        if (fabs(v[k]) >= bound && bound > 0.0) {
            if (oci) oci[o + n] = j;
            ++n;
        }
    }
    if (cnt) cnt[i] = n;
}

// ---------------------------------------------------------------- pass 1: LFMIS on the conflict relation
enum : int { UNDEC = 0, SEED = 1, NOTSEED = 2 };

// Persistent kernel: warps take 32-node tickets in index order. A node is NOTSEED as soon as a
// lower conflicting node is a SEED, and SEED once every lower conflicting node is NOTSEED.
// Lower conflicting nodes of i: s < i with s ∈ {u} ∪ in(u) for some u ∈ N[i] = {i} ∪ out(i).
// Progress: the warp holding the globally lowest undecided node can always decide it.
__global__ void __launch_bounds__(256) k_lfmis(int n, const int* __restrict__ srp, const int* __restrict__ sci,
                                               const int* __restrict__ trp, const int* __restrict__ tci,
                                               int* status, unsigned* ticket) {
    __shared__ int wstat[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    volatile int* gstat = status;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(ticket, 1u);
        t = __shfl_sync(kFull, t, 0);
        const long long base = (long long)t * 32;
        if (base >= n) return;
        const int i = (int)base + lane;
        int st = i < n ? UNDEC : NOTSEED;
        wstat[w][lane] = st;
        __syncwarp();
        // resume cursor: every candidate before (cq, cr) was NOTSEED when last seen, and NOTSEED is
        // final, so a re-scan starts at the first candidate that was still undecided
        const int ob = i < n ? srp[i] : 0, oe = i < n ? srp[i + 1] : 0;
        int cq = ob - 1, cr = -1;
        bool fresh = true;
        while (__any_sync(kFull, st == UNDEC)) {
            if (st == UNDEC) {
                bool pending = false, hit = false;
                int nq = cq, nr = cr;
                // u = i itself and u in out(i)
                for (int q = cq; q < oe && !hit; ++q) {
                    const int u = q < ob ? i : sci[q];
                    // candidates s = u (if u < i) and s in in(u) with s < i
                    const int tb = trp[u], te = trp[u + 1];
                    for (int r = (q == cq && !fresh) ? cr : tb - 1; r < te; ++r) {
                        const int s = r < tb ? u : tci[r];
                        if (s >= i) {
                            if (r >= tb) break;  // in-lists are sorted: the rest are >= i
                            continue;
                        }
                        const int ss = (s >= base) ? wstat[w][s - base] : gstat[s];
                        if (ss == SEED) {
                            hit = true;
                            break;
                        }
                        if (ss == UNDEC && !pending) {
                            pending = true;
                            nq = q, nr = r;
                        }
                    }
                }
                if (hit)
                    st = NOTSEED;
                else if (!pending)
                    st = SEED;
                else
                    cq = nq, cr = nr, fresh = false;
                if (st != UNDEC) {
                    gstat[i] = st;
                    wstat[w][lane] = st;
                }
            }
            __syncwarp();
        }
    }
}

// Pass 1, the reference's sequential loop itself (amg.hpp:85-95), run by ONE warp with the
// "assigned" set as a bitmap in shared memory. Lanes test a row's columns in parallel (ballot); rows
// arrive through a cp.async ring kGD rows ahead. Kept as the plainest restatement (IBMGPU_AGG=seq);
// k_greedy_chunk below computes the same seeds faster on every level measured.
constexpr int kGD = 16, kGW = 256, kWin = 1024;

__device__ __forceinline__ void cp_async4(int* dst, const int* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::); }
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(kGD - 1)); }

__global__ void __launch_bounds__(32) k_greedy_seq(int n, const int* __restrict__ srp, const int* __restrict__ sci,
                                                   int* __restrict__ status) {
    extern __shared__ unsigned smem[];
    const int nwords = (n + 31) >> 5;
    unsigned* bits = smem;
    int* ring = reinterpret_cast<int*>(bits + nwords);
    int* rpw = ring + kGD * kGW;  // row pointers of the current window (kWin + kGD + 1)
    const int lane = threadIdx.x;
    for (int w = lane; w < nwords; w += 32) bits[w] = 0u;
    int w0 = 0;
    auto load_window = [&](int base) {
        w0 = base;
        for (int t = lane; t <= kWin + kGD; t += 32) rpw[t] = __ldg(srp + min(base + t, n));
        __syncwarp();
    };
    auto issue = [&](int j) {  // prefetch row j into its slot; one commit group per row, always
        if (j < n) {
            const int b = rpw[j - w0], len = min(rpw[j - w0 + 1] - b, kGW);
            int* slot = ring + (j % kGD) * kGW;
            for (int k = lane; k < len; k += 32) cp_async4(slot + k, sci + b + k);
        }
        cp_commit();
    };
    load_window(0);
    for (int j = 0; j < kGD; ++j) issue(j);
    for (int i = 0; i < n; ++i) {
        if (i - w0 == kWin) load_window(i);
        cp_wait();
        __syncwarp();
        const int b = rpw[i - w0], len = rpw[i - w0 + 1] - b;
        const int* slot = ring + (i % kGD) * kGW;
        bool covered = (bits[i >> 5] >> (i & 31)) & 1u;
        if (!covered) {
            bool hit = false;
            for (int k = lane; k < len; k += 32) {
                const int cidx = k < kGW ? slot[k] : __ldg(sci + b + k);
                hit |= (bits[cidx >> 5] >> (cidx & 31)) & 1u;
            }
            covered = __any_sync(kFull, hit);
        }
        if (!covered) {  // seed: assign N[i] = {i} and its strong neighbours
            if (lane == 0) atomicOr(bits + (i >> 5), 1u << (i & 31));
            for (int k = lane; k < len; k += 32) {
                const int cidx = k < kGW ? slot[k] : __ldg(sci + b + k);
                atomicOr(bits + (cidx >> 5), 1u << (cidx & 31));
            }
        }
        if (lane == 0) status[i] = covered ? NOTSEED : SEED;
        __syncwarp();
        issue(i + kGD);  // the slot of row i is free again
    }
    asm volatile("cp.async.wait_all;" ::);
}

// Pass 1 for dense levels of any size that fit a shared-memory bitmap: the same sequential loop,
// split so that only its truly serial part is serial. Rows go in chunks of <= kChunk rows whose
// strong-neighbour lists (contiguous in S) are staged in shared memory by cp.async one chunk ahead.
//   phase A (32 warps): a row is "covered" if it or a strong neighbour is assigned at chunk start;
//                       covering only grows, so a row covered now is covered in the reference too;
//   phase B (warp 0):   the remaining candidates in index order; the first one is a seed outright,
//                       later ones are re-tested against the bits the chunk's earlier seeds set.
// Same seeds as k_greedy_seq; on levels with tens of strong neighbours per row most rows are
// settled in phase A.
constexpr int kChunk = 1024;

// any assigned node among cols[q0, q1): four independent column loads in flight per step
__device__ __forceinline__ bool any_assigned(const unsigned* bits, const int* cols, int q0, int q1) {
    int q = q0;
    for (; q + 4 <= q1; q += 4) {
        const int j0 = cols[q], j1 = cols[q + 1], j2 = cols[q + 2], j3 = cols[q + 3];
        const unsigned b = (bits[j0 >> 5] >> (j0 & 31)) | (bits[j1 >> 5] >> (j1 & 31)) |
                           (bits[j2 >> 5] >> (j2 & 31)) | (bits[j3 >> 5] >> (j3 & 31));
        if (b & 1u) return true;
    }
    for (; q < q1; ++q) {
        const int j = cols[q];
        if ((bits[j >> 5] >> (j & 31)) & 1u) return true;
    }
    return false;
}

template <bool kLane>
__global__ void __launch_bounds__(kChunk) k_greedy_chunk(int n, const int* __restrict__ srp,
                                                         const int* __restrict__ sci, int* __restrict__ status,
                                                         int cap) {
    extern __shared__ __align__(16) unsigned csm[];
    const int nwords = (n + 31) >> 5;
    unsigned* bits = csm;
    int* rpb = reinterpret_cast<int*>(bits + ((nwords + 3) & ~3));  // [2][kChunk + 1] row pointers
    int* cflag = rpb + 2 * (kChunk + 4);                             // [kChunk] candidate flags
    int* meta = cflag + kChunk;                                      // [2][4]: base, end, aligned start
    int* buf = meta + 8;                                             // [2][cap] column lists
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    for (int k = t; k < nwords; k += kChunk) bits[k] = 0u;

    // bounds of the chunk starting at `base` and its loads into slot `sl`; one commit group per call
    auto stage = [&](int base, int sl) {
        int* rpw = rpb + sl * (kChunk + 4);
        int* m = meta + 4 * sl;
        const int s = base < n ? __ldg(srp + base) : 0;
        const int a = s & ~3;
        int e = 0;
        bool in = false;
        if (base + t < n) {
            e = __ldg(srp + base + t + 1);
            in = e - a <= cap;
            rpw[t + 1] = e;
        }
        int rows = __syncthreads_count(in);  // the predicate is monotone in t: a prefix
        if (base < n && rows == 0) rows = 1;  // one row longer than the buffer: read it from global
        const int end = min(base + rows, n);
        const int ee = base < n ? __ldg(srp + end) : 0;
        const bool global = ee - a > cap;
        if (t == 0) {
            rpw[0] = s;
            m[0] = base, m[1] = end, m[2] = a, m[3] = global;
        }
        if (base < n && !global) {
            int* dst = buf + sl * cap;
            const int v1 = ee >> 2;  // whole int4s [a/4, v1), then the tail ints
            for (int v = (a >> 2) + t; v < v1; v += kChunk) {
                const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst + (v * 4 - a)));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(sci + v * 4));
            }
            for (int x = max(v1 * 4, a) + t; x < ee; x += kChunk) cp_async4(dst + (x - a), sci + x);
        }
        cp_commit();
    };

    stage(0, 0);
    for (int k = 0;; ++k) {
        const int sl = k & 1;
        __syncthreads();
        const int base = meta[4 * sl], end = meta[4 * sl + 1], a = meta[4 * sl + 2];
        if (base >= n) break;
        stage(end, sl ^ 1);  // prefetch the next chunk while this one is processed
        asm volatile("cp.async.wait_group 1;" ::);
        __syncthreads();
        const int* rpw = rpb + sl * (kChunk + 4);
        const int* cols = meta[4 * sl + 3] ? sci + a : buf + sl * cap;  // column q at cols[q - a]
        const int rows = end - base;
        // phase A: short rows one per thread; long rows one per warp, lanes across the columns
        if (kLane) {
            if (t < rows) {
                const int i = base + t;
                const bool cov = ((bits[i >> 5] >> (i & 31)) & 1u) || any_assigned(bits, cols - a, rpw[t], rpw[t + 1]);
                cflag[t] = !cov;
            }
        } else
        for (int r = w; r < rows; r += kChunk / 32) {
            const int i = base + r;
            bool cov = (bits[i >> 5] >> (i & 31)) & 1u;
            if (!cov) {
                bool hit = false;
                for (int q = rpw[r] + lane; q < rpw[r + 1]; q += 32) {
                    const int j = cols[q - a];
                    hit |= (bits[j >> 5] >> (j & 31)) & 1u;
                }
                cov = __any_sync(kFull, hit);
            }
            if (lane == 0) cflag[r] = !cov;
        }
        __syncthreads();
        // phase B: candidates in index order
        if (kLane && w == 0) {
            // lane-parallel rounds over 32 rows: every undecided candidate re-tests its own row; the
            // lowest still-uncovered one is a seed (everything below it is decided), the covered
            // ones are final; repeat until the group is decided
            for (int g = 0; g < rows; g += 32) {
                const int r = g + lane, i = base + r;
                bool und = r < rows && cflag[r];
                const int q0 = r < rows ? rpw[r] : 0, q1 = r < rows ? rpw[r + 1] : 0;
                // the first kReg columns of the row stay in registers for the repeated tests: each
                // round is then kReg independent bitmap loads instead of a dependent column walk
                constexpr int kReg = 16;
                int rc[kReg];
#pragma unroll
                for (int u = 0; u < kReg; ++u) rc[u] = (und && q0 + u < q1) ? cols[q0 + u - a] : i;
                for (;;) {
                    bool cov = false;
                    if (und) {
                        unsigned b = bits[i >> 5] >> (i & 31);
#pragma unroll
                        for (int u = 0; u < kReg; ++u) b |= bits[rc[u] >> 5] >> (rc[u] & 31);
                        cov = (b & 1u) || (q1 - q0 > kReg && any_assigned(bits, cols - a, q0 + kReg, q1));
                    }
                    und = und && !cov;
                    const unsigned U = __ballot_sync(kFull, und);
                    if (!U) break;
                    const int leader = __ffs(U) - 1;
                    const int s0 = __shfl_sync(kFull, q0, leader), s1 = __shfl_sync(kFull, q1, leader);
                    if (lane == leader) {
                        atomicOr(bits + (i >> 5), 1u << (i & 31));
                        status[i] = SEED;
                        und = false;
                    }
                    for (int q = s0 + lane; q < s1; q += 32) {
                        const int j = cols[q - a];
                        atomicOr(bits + (j >> 5), 1u << (j & 31));
                    }
                    __syncwarp();
                }
            }
        } else if (w == 0) {
            bool seeded = false;
            for (int g = 0; g < rows; g += 32) {
                unsigned m = __ballot_sync(kFull, g + lane < rows && cflag[g + lane]);
                while (m) {
                    const int r = g + __ffs(m) - 1;
                    m &= m - 1;
                    const int i = base + r, q0 = rpw[r], q1 = rpw[r + 1];
                    bool cov = false;
                    if (seeded) {
                        bool hit = lane == 0 && ((bits[i >> 5] >> (i & 31)) & 1u);
                        for (int q = q0 + lane; q < q1; q += 32) {
                            const int j = cols[q - a];
                            hit |= (bits[j >> 5] >> (j & 31)) & 1u;
                        }
                        cov = __any_sync(kFull, hit);
                    }
                    if (!cov) {  // seed: assign N[i]
                        if (lane == 0) {
                            atomicOr(bits + (i >> 5), 1u << (i & 31));
                            status[i] = SEED;
                        }
                        for (int q = q0 + lane; q < q1; q += 32) {
                            const int j = cols[q - a];
                            atomicOr(bits + (j >> 5), 1u << (j & 31));
                        }
                        seeded = true;
                    }
                    __syncwarp();
                }
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::);
}

// shared memory of k_greedy_chunk for n rows and a column buffer of cap ints per slot
inline size_t chunk_smem(int n, int cap) {
    const size_t words = (size_t)(((n + 31) / 32 + 3) & ~3);
    return sizeof(int) * (words + 2 * (kChunk + 4) + kChunk + 8 + 2 * (size_t)cap);
}

// ---------------------------------------------------------------- pass 1 on a grid-shaped graph
// When every strength edge of row i goes to i-S, i-1, i+1 or i+S of a grid of NY lines of S
// cells (the level-0 pressure stencil), the sequential greedy of amg.hpp:84-96 is a recurrence
// with short reach. In index order, the decision for cell (j, x) needs:
//   * its own coverage so far: seed(j, x-1) over a +1 edge, or seed(j-1, x) over a +S edge;
//   * for a -S edge, whether (j-1, x) was covered by a seed before (j, x):
//     seed(j-1, x) itself, seed(j-1, x-+1) over +-1 edges, or seed(j-2, x) over +S;
//   * for a -1 edge, whether (j, x-1) was covered: seed(j, x-1), seed(j, x-2) over +1, or
//     seed(j-1, x-1) over +S;
//   * for a +1 edge, whether (j, x+1) was covered: only seed(j-1, x+1) over +S can have;
//   * nothing for a +S edge: no earlier seed reaches (j+1, x).
// So a line only needs the line above's decisions two columns ahead. A warp runs 32 lines
// (lane l is line 32w + l, two columns behind lane l - 1), passing each step's two bits down by
// shuffle. The warp below reads its top line's bits from the warp above through global words
// published every 32 columns. The output is the same seed set as the sequential loop, by
// construction (tests compare the aggregates with the reference's).
constexpr int kGridEP = 16;  // ebits row pitch multiple (uint4 loads)

// edge bits per cell: 1 = -S, 2 = -1, 4 = +1, 8 = +S; *bad if an edge is anything else
__global__ void k_grid_ebits(int n_core, int S, int pitch, const int* __restrict__ srp, const int* __restrict__ sci,
                             unsigned char* __restrict__ eb, int* __restrict__ bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_core) return;
    const int x = i % S, j = i / S;
    unsigned b = 0;
    for (int k = srp[i]; k < srp[i + 1]; ++k) {
        const int d = sci[k] - i;
        if (d == -S) b |= 1u;
        else if (d == -1 && x > 0) b |= 2u;
        else if (d == 1 && x < S - 1) b |= 4u;
        else if (d == S) b |= 8u;
        else atomicOr(bad, 1);
    }
    eb[(size_t)j * pitch + x] = (unsigned char)b;
}

__device__ __forceinline__ unsigned grid_byte(const uint4& q, int k) {  // byte k (0..15) of q
    const unsigned w = k < 8 ? (k < 4 ? q.x : q.y) : (k < 12 ? q.z : q.w);
    return (w >> (8 * (k & 3))) & 0xffu;
}

__global__ void __launch_bounds__(32) k_greedy_grid(int S, int NY, int pitch, const unsigned char* __restrict__ eb,
                                                    unsigned* hC, unsigned* hS, int* progress, unsigned* ticket,
                                                    int* status) {
    __shared__ int ws;
    if (threadIdx.x == 0) ws = (int)atomicAdd(ticket, 1u);  // warps start in line order
    __syncwarp();
    const int w = ws, lane = threadIdx.x;
    const int j = w * 32 + lane;
    const bool line = j < NY;
    const int nwords = (S + 31) / 32;
    const unsigned char* row = eb + (size_t)(line ? j : 0) * pitch;
    unsigned covB = 0, sP1 = 0;   // (j, x-1) covered before (j, x); seed(j, x-1) over a +1 edge
    unsigned outC = 0, outS = 0;  // published: C(j, x-1) and sPS(j, x) of this lane's last column
    unsigned sPSup = 0;           // sPS(j-1, x), received the step before
    unsigned accC = 0, accS = 0;  // lane 31: words being assembled
    int cwC = -1, cwS = -1, have = 0;         // lane 0: cached words of the warp above
    unsigned vC = 0, vS = 0;
    uint4 cur = make_uint4(0, 0, 0, 0), nxt = make_uint4(0, 0, 0, 0);
    if (line) {
        cur = *reinterpret_cast<const uint4*>(row);
        if (kGridEP < pitch) nxt = *reinterpret_cast<const uint4*>(row + kGridEP);
    }
    // t = -1: lane 0's column -1 step, which fetches sPS of the line above at column 0
    const int T = S + 1 + 2 * 31;
    for (int t = -1; t < T; ++t) {
        const int x = t - 2 * lane;
        // from the line above: C(j-1, x) and sPS(j-1, x+1) (its previous step's column x+1)
        unsigned inC = __shfl_up_sync(kFull, outC, 1), inS = __shfl_up_sync(kFull, outS, 1);
        if (lane == 0) {
            inC = inS = 0;
            if (w > 0 && x >= -1 && x < S) {
                const int need = min(nwords, (x + 1) / 32 + 1);  // words holding x and x+1
                if (have < need) {
                    while ((have = *reinterpret_cast<volatile int*>(progress + w - 1)) < need) __nanosleep(32);
                    __threadfence();
                }
                if (x >= 0) {
                    IBM_DCHECK(x / 32 < have);
                    if (x / 32 != cwC) cwC = x / 32, vC = __ldcg(hC + (size_t)(w - 1) * nwords + cwC);
                    inC = (vC >> (x & 31)) & 1u;
                }
                if (x + 1 < S) {
                    if ((x + 1) / 32 != cwS) cwS = (x + 1) / 32, vS = __ldcg(hS + (size_t)(w - 1) * nwords + cwS);
                    inS = (vS >> ((x + 1) & 31)) & 1u;
                }
            }
        }
        if (x >= 0 && x <= S) {
            unsigned e = 0;
            if (line && x < S) {
                const int k = x & (kGridEP - 1);
                e = grid_byte(cur, k);
                if (k == kGridEP - 1) {  // next 16-column window; prefetch the one after
                    cur = nxt;
                    if (x + 1 + kGridEP < pitch) nxt = *reinterpret_cast<const uint4*>(row + x + 1 + kGridEP);
                }
            }
            const unsigned cov = sP1 | sPSup;
            unsigned seed = 0;
            if (line && x < S) {
                bool fr = cov == 0;
                if (e & 1u) fr = fr && !inC;
                if (e & 2u) fr = fr && !covB;
                if (e & 4u) fr = fr && !inS;
                if (fr) {
                    seed = 1;
                    IBM_DCHECK((size_t)j * S + x < (size_t)NY * S);
                    status[(size_t)j * S + x] = SEED;
                }
            }
            outC = covB | (seed & ((e >> 1) & 1u));  // C(j, x-1): a -1 edge of this seed covers it
            outS = seed & ((e >> 3) & 1u);           // sPS(j, x)
            covB = cov | seed;
            sP1 = seed & ((e >> 2) & 1u);
            if (lane == 31 && line) {
                // an sPS word is complete one column before the C word of the same index: it is
                // stored at once, and the C word's progress bump (after the fence) publishes both
                if (x < S) {
                    accS |= outS << (x & 31);
                    if ((x & 31) == 31 || x == S - 1) {
                        hS[(size_t)w * nwords + x / 32] = accS;
                        accS = 0;
                    }
                }
                if (x >= 1) {
                    accC |= outC << ((x - 1) & 31);
                    if (((x - 1) & 31) == 31 || x - 1 == S - 1) {
                        const int wd = (x - 1) / 32;
                        hC[(size_t)w * nwords + wd] = accC;
                        accC = 0;
                        __threadfence();
                        atomicExch(progress + w, wd + 1);
                    }
                }
            }
        }
        if (x >= -1) sPSup = inS;  // sPS(j-1, x+1): the next column's sPS(j-1, x)
    }
}

__global__ void k_seed_flags(int n, const int* __restrict__ status, int* __restrict__ flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = status[i] == SEED;
}

// seeds cover N[s]; conflict-freeness of seeds makes the writes race-free
__global__ void k_cover(int n, const int* __restrict__ status, const int* __restrict__ seed_id,
                        const int* __restrict__ srp, const int* __restrict__ sci, int* __restrict__ agg) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n || status[s] != SEED) return;
    const int id = seed_id[s];
    agg[s] = id;
    for (int q = srp[s]; q < srp[s + 1]; ++q) agg[sci[q]] = id;
}

// pass 2 target: first out-neighbour j (column order) that is pass-1 assigned or a lower leftover
__global__ void k_pass2_target(int n, const int* __restrict__ agg1, const int* __restrict__ srp,
                               const int* __restrict__ sci, int* __restrict__ tgt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (agg1[i] != -1) {
        tgt[i] = -1;
        return;
    }
    int t = -2;  // -2: no assigned neighbour (pass 3; only reachable for an asymmetric S)
    for (int q = srp[i]; q < srp[i + 1]; ++q) {
        const int j = sci[q];
        if (agg1[j] != -1 || j < i) {
            t = j;
            break;
        }
    }
    tgt[i] = t;
}

// pointer jumping along leftover chains until every target is a pass-1-assigned node. Every
// leftover has a pass-1-assigned out-neighbour (it was not a seed, so a seed covered part of
// N[i], and i itself is uncovered), so each lower leftover is assigned by the time i is visited.
__global__ void k_pass2_jump(int n, const int* __restrict__ agg1, int* tgt, int* changed) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int t = tgt[i];
    if (t < 0 || agg1[t] != -1) return;
    const int tt = tgt[t];
    if (tt >= 0 && tt != t) {
        tgt[i] = tt;
        *changed = 1;
    }
}

__global__ void k_pass2_apply(int n, const int* __restrict__ agg1, const int* __restrict__ tgt, int* __restrict__ agg) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || agg1[i] != -1) return;
    const int t = tgt[i];
    agg[i] = t >= 0 ? agg1[t] : -1;
}

__global__ void k_unassigned(int n, const int* __restrict__ agg, int* __restrict__ flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = agg[i] == -1;
}

__global__ void k_pass3(int n, int base, const int* __restrict__ flag, const int* __restrict__ pos, int* __restrict__ agg) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) agg[i] = base + pos[i];
}

// ---------------------------------------------------------------- prolongator pieces
__global__ void k_agg_size(int n, const int* __restrict__ agg, int* __restrict__ size) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        IBM_DCHECK(agg[i] >= 0);  // pass 3 leaves no row unassigned
        atomicAdd(size + agg[i], 1);
    }
}

// P_tent (amg.hpp:156-161): rows < n_core hold (agg[i], 1/sqrt(|agg|)); tail rows empty
__global__ void k_ptent(int rows, int n_core, const int* __restrict__ agg, const int* __restrict__ size,
                        int* __restrict__ rp, int* __restrict__ ci, double* __restrict__ v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > rows) return;
    rp[i] = i < n_core ? i : n_core;
    if (i < n_core) {
        const int a = agg[i];
        ci[i] = a;
        v[i] = __ddiv_rn(1.0, __dsqrt_rn((double)size[a]));
    }
}

// P (amg.hpp:163-178) in one pass, one warp per row of P: core row i is
//   add_sparse(1.0, P_tent, -omega, spmm(D^{-1}A, P_tent)) row i
// = for each column a: (0.0 [+ 1.0 * ptent_i if a == agg_i]) + (-omega) * dap_a, exact zeros
// dropped, where dap_a sums mul(mul(a_ik, invd_i), ptent_k) over k in A-row order with agg_k == a
// (Gustavson over the one-entry rows of P_tent; tail columns of A meet empty P_tent rows);
// tail row n_core + t is the identity entry (n_agg + t, 1.0). Rows with more than kSmallCap
// core entries set *over and the caller takes the general path.
__device__ __forceinline__ double ptent_val(const int* __restrict__ size, int a) {
    return __ddiv_rn(1.0, __dsqrt_rn((double)size[a]));
}

__global__ void __launch_bounds__(kSmallWarps * 32)
    k_smooth_p(int rows, int n_core, int n_agg, double omega, const int* __restrict__ arp,
               const int* __restrict__ aci, const double* __restrict__ av, const double* __restrict__ invd,
               const int* __restrict__ agg, const int* __restrict__ size, int* __restrict__ cnt,
               const int* __restrict__ orp, int* __restrict__ oci, double* __restrict__ ov, int* __restrict__ over) {
    __shared__ SmallRow ws[kSmallWarps];
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    SmallRow& w = ws[wi];
    for (int i = blockIdx.x * kSmallWarps + wi; i < rows; i += gridDim.x * kSmallWarps) {
        if (i >= n_core) {
            if (lane == 0) {
                if (cnt) {
                    cnt[i] = 1;
                } else {
                    oci[orp[i]] = n_agg + (i - n_core);
                    ov[orp[i]] = 1.0;
                }
            }
            continue;
        }
        const int b = arp[i], e = arp[i + 1];
        // products in A-row order (core columns only: P_tent's tail rows are empty)
        int n = 0;
        const double di = invd[i];
        for (int k0 = b; k0 < e; k0 += 32) {
            const int k = k0 + lane;
            const bool core = k < e && aci[k] < n_core;
            const unsigned m = __ballot_sync(0xffffffffu, core);
            if (n + __popc(m) > kSmallCap) {
                if (lane == 0) *over = 1;
                n = -1;
                break;
            }
            if (core) {
                const int kk = aci[k];
                const int a = agg[kk];
                const int pos = n + __popc(m & ((1u << lane) - 1));
                w.col[pos] = a;
                w.val[pos] = mul(mul(av[k], di), ptent_val(size, a));
            }
            n += __popc(m);
        }
        __syncwarp();
        if (n < 0) continue;
        const int u = small_reduce(w, n, lane);  // DAP row: columns sorted, Gustavson sums
        const int ai = agg[i];
        const double pti = ptent_val(size, ai);
        // merge with the single P_tent entry (ai, pti); values (0 + 1.0*pt) + (-omega)*dap
        bool has_ai = false;
        for (int q = lane; q < u; q += 32) has_ai |= w.scol[q] == ai;
        has_ai = __any_sync(0xffffffffu, has_ai);
        const int total = u + (has_ai ? 0 : 1);
        // write in column order; an exact-zero sum is dropped (from_triplets), counted by ballot
        int outn = 0;
        const int o = cnt ? 0 : orp[i];
        for (int base = 0; base < total; base += 32) {
            const int q = base + lane;
            int col = 0;
            double v = 0.0;
            bool keep = false;
            if (q < total) {
                // position q of the merged list: ai inserted before the first column > ai
                int ins = 0;  // number of DAP columns < ai
                for (int t = 0; t < u; ++t) ins += w.scol[t] < ai;
                if (has_ai) {
                    col = w.scol[q];
                    v = addd(col == ai ? addd(0.0, mul(1.0, pti)) : 0.0, mul(-omega, w.sval[q]));
                } else if (q == ins) {
                    col = ai;
                    v = addd(0.0, mul(1.0, pti));
                } else {
                    const int t = q < ins ? q : q - 1;
                    col = w.scol[t];
                    v = addd(0.0, mul(-omega, w.sval[t]));
                }
                keep = v != 0.0;
            }
            const unsigned km = __ballot_sync(0xffffffffu, keep);
            if (!cnt && keep) {
                const int pos = o + outn + __popc(km & ((1u << lane) - 1));
                oci[pos] = col;
                ov[pos] = v;
            }
            outn += __popc(km);
        }
        if (cnt && lane == 0) cnt[i] = outn;
        __syncwarp();
    }
}

__global__ void k_invd(int n, const double* __restrict__ d, double omega, double* __restrict__ invd,
                       double* __restrict__ wd, int* __restrict__ zero) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double di = d[i];
    if (di == 0.0) {
        *zero = 1;
        invd[i] = 0.0;
    } else {
        invd[i] = __ddiv_rn(1.0, di);
    }
    if (wd) wd[i] = mul(omega, invd[i]);
}

// ---------------------------------------------------------------- power iteration (amg.hpp:58-75)
__host__ __device__ inline void lcg_compose(unsigned long long& a, unsigned long long& c, unsigned long long a2,
                                            unsigned long long c2) {
    // (x -> a2 (a x + c) + c2)
    c = a2 * c + c2;
    a = a2 * a;
}

__global__ void k_lcg_start(int n, double* __restrict__ v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // s_{i+1} = f^{i+1}(s0), f(x) = x*A + C mod 2^64
    unsigned long long ra = 1, rc = 0, pa = 6364136223846793005ull, pc = 1442695040888963407ull;
    unsigned long long e = (unsigned long long)i + 1;
    while (e) {
        if (e & 1) lcg_compose(ra, rc, pa, pc);
        // square: f∘f
        const unsigned long long na = pa * pa, nc = pa * pc + pc;
        pa = na, pc = nc;
        e >>= 1;
    }
    const unsigned long long s = ra * 0x9e3779b97f4a7c15ull + rc;
    v[i] = 0.5 + (double)(s >> 11) / (double)(1ull << 53);
}

struct PowerState {
    double lambda;
    int zero;
};

struct EpiPower {  // w_i = s * invd_i ; reduce w^2 ; lambda = sqrt(sum)
    static constexpr int NR = 1;
    const double* invd;
    double* w;
    RedSlot rs;
    PowerState* ps;
    __device__ bool skip() const { return ps->zero != 0; }
    __device__ void row(int i, double s, double* acc) const {
        const double wi = mul(s, invd[i]);
        w[i] = wi;
        acc[0] += wi * wi;
    }
    __device__ RedSlot slot() const { return rs; }
    __device__ void fin(double* tot) const {
        const double lam = __dsqrt_rn(tot[0]);
        ps->lambda = lam;
        if (lam == 0.0) ps->zero = 1;
    }
};

__global__ void k_normalize(int n, const double* __restrict__ w, const PowerState* ps, double* __restrict__ v) {
    if (ps->zero) return;
    const double lam = ps->lambda;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = __ddiv_rn(w[i], lam);
}

double rho_dinv_a(Ctx* c, Mat* A, const double* invd, int iters) {
    const int n = A->rows;
    if (!A->planned) mat_plan(c, A);
    DBuf<double> v(c, n), w(c, n);
    DBuf<PowerState> ps(c, 1);
    CK(cudaMemsetAsync(ps.p, 0, sizeof(PowerState), c->stream));
    const int g = spmv_grid(A);
    DBuf<double> part(c, (size_t)std::max(g, 1));
    DBuf<unsigned> cnt(c, 1);
    CK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned), c->stream));
    k_lcg_start<<<blocks(n), 256, 0, c->stream>>>(n, v.p);
    CK_LAUNCH(c);
    for (int it = 0; it < iters; ++it) {
        launch_spmv(c, A, XPlain{v.p}, EpiPower{invd, w.p, RedSlot{part.p, cnt.p}, ps.p}, c->stream);
        k_normalize<<<elem_grid(c, n), 256, 0, c->stream>>>(n, w.p, ps.p, v.p);
        CK_LAUNCH(c);
    }
    PowerState h = d2h_scalar(c, ps.p);
    if (iters == 0) return 1.0;
    return h.zero ? 1.0 : h.lambda;
}

// Fused coarse sub-cycle (coarse.cuh): every level from the first one whose operator is small
// enough (<= kFuseRows rows) down to the dense solve runs in one persistent launch. Level 0 is
// never fused (its post-smoother carries the PCG's fused r.z reduction).
constexpr int kFuseRows = 0;  // measured slower than separate graph launches on B200; opt in via IBMGPU_FUSE_ROWS

void build_fused_coarse(Ctx* c, Hier* h) {
    const int L = (int)h->levels.size();
    const char* ev = std::getenv("IBMGPU_FUSE_ROWS");
    const int fuse_rows = ev ? std::atoi(ev) : kFuseRows;
    const char* ec = std::getenv("IBMGPU_FUSE_CTAS");
    const int ctas_per_sm = ec ? std::max(1, std::atoi(ec)) : 1;
    int F = L;
    while (F > 1 && h->levels[F - 1]->A->rows <= fuse_rows) --F;
    if (F >= L) return;
    std::vector<Phase> ph;
    auto spmv_phase = [&](int kind, Mat* M) {
        mat_plan_adaptive(c, M);
        Phase p{};
        p.kind = kind;
        p.n_blocks = M->n_blocks;
        p.pl = AdaptPlan{M->blk_meta.p, M->lrow.p, M->lpart.p, M->lcnt.p};
        p.rp = M->rp.p;
        p.ci = M->ci.p;
        p.v = M->v.p;
        return p;
    };
    for (int l = F; l < L; ++l) {
        Level& lv = *h->levels[l];
        Phase k1 = spmv_phase(PH_JACOBI, lv.A);
        k1.wd = lv.wd.p, k1.b = lv.b.p, k1.x = lv.x.p, k1.out = lv.r.p;
        ph.push_back(k1);
        Phase k2 = spmv_phase(PH_STORE, lv.Pt);
        k2.x = lv.r.p, k2.out = l + 1 < L ? h->levels[l + 1]->b.p : h->cb.p;
        ph.push_back(k2);
    }
    Phase g{};
    g.kind = PH_GEMV;
    g.n_blocks = h->n_c;
    g.v = h->coarse_inv.p;
    g.x = h->cb.p;
    g.out = h->cx.p;
    ph.push_back(g);
    for (int l = L - 1; l >= F; --l) {
        Level& lv = *h->levels[l];
        Phase k3 = spmv_phase(PH_ADD, lv.P);
        k3.x = l + 1 < L ? h->levels[l + 1]->xo.p : h->cx.p;
        k3.out = lv.x.p;
        ph.push_back(k3);
        Phase k4 = spmv_phase(PH_POST, lv.A);
        k4.wd = lv.wd.p, k4.b = lv.b.p, k4.x = lv.x.p, k4.out = lv.xo.p;
        ph.push_back(k4);
    }
    h->fuse_from = F;
    h->n_phases = (int)ph.size();
    h->phases.alloc(c, ph.size());
    h2d(c, h->phases.p, ph.data(), ph.size());
    h->bar.alloc(c, 2);
    CK(cudaMemsetAsync(h->bar.p, 0, 2 * sizeof(unsigned), c->stream));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coarse_cycle, kBlock, 0));
    // every CTA must be co-resident for the software grid barrier
    h->coarse_grid = std::max(1, std::min(per_sm, ctas_per_sm) * c->num_sms);
}

}  // namespace

namespace {
// IBMGPU_SETUP_PROFILE=1: per-phase wall times of the hierarchy build on stderr (syncs per phase)
struct SetupClock {
    Ctx* c;
    bool on;
    std::chrono::steady_clock::time_point t;
    explicit SetupClock(Ctx* c_) : c(c_) {
        const char* e = std::getenv("IBMGPU_SETUP_PROFILE");
        on = e && e[0] == '1';
        t = std::chrono::steady_clock::now();
    }
    void lap(const char* what, int lev) {
        if (!on) return;
        sync(c);
        const auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[sa_build] L%d %-10s %8.3f ms\n", lev, what,
                     std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};
}  // namespace

// Strength graph + exact greedy aggregation; returns aggregate count, agg sized n_core.
__global__ void k_neq(int n, const int* __restrict__ a, const int* __restrict__ b, int* __restrict__ diff) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (a[i] != b[i]) {
            *diff = 1;
            return;
        }
}

int aggregate_device(Ctx* c, const Mat* A, double theta, int n_core, DBuf<int>& agg, AggCache::Lv* cache,
                     bool* hit, int grid_S) {
    if (grid_S == 0 && A->kind == SPMV_STENCIL && A->st_S2 == 0) grid_S = A->st_S1;
    if (hit) *hit = false;
    agg.alloc(c, (size_t)std::max(n_core, 1));
    if (n_core == 0) return 0;
    DBuf<double> diag(c, (size_t)A->rows);
    diag_of(c, A, diag.p);
    // S (pattern only)
    DBuf<int> cnt(c, (size_t)n_core + 1);
    Mat S;
    S.rows = S.cols = n_core;
    S.rp.alloc(c, (size_t)n_core + 1);
    k_strength<<<blocks(n_core), 256, 0, c->stream>>>(n_core, theta, A->rp.p, A->ci.p, A->v.p, diag.p, cnt.p, nullptr,
                                                      nullptr);
    CK_LAUNCH(c);
    exclusive_scan_total(c, cnt.p, S.rp.p, n_core);
    S.nnz = d2h_scalar(c, S.rp.p + n_core);
    S.ci.alloc(c, (size_t)S.nnz);
    S.v.alloc(c, (size_t)S.nnz);
    CK(cudaMemsetAsync(S.v.p, 0, sizeof(double) * (size_t)S.nnz, c->stream));
    k_strength<<<blocks(n_core), 256, 0, c->stream>>>(n_core, theta, A->rp.p, A->ci.p, A->v.p, diag.p, nullptr,
                                                      S.rp.p, S.ci.p);
    CK_LAUNCH(c);
    if (cache && cache->n_core == n_core && cache->nnz == S.nnz) {
        DBuf<int> diff(c, 1);
        CK(cudaMemsetAsync(diff.p, 0, sizeof(int), c->stream));
        const int g = std::max(1, std::min(c->num_sms * 8, blocks(std::max(S.nnz, n_core + 1))));
        k_neq<<<g, 256, 0, c->stream>>>(n_core + 1, S.rp.p, cache->rp.p, diff.p);
        CK_LAUNCH(c);
        if (S.nnz) {
            k_neq<<<g, 256, 0, c->stream>>>(S.nnz, S.ci.p, cache->ci.p, diff.p);
            CK_LAUNCH(c);
        }
        if (!d2h_scalar(c, diff.p)) {
            d2d(c, agg.p, cache->agg.p, (size_t)n_core);
            if (hit) *hit = true;
            return cache->n_agg;
        }
    }
    SetupClock clk(c);
    Mat* St = transpose(c, &S);  // in-neighbour lists (sorted by source row)
    clk.lap("  agg:S+St", -2);

    // pass 1
    DBuf<int> status(c, (size_t)n_core), seedflag(c, (size_t)n_core), seed_id(c, (size_t)n_core + 1);
    DBuf<unsigned> ticket(c, 1);
    CK(cudaMemsetAsync(status.p, 0, sizeof(int) * (size_t)n_core, c->stream));
    CK(cudaMemsetAsync(ticket.p, 0, sizeof(unsigned), c->stream));
    // IBMGPU_AGG=seq|chunkl|chunkw|lfmis forces a pass-1 kernel (A/B timing, tests); all give the same seeds
    const char* force = std::getenv("IBMGPU_AGG");
    const std::string pick = force ? force : "";
    int max_smem = 0;
    CK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
    const size_t fixed = chunk_smem(n_core, 0);
    const int cap = fixed < (size_t)max_smem ? (int)(((size_t)max_smem - fixed) / 8) & ~3 : 0;
    // Default: the chunked loop (one row per thread/lane) up to kChunkMax rows, the LFMIS above.
    // Measured (ms, chunked-lane vs LFMIS): flapping L2 66k rows 5.6 vs 19.0, L3 6.3k 0.49 vs 4.5;
    // S-4M L3 78k 7.9 vs 16.6, L2 351k 42.9 vs 19.6; flapping L1 199k 32 vs 3.7 (the single CTA's
    // serial rounds grow with the seed count; the LFMIS spreads over all SMs).
    constexpr int kChunkMax = 131072;
    const bool chunk_ok = cap >= 4096;
    const bool lane = pick != "chunkw";
    const bool use_chunk = pick.rfind("chunk", 0) == 0 ? chunk_ok : pick.empty() ? chunk_ok && n_core <= kChunkMax : false;
    // grid-shaped strength graph (level 0 of a stencil operator): the line-pipelined replica
    bool grid_ok = false;
    int gpitch = 0, gwarps = 0;
    DBuf<unsigned char> gebits;
    DBuf<unsigned> ghC, ghS;
    DBuf<int> gprog;
    if (!use_chunk && grid_S > 1 && n_core % grid_S == 0 && (pick.empty() || pick == "grid")) {
        const int NY = n_core / grid_S;
        gpitch = (grid_S + kGridEP - 1) / kGridEP * kGridEP;
        gwarps = (NY + 31) / 32;
        gebits.alloc(c, (size_t)NY * gpitch);
        DBuf<int> gbad(c, 1);
        CK(cudaMemsetAsync(gbad.p, 0, sizeof(int), c->stream));
        k_grid_ebits<<<blocks(n_core), 256, 0, c->stream>>>(n_core, grid_S, gpitch, S.rp.p, S.ci.p, gebits.p, gbad.p);
        CK_LAUNCH(c);
        grid_ok = d2h_scalar(c, gbad.p) == 0;
        if (grid_ok) {
            const size_t nw = (size_t)gwarps * ((grid_S + 31) / 32);
            ghC.alloc(c, nw), ghS.alloc(c, nw), gprog.alloc(c, (size_t)gwarps);
            CK(cudaMemsetAsync(gprog.p, 0, sizeof(int) * (size_t)gwarps, c->stream));
        }
    }
    if (use_chunk) {
        const size_t smem = chunk_smem(n_core, cap);
        IBM_SMEM_OPTIN(c, k_greedy_chunk<true>);
        IBM_SMEM_OPTIN(c, k_greedy_chunk<false>);
        auto kern = lane ? k_greedy_chunk<true> : k_greedy_chunk<false>;
        kern<<<1, kChunk, smem, c->stream>>>(n_core, S.rp.p, S.ci.p, status.p, cap);
        CK_LAUNCH(c);
    } else if (grid_ok) {
        k_greedy_grid<<<gwarps, 32, 0, c->stream>>>(grid_S, n_core / grid_S, gpitch, gebits.p, ghC.p, ghS.p,
                                                     gprog.p, ticket.p, status.p);
        CK_LAUNCH(c);
    } else if (pick == "seq") {
        const size_t smem = sizeof(unsigned) * (size_t)((n_core + 31) / 32) + sizeof(int) * (kGD * kGW + kWin + kGD + 1);
        IBM_SMEM_OPTIN(c, k_greedy_seq);
        k_greedy_seq<<<1, 32, smem, c->stream>>>(n_core, S.rp.p, S.ci.p, status.p);
        CK_LAUNCH(c);
    } else {
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lfmis, 256, 0));
        const int grid = std::max(1, std::min(per_sm * c->num_sms, (n_core + 255) / 256));
        k_lfmis<<<grid, 256, 0, c->stream>>>(n_core, S.rp.p, S.ci.p, St->rp.p, St->ci.p, status.p, ticket.p);
        CK_LAUNCH(c);
    }
    clk.lap("  agg:lfmis", -2);
    k_seed_flags<<<blocks(n_core), 256, 0, c->stream>>>(n_core, status.p, seedflag.p);
    CK_LAUNCH(c);
    exclusive_scan_total(c, seedflag.p, seed_id.p, n_core);
    const int n_seeds = d2h_scalar(c, seed_id.p + n_core);
    DBuf<int> agg1(c, (size_t)n_core);
    CK(cudaMemsetAsync(agg1.p, 0xff, sizeof(int) * (size_t)n_core, c->stream));
    k_cover<<<blocks(n_core), 256, 0, c->stream>>>(n_core, status.p, seed_id.p, S.rp.p, S.ci.p, agg1.p);
    CK_LAUNCH(c);

    // pass 2: pointer jumping over "first assigned neighbour" chains
    DBuf<int> tgt(c, (size_t)n_core), changed(c, 1);
    k_pass2_target<<<blocks(n_core), 256, 0, c->stream>>>(n_core, agg1.p, S.rp.p, S.ci.p, tgt.p);
    CK_LAUNCH(c);
    for (int round = 0; round < 64; ++round) {
        CK(cudaMemsetAsync(changed.p, 0, sizeof(int), c->stream));
        k_pass2_jump<<<blocks(n_core), 256, 0, c->stream>>>(n_core, agg1.p, tgt.p, changed.p);
        CK_LAUNCH(c);
        if (!d2h_scalar(c, changed.p)) break;
    }
    clk.lap("  agg:cover+p2", -2);
    d2d(c, agg.p, agg1.p, (size_t)n_core);
    k_pass2_apply<<<blocks(n_core), 256, 0, c->stream>>>(n_core, agg1.p, tgt.p, agg.p);
    CK_LAUNCH(c);

    // pass 3: leftovers numbered after the seeds in index order
    DBuf<int> flag(c, (size_t)n_core), pos(c, (size_t)n_core + 1);
    k_unassigned<<<blocks(n_core), 256, 0, c->stream>>>(n_core, agg.p, flag.p);
    CK_LAUNCH(c);
    exclusive_scan_total(c, flag.p, pos.p, n_core);
    const int n3 = d2h_scalar(c, pos.p + n_core);
    if (n3) {
        k_pass3<<<blocks(n_core), 256, 0, c->stream>>>(n_core, n_seeds, flag.p, pos.p, agg.p);
        CK_LAUNCH(c);
    }
    delete St;
    if (cache) {
        cache->n_core = n_core;
        cache->nnz = S.nnz;
        cache->n_agg = n_seeds + n3;
        cache->rp = std::move(S.rp);
        cache->ci = std::move(S.ci);
        cache->agg.alloc(c, (size_t)n_core);
        d2d(c, cache->agg.p, agg.p, (size_t)n_core);
    }
    return n_seeds + n3;
}


// k_smooth_p with one thread per row, for rows of at most kThreadCap core entries (level 0:
// at most 16); a longer row sets *over and the warp kernel runs instead
constexpr int kThreadCap = 24;
__global__ void k_smooth_p_thread(int rows, int n_core, int n_agg, double omega, const int* __restrict__ arp,
                                  const int* __restrict__ aci, const double* __restrict__ av,
                                  const double* __restrict__ invd, const int* __restrict__ agg,
                                  const int* __restrict__ size, int* __restrict__ cnt, const int* __restrict__ orp,
                                  int* __restrict__ oci, double* __restrict__ ov, int* __restrict__ over) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    if (i >= n_core) {
        if (cnt) {
            cnt[i] = 1;
        } else {
            oci[orp[i]] = n_agg + (i - n_core);
            ov[orp[i]] = 1.0;
        }
        return;
    }
    int col[kThreadCap + 1];
    double val[kThreadCap + 1];
    int n = 0;
    const double di = invd[i];
    for (int k = arp[i]; k < arp[i + 1]; ++k) {
        const int kk = aci[k];
        if (kk >= n_core) continue;  // P_tent's tail rows are empty
        if (n == kThreadCap) {
            *over = 1;
            return;
        }
        const int a = agg[kk];
        const double p = mul(mul(av[k], di), ptent_val(size, a));
        // Gustavson: the first product of a column starts from 0.0, later ones add in A-row order
        int t = 0;
        while (t < n && col[t] != a) ++t;
        if (t < n) {
            val[t] = addd(val[t], p);
        } else {
            col[n] = a;
            val[n] = addd(0.0, p);
            ++n;
        }
    }
    // the P_tent entry of the row's own aggregate, then columns in increasing order
    const int ai = agg[i];
    const double pti = addd(0.0, mul(1.0, ptent_val(size, ai)));
    bool has_ai = false;
    for (int t = 0; t < n; ++t) has_ai |= col[t] == ai;
    if (!has_ai) {
        col[n] = ai;
        val[n] = 0.0;  // marker: no DAP entry (handled below)
    }
    const int total = n + (has_ai ? 0 : 1);
    int outn = 0;
    const int o = cnt ? 0 : orp[i];
    int last = -1;
    for (int q = 0; q < total; ++q) {
        int best = -1;  // next column above `last` (selection: rows are short)
        for (int t = 0; t < total; ++t)
            if (col[t] > last && (best < 0 || col[t] < col[best])) best = t;
        last = col[best];
        double v;
        if (best == n)  // P_tent only
            v = pti;
        else
            v = addd(col[best] == ai ? pti : 0.0, mul(-omega, val[best]));
        if (v != 0.0) {
            if (!cnt) {
                oci[o + outn] = col[best];
                ov[o + outn] = v;
            }
            ++outn;
        }
    }
    if (cnt) cnt[i] = outn;
}

// P in one fused pass (k_smooth_p); nullptr when a row is too long for it
Mat* smoothed_prolongator(Ctx* c, const Mat* A, const double* invd, const int* agg, const int* size, int n_core,
                          int n_agg, double omega) {
    const int rows = A->rows, tail = rows - n_core;
    DBuf<int> cnt(c, (size_t)rows + 1), over(c, 1);
    CK(cudaMemsetAsync(over.p, 0, sizeof(int), c->stream));
    const int grid = std::max(1, std::min(blocks(rows, kSmallWarps), c->num_sms * 8));
    int hv[2];
    // thread per row first; the warp kernel when some row is longer than kThreadCap
    bool thread = true;
    k_smooth_p_thread<<<blocks(rows), 256, 0, c->stream>>>(rows, n_core, n_agg, omega, A->rp.p, A->ci.p, A->v.p,
                                                           invd, agg, size, cnt.p, nullptr, nullptr, nullptr, over.p);
    CK_LAUNCH(c);
    hv[0] = d2h_scalar(c, over.p);
    if (hv[0]) {
        thread = false;
        CK(cudaMemsetAsync(over.p, 0, sizeof(int), c->stream));
        k_smooth_p<<<grid, kSmallWarps * 32, 0, c->stream>>>(rows, n_core, n_agg, omega, A->rp.p, A->ci.p, A->v.p,
                                                             invd, agg, size, cnt.p, nullptr, nullptr, nullptr, over.p);
        CK_LAUNCH(c);
    }
    Mat* P = mat_new(c, rows, n_agg + tail, 0);
    exclusive_scan_total(c, cnt.p, P->rp.p, rows);
    d2h(c, hv, over.p, 1);
    d2h(c, hv + 1, P->rp.p + rows, 1);
    sync(c);
    if (hv[0]) {
        delete P;
        return nullptr;
    }
    P->nnz = hv[1];
    P->ci.alloc(c, (size_t)std::max(P->nnz, 1));
    P->v.alloc(c, (size_t)std::max(P->nnz, 1));
    if (thread)
        k_smooth_p_thread<<<blocks(rows), 256, 0, c->stream>>>(rows, n_core, n_agg, omega, A->rp.p, A->ci.p, A->v.p,
                                                               invd, agg, size, nullptr, P->rp.p, P->ci.p, P->v.p,
                                                               over.p);
    else
        k_smooth_p<<<grid, kSmallWarps * 32, 0, c->stream>>>(rows, n_core, n_agg, omega, A->rp.p, A->ci.p, A->v.p,
                                                             invd, agg, size, nullptr, P->rp.p, P->ci.p, P->v.p,
                                                             over.p);
    CK_LAUNCH(c);
    return P;
}

// A second stream (and context view of the same device) for setup work that runs beside the
// main stream's critical path.
struct AuxStream {
    Ctx c;
    cudaEvent_t fork = nullptr, join = nullptr;
    explicit AuxStream(Ctx* main) {
        c.device = main->device;
        c.num_sms = main->num_sms;
        c.eager = main->eager;
        c.pool = main->pool;
        CK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    }
    ~AuxStream() {
        cudaStreamSynchronize(c.stream);
        zero_scratch_free(&c);
        cudaEventDestroy(fork);
        cudaEventDestroy(join);
        cudaStreamDestroy(c.stream);
        c.stream = nullptr;
    }
};

Hier* sa_build(Ctx* c, const Mat* A_fine, const ibm_sa_options& o, AggCache* cache) {
    require(A_fine->rows == A_fine->cols, "sa: square matrix required");
    SetupClock clk(c);
    static std::atomic<long long> next_id{1};
    auto* h = new Hier();
    h->id = next_id++;
    try {
        const int tail = std::min(o.keep_fine_tail, A_fine->rows);
        AuxStream aux(c);
        // level-0 A is a private copy (the hierarchy owns every level, as SaLevel::A does)
        Mat* A = scale(c, A_fine, 0, 1.0, nullptr);
        for (int lev = 0; lev < o.max_levels && A->rows > o.max_coarse + tail; ++lev) {
            const double theta_l = o.theta * std::pow(0.5, lev);
            const int n_core = A->rows - tail;
            auto L = std::make_unique<Level>();
            if (cache && cache->lv.size() <= (size_t)lev) cache->lv.resize(lev + 1);
            const int n = A->rows;
            DBuf<double> d(c, (size_t)n);
            diag_of(c, A, d.p);
            L->invd.alloc(c, (size_t)n);
            DBuf<int> zero(c, 1);
            CK(cudaMemsetAsync(zero.p, 0, sizeof(int), c->stream));
            k_invd<<<blocks(n), 256, 0, c->stream>>>(n, d.p, 0.0, L->invd.p, nullptr, zero.p);
            CK_LAUNCH(c);
            // The power iteration (amg.hpp:58-75, with this level's SpMV plan) only needs A and
            // 1/diag, the aggregation (amg.hpp:79-123) only A: they run concurrently, the power
            // iteration from a helper thread on the aux stream. Same kernels, same results.
            CK(cudaEventRecord(aux.fork, c->stream));
            CK(cudaStreamWaitEvent(aux.c.stream, aux.fork, 0));
            const double* invd_p = L->invd.p;
            static const bool aux_on = [] {
                const char* e = std::getenv("IBMGPU_AUX");  // IBMGPU_AUX=0: power iteration inline
                return !(e && e[0] == '0');
            }();
            auto rho_f = std::async(aux_on ? std::launch::async : std::launch::deferred,
                                    [&aux, A, invd_p, &o, dev = c->device] {
                                        CK(cudaSetDevice(dev));
                                        return rho_dinv_a(&aux.c, A, invd_p, o.power_iterations);
                                    });
            bool hit = false;
            int n_agg = 0;
            try {
                // level 0 of a stencil operator: the copy is not planned yet, the input's plan has the stride
                const int gS = lev == 0 && A_fine->kind == SPMV_STENCIL && A_fine->st_S2 == 0 ? A_fine->st_S1 : 0;
                n_agg = aggregate_device(c, A, theta_l, n_core, L->agg, cache ? &cache->lv[lev] : nullptr, &hit, gS);
            } catch (...) {
                rho_f.wait();
                throw;
            }
            const double rho = rho_f.get();
            c->launches += aux.c.launches;
            aux.c.launches = 0;
            CK(cudaEventRecord(aux.join, aux.c.stream));
            CK(cudaStreamWaitEvent(c->stream, aux.join, 0));
            mat_rehome(A, c->stream);  // its SpMV plan was built on the aux stream
            if (cache) ++(hit ? cache->hits : cache->misses);
            clk.lap("aggregate+rho", lev);
            if (n_agg >= n_core) {
                h->stalled = true;
                break;
            }
            if (d2h_scalar(c, zero.p)) {
                delete A;
                fail(IBMGPU_EINVAL, "sa: zero diagonal");
            }
            const double omega = (4.0 / 3.0) / rho;
            L->wd.alloc(c, (size_t)n);
            k_invd<<<blocks(n), 256, 0, c->stream>>>(n, d.p, omega, L->invd.p, L->wd.p, zero.p);
            CK_LAUNCH(c);

            // tentative prolongator
            DBuf<int> size(c, (size_t)n_agg);
            CK(cudaMemsetAsync(size.p, 0, sizeof(int) * (size_t)n_agg, c->stream));
            k_agg_size<<<blocks(n_core), 256, 0, c->stream>>>(n_core, L->agg.p, size.p);
            CK_LAUNCH(c);
            // P = (I - omega D^{-1} A) P_tent on the core; identity on the tail
            Mat* P = smoothed_prolongator(c, A, L->invd.p, L->agg.p, size.p, n_core, n_agg, omega);
            if (!P) {  // a row with more than kSmallCap core entries: the general product
                Mat* Ptent = mat_new(c, n, n_agg, n_core);
                k_ptent<<<blocks(n + 1), 256, 0, c->stream>>>(n, n_core, L->agg.p, size.p, Ptent->rp.p, Ptent->ci.p,
                                                              Ptent->v.p);
                CK_LAUNCH(c);
                Mat* DA = scale(c, A, 1, 0.0, L->invd.p);
                Mat* DAP = spmm_rows(c, DA, 0, DA->rows, Ptent);
                delete DA;
                Mat* Pcore = add(c, 1.0, Ptent, -omega, DAP);
                delete DAP;
                delete Ptent;
                P = tail > 0 ? identity_tail_append(c, Pcore, n_core, n_agg, tail) : Pcore;
                if (tail > 0) delete Pcore;
            }
            clk.lap("P", lev);
            Mat* Pt = transpose(c, P);
            clk.lap("transpose", lev);
            Mat* Ac = triple_product(c, Pt, A, P, std::max(1, Pt->rows), nullptr, nullptr);
            clk.lap("galerkin", lev);

            L->A = A;
            L->P = P;
            L->Pt = Pt;
            L->omega = omega;
            L->n_core = n_core;
            L->n_agg = n_agg;
            h->levels.push_back(std::move(L));
            A = Ac;
        }
        h->coarse_A = A;
        h->n_c = A->rows;
        // V-cycle plans + work vectors
        for (size_t l = 0; l < h->levels.size(); ++l) {
            Level& lv = *h->levels[l];
            for (Mat* m : {lv.A, lv.P, lv.Pt})
                if (!m->planned) mat_plan(c, m);
            const size_t n = (size_t)lv.A->rows;
            if (l > 0) lv.b.alloc(c, n), lv.xj.alloc(c, n);
            lv.x.alloc(c, n);
            lv.r.alloc(c, n);
            lv.xo.alloc(c, n);
        }
        clk.lap("plans", -1);
        h->coarse_inv.alloc(c, (size_t)h->n_c * h->n_c);
        dense_spd_inverse(c, h->coarse_A, h->coarse_inv.p);
        clk.lap("coarse", -1);
        h->n_dense = h->n_c;
        fold_tail(c, h, kSymvTile);
        clk.lap("fold", -1);
        const int nd = h->n_dense;
        h->coarse_tiles.alloc(c, packed_tiles_doubles(nd));
        h->prow.alloc(c, packed_partials_doubles(nd));
        h->pcol.alloc(c, packed_partials_doubles(nd));
        pack_symmetric_tiles(c, nd, h->n_fold ? h->dense.p : h->coarse_inv.p, h->coarse_tiles.p);
        h->cb.alloc(c, (size_t)nd);
        h->cx.alloc(c, (size_t)nd);
        if (h->n_fold) {
            h->dense.release();
            h->coarse_inv.release();
        } else {
            build_fused_coarse(c, h);
        }
        xfer0_setup(c, h);
        clk.lap("xfer0", -1);
        sync(c);
    } catch (...) {
        delete h;
        throw;
    }
    return h;
}

}  // namespace ibmgpu
