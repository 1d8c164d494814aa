// dist_plan.cpp — see dist_plan.hpp.
#include "dist_plan.hpp"

#include <algorithm>
#include <cstring>
#include <stdexcept>

#include "../../../include/ibmgpu.h"

namespace ibmhost {

DistPlan make_dist_plan(int rows, int cols, const int* rp, const int* ci, const double* v, const int* row_owner,
                        const int* col_owner, int rank, int nranks) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("dist: bad rank");
    DistPlan P;
    P.rank = rank;
    P.nranks = nranks;
    P.rows_global = rows;
    P.cols_global = cols;
    // owned input entries and their local positions
    std::vector<int> g2l(static_cast<size_t>(cols), -1);
    for (int c = 0; c < cols; ++c)
        if (col_owner[c] == rank) {
            g2l[c] = static_cast<int>(P.own.size());
            P.own.push_back(c);
        }
    P.n_own = static_cast<int>(P.own.size());
    // halo: remote columns referenced by owned rows, grouped by peer (ascending within peer)
    std::vector<std::vector<int>> by_peer(static_cast<size_t>(nranks));
    std::vector<char> seen(static_cast<size_t>(cols), 0);
    for (int r = 0; r < rows; ++r) {
        if (row_owner[r] != rank) continue;
        P.rows.push_back(r);
        for (int k = rp[r]; k < rp[r + 1]; ++k) {
            const int c = ci[k];
            if (col_owner[c] != rank && !seen[c]) {
                seen[c] = 1;
                by_peer[col_owner[c]].push_back(c);
            }
        }
    }
    P.recv_off.assign(static_cast<size_t>(nranks) + 1, 0);
    for (int q = 0; q < nranks; ++q) {
        auto& h = by_peer[q];
        std::sort(h.begin(), h.end());
        for (int c : h) {
            g2l[c] = P.n_own + static_cast<int>(P.halo.size());
            P.halo.push_back(c);
        }
        P.recv_off[q + 1] = static_cast<int>(P.halo.size());
    }
    // local CSR in extended numbering (entry order unchanged)
    P.rp.push_back(0);
    for (int r : P.rows) {
        for (int k = rp[r]; k < rp[r + 1]; ++k) {
            P.ci.push_back(g2l[ci[k]]);
            P.v.push_back(v ? v[k] : 0.0);
        }
        P.rp.push_back(static_cast<int>(P.ci.size()));
    }
    // send lists: for every peer q, the owned columns its rows reference (ascending) — the same
    // set and order as q's halo segment for this rank
    P.send_off.assign(static_cast<size_t>(nranks) + 1, 0);
    std::vector<int> mark(static_cast<size_t>(cols), -1);
    for (int q = 0; q < nranks; ++q) {
        std::vector<int> need;
        if (q != rank) {
            for (int r = 0; r < rows; ++r) {
                if (row_owner[r] != q) continue;
                for (int k = rp[r]; k < rp[r + 1]; ++k) {
                    const int c = ci[k];
                    if (col_owner[c] == rank && mark[c] != q) {
                        mark[c] = q;
                        need.push_back(c);
                    }
                }
            }
            std::sort(need.begin(), need.end());
        }
        for (int c : need) {
            // owned-local index of c (position in `own`)
            P.send_idx.push_back(static_cast<int>(std::lower_bound(P.own.begin(), P.own.end(), c) - P.own.begin()));
        }
        P.send_off[q + 1] = static_cast<int>(P.send_idx.size());
    }
    return P;
}

std::vector<int> partition_lambda(int nx, int ny, int n_b, const int* body_cell_j, int nranks) {
    std::vector<int> slab_of_j(static_cast<size_t>(ny));
    for (int j = 0; j < ny; ++j) slab_of_j[j] = static_cast<int>((static_cast<long long>(j) * nranks) / ny);
    std::vector<int> owner(static_cast<size_t>(nx) * ny + 2 * static_cast<size_t>(n_b));
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) owner[static_cast<size_t>(i) + static_cast<size_t>(j) * nx] = slab_of_j[j];
    const size_t np = static_cast<size_t>(nx) * ny;
    for (int k = 0; k < n_b; ++k) {
        const int jj = std::clamp(body_cell_j[k], 0, ny - 1);
        owner[np + k] = slab_of_j[jj];
        owner[np + n_b + k] = slab_of_j[jj];
    }
    return owner;
}

std::vector<int> partition_coarse(const std::vector<int>& owner_l, const int* agg, int n_core, int n_agg, int tail) {
    std::vector<int> out(static_cast<size_t>(n_agg) + tail, -1);
    for (int i = 0; i < n_core; ++i)
        if (out[agg[i]] < 0) out[agg[i]] = owner_l[i];  // rows visited ascending: lowest member wins
    for (int t = 0; t < tail; ++t) out[static_cast<size_t>(n_agg) + t] = owner_l[static_cast<size_t>(n_core) + t];
    for (int& o : out)
        if (o < 0) o = 0;
    return out;
}

}  // namespace ibmhost

// ---------------------------------------------------------------- host-only C entry points
struct ibmgpu_distplan {
    ibmhost::DistPlan p;
};

extern "C" {

int ibmgpu_distplan_build(int rows, int cols, const int* rp, const int* ci, const double* v, const int* row_owner,
                          const int* col_owner, int rank, int nranks, ibmgpu_distplan_t* out) {
    try {
        auto* d = new ibmgpu_distplan();
        d->p = ibmhost::make_dist_plan(rows, cols, rp, ci, v, row_owner, col_owner, rank, nranks);
        *out = d;
        return 0;
    } catch (const std::invalid_argument&) {
        return IBMGPU_EINVAL;
    } catch (...) {
        return IBMGPU_ECUDA;
    }
}

int ibmgpu_distplan_sizes(ibmgpu_distplan_t d, int* out6) {
    const auto& p = d->p;
    out6[0] = static_cast<int>(p.rows.size());
    out6[1] = p.n_own;
    out6[2] = p.n_halo();
    out6[3] = static_cast<int>(p.ci.size());
    out6[4] = static_cast<int>(p.send_idx.size());
    out6[5] = p.nranks;
    return 0;
}

int ibmgpu_distplan_get(ibmgpu_distplan_t d, int* rows, int* own, int* rp, int* ci, double* v, int* recv_off,
                        int* halo, int* send_off, int* send_idx) {
    const auto& p = d->p;
    auto cp = [](int* dst, const std::vector<int>& s) {
        if (dst && !s.empty()) std::memcpy(dst, s.data(), sizeof(int) * s.size());
    };
    cp(rows, p.rows);
    cp(own, p.own);
    cp(rp, p.rp);
    cp(ci, p.ci);
    if (v && !p.v.empty()) std::memcpy(v, p.v.data(), sizeof(double) * p.v.size());
    cp(recv_off, p.recv_off);
    cp(halo, p.halo);
    cp(send_off, p.send_off);
    cp(send_idx, p.send_idx);
    return 0;
}

int ibmgpu_distplan_free(ibmgpu_distplan_t d) {
    delete d;
    return 0;
}

int ibmgpu_partition_lambda(int nx, int ny, int n_b, const int* body_cell_j, int nranks, int* owner) {
    if (nranks < 1) return IBMGPU_EINVAL;
    const auto o = ibmhost::partition_lambda(nx, ny, n_b, body_cell_j, nranks);
    std::memcpy(owner, o.data(), sizeof(int) * o.size());
    return 0;
}

int ibmgpu_partition_coarse(int n_core, const int* agg, int n_agg, int tail, const int* owner_fine, int* owner_coarse) {
    if (n_core < 0 || n_agg < 0 || tail < 0) return IBMGPU_EINVAL;
    const std::vector<int> of(owner_fine, owner_fine + n_core + tail);
    const auto o = ibmhost::partition_coarse(of, agg, n_core, n_agg, tail);
    std::memcpy(owner_coarse, o.data(), sizeof(int) * o.size());
    return 0;
}

}  // extern "C"
