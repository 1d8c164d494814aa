// dist_plan.hpp — row-slab distribution of the solve-2 operators across ranks.
//
// Every rank holds the full operators and SA hierarchy (built redundantly and deterministically,
// so bit-identical on all ranks) and extracts, per distributed matrix, its owned rows with the
// column indices remapped to an *extended* local numbering:
//     [0, n_own)              owned entries of the input vector, in global order
//     [n_own, n_own + n_halo) remote entries, grouped by owning peer, ascending within a peer
// Entry order inside each row is the global column order, so a local thread-per-row SpMV sums in
// exactly the reference's order. The send lists are the transpose of the peers' halo lists and
// are computed locally (every rank sees the full matrix), so no plan exchange is needed.
#pragma once
#include <vector>

namespace ibmhost {

struct DistPlan {
    int rank = 0, nranks = 1;
    int rows_global = 0, cols_global = 0;
    std::vector<int> rows;         // owned output rows (global ids, ascending)
    int n_own = 0;                 // owned input entries
    std::vector<int> own;          // their global ids (ascending)
    std::vector<int> rp, ci;       // local CSR, ci in extended numbering
    std::vector<double> v;
    std::vector<int> recv_off;     // per peer: offset into the halo region (size nranks+1)
    std::vector<int> halo;         // halo global ids, grouped by peer
    std::vector<int> send_off;     // per peer: offset into send_idx (size nranks+1)
    std::vector<int> send_idx;     // owned-local indices to send, grouped by peer
    int n_halo() const { return static_cast<int>(halo.size()); }
};

// M (rows x cols CSR); row_owner[rows], col_owner[cols] in [0, nranks).
DistPlan make_dist_plan(int rows, int cols, const int* rp, const int* ci, const double* v, const int* row_owner,
                        const int* col_owner, int rank, int nranks);

// Row partition of the coupled system (n_p pressure cells, nx x ny, then 2 n_b force rows):
// pressure rows by balanced j-slabs, force rows k and n_b+k by the slab of body point k's cell.
std::vector<int> partition_lambda(int nx, int ny, int n_b, const int* body_cell_j, int nranks);

// Partition of level l+1 from level l: aggregate a is owned by the owner of its lowest-index
// member; tail (force) unknowns keep their owner (amg.hpp:166-178 identity tail).
std::vector<int> partition_coarse(const std::vector<int>& owner_l, const int* agg, int n_core, int n_agg, int tail);

}  // namespace ibmhost
