// refresh.cuh — incremental refresh_body_operators (refresh.cu).
#pragma once
#include "internal.cuh"

namespace ibmgpu {

// What a moving body never changes: G^T and the pinned pressure-pressure block of lhs2.
struct RefreshCache {
    Mat* GT = nullptr;   // n_p x n_q
    Mat* Lpp = nullptr;  // n_p rows of lhs2, columns < n_p
    int n_p = 0, pin = 0, n_order = 1;
    // false (and not ready) when B^N's pattern is not symmetric: then the full assembly runs
    bool init(Ctx* c, const Mat* G, const Mat* BN, const Mat* lhs2, int n_p, int pin, int n_order);
    bool ready() const { return GT && Lpp; }
    ~RefreshCache();
};

Mat* row_slice(Ctx* c, const Mat* A, int r0, int r1);
Mat* block_lt(Ctx* c, const Mat* A, int rows, int colmax);
Mat* vcat(Ctx* c, const Mat* A, const Mat* B);
Mat* triple_small(Ctx* c, const Mat* A, const Mat* B, const Mat* C);  // (A B) C, short rows
bool mat_equal(Ctx* c, const Mat* A, const Mat* B);  // structure + bitwise values (debug checks)

// Q, Q^T and lhs2 for new E (operators.hpp:408-417 + 381-392), bit-exact with coupled_system.
void coupled_refresh(Ctx* c, const RefreshCache& rc, const Mat* G, const Mat* E, const Mat* BN, Mat** Q, Mat** QT,
                     Mat** lhs2);

}  // namespace ibmgpu
