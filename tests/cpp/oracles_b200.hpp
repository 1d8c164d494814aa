// oracles_b200.hpp — test-only dense helpers for the drop-in acceptance driver, independent of the
// code under test (the reference keeps the same kind of helpers in proj/tests/oracles.hpp).
#pragma once
#include <algorithm>
#include <cmath>
#include <random>
#include <vector>

#include "ibm_b200.hpp"

namespace oracle {

using Dense = std::vector<std::vector<double>>;

inline Dense to_dense(const ibm_b200::SparseMatrix& A) {
    Dense d((size_t)A.rows(), std::vector<double>((size_t)A.cols(), 0.0));
    const auto& rp = A.row_ptr();
    const auto& ci = A.col_idx();
    const auto& v = A.values();
    for (int r = 0; r < A.rows(); ++r)
        for (int k = rp[(size_t)r]; k < rp[(size_t)r + 1]; ++k) d[(size_t)r][(size_t)ci[(size_t)k]] = v[(size_t)k];
    return d;
}

// Number of eigenvalues of the symmetric matrix a below sigma (Sylvester's law of inertia: the
// negative pivots of an LDL^T factorisation of a - sigma I).
inline int eigenvalues_below(Dense a, double sigma) {
    const size_t n = a.size();
    for (size_t i = 0; i < n; ++i) a[i][i] -= sigma;
    int neg = 0;
    for (size_t k = 0; k < n; ++k) {
        const double piv = a[k][k];
        if (piv < 0.0) ++neg;
        const double inv = piv != 0.0 ? 1.0 / piv : 0.0;
        for (size_t i = k + 1; i < n; ++i) {
            const double l = a[i][k] * inv;
            if (l == 0.0) continue;
            for (size_t j = k + 1; j <= i; ++j) a[i][j] -= l * a[j][k];
        }
        for (size_t i = k + 1; i < n; ++i) a[k][i] = a[i][k];
    }
    return neg;
}

// largest |eigenvalue| bound (Gershgorin)
inline double spectral_bound(const Dense& a) {
    double m = 0.0;
    for (const auto& row : a) {
        double s = 0.0;
        for (double x : row) s += std::fabs(x);
        m = std::max(m, s);
    }
    return m;
}

inline ibm_b200::SparseMatrix random_sparse(int rows, int cols, double fill, unsigned seed) {
    std::mt19937 gen(seed);
    std::uniform_real_distribution<double> coin(0.0, 1.0), value(-1.0, 1.0);
    std::vector<ibm_b200::Triplet> t;
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c)
            if (coin(gen) < fill) t.push_back({r, c, value(gen)});
    if (t.empty()) t.push_back({0, 0, 1.0});
    return ibm_b200::SparseMatrix::from_triplets(rows, cols, t);
}

}  // namespace oracle
