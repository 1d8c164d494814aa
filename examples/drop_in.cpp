// Drop-in example: the reference's call sequence (operators + solvers + Stepper), unchanged
// except for `using namespace ibm_b200` instead of `ibm`. Build:
//   g++ -std=c++20 -O2 -Iinclude examples/drop_in.cpp -Lpaper_1109_3524_b200 -libmgpu \
//       -Wl,-rpath,$PWD/paper_1109_3524_b200 -o build/drop_in
#include <cmath>
#include <cstdio>

#include "ibm_b200.hpp"

using namespace ibm_b200;

int main(int argc, char** argv) {
    // 2-D five-point Poisson (proj/tests/oracles.hpp poisson5), solved with SA-PCG
    const int n = 64;
    std::vector<Triplet> t;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            const int p = i + j * n;
            t.push_back({p, p, 4.0});
            if (i > 0) t.push_back({p, p - 1, -1.0});
            if (i < n - 1) t.push_back({p, p + 1, -1.0});
            if (j > 0) t.push_back({p, p - n, -1.0});
            if (j < n - 1) t.push_back({p, p + n, -1.0});
        }
    SparseMatrix A = SparseMatrix::from_triplets(n * n, n * n, t);
    std::vector<double> b(n * n);
    for (int i = 0; i < n * n; ++i) b[i] = std::sin(0.7 * i + 0.3);
    SaHierarchy h = build_sa_hierarchy(A);
    SolveResult r = pcg(A, b, {}, SaPreconditioner(h), SolverParams{});
    std::printf("poisson5(%d): pcg-sa %s in %d iterations, rel residual %.3e, levels %zu\n", n,
                r.converged() ? "converged" : "FAILED", r.iterations, r.rel_residual, h.level_count());
    if (!r.converged()) return 1;
    if (argc > 1) {
        Stepper st(argv[1]);
        for (int k = 0; k < 3; ++k) {
            StepReport rep = st.advance();
            const auto f = st.forces();
            std::printf("step %d ok=%d s1=%d s2=%d div=%.2e slip=%.2e cd=%.6f\n", k + 1, rep.ok, rep.solve1_iters,
                        rep.solve2_iters, rep.div_residual, rep.noslip_residual, f[2]);
            if (!rep.ok) return 1;
        }
        // io.hpp checkpoint round trip: a second stepper resumes from the file and stays identical
        write_checkpoint("/tmp/ibm_b200_drop_in.ckpt", st);
        Stepper resumed(argv[1]);
        read_checkpoint("/tmp/ibm_b200_drop_in.ckpt", resumed);
        const bool same = st.advance().ok && resumed.advance().ok && st.state().q == resumed.state().q;
        std::printf("checkpoint resume %s\n", same ? "bitwise identical" : "DIFFERS");
        if (!same) return 1;
    }
    try {
        SolverParams bad;
        bad.rel_tol = 2.0;
        pcg(A, b, {}, IdentityPreconditioner{}, bad);
        return 1;
    } catch (const std::invalid_argument&) {
        std::printf("invalid_argument surfaced as in the reference\n");
    }
    return 0;
}
