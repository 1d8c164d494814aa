// acceptance_b200.cpp — the reference acceptance suite's structural criteria 5, 7, 8 and 9
// (proj/tests/acceptance/acceptance.cpp:216-410), driven through the drop-in shim: the same
// library calls in the same order as the reference's driver, with `#include "ibm_b200.hpp"` and
// `using namespace ibm_b200` in place of the reference headers and `using namespace ibm`. Plus
// the extension points the reference exposes: a user Preconditioner subclass, spmv_into on host
// pointers and the public SaHierarchy levels. Prints one PASS/FAIL line per criterion; exit code 0
// iff all pass.
//   build: g++ -std=c++20 -O2 -Iinclude tests/cpp/acceptance_b200.cpp -Lpaper_1109_3524_b200 -libmgpu
//   run:   acceptance_b200 <cases dir>
#include <cstdarg>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "ibm_b200.hpp"
#include "oracles_b200.hpp"

using namespace ibm_b200;

namespace {

std::string g_cases = "cases";

struct Outcome {
    bool pass = true;
    std::string detail;
};

std::string fmt(const char* f, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, f);
    std::vsnprintf(buf, sizeof buf, f, ap);
    va_end(ap);
    return buf;
}

void expect(Outcome& o, bool ok, const std::string& what) {
    if (ok) return;
    o.pass = false;
    o.detail += (o.detail.empty() ? "" : "; ") + what + " FAILED";
}

// criterion 5: step invariants, coupled-matrix symmetry, one zero eigenvalue before pinning
Outcome step_invariants_and_symmetry() {
    Outcome o;
    {
        CaseConfig c = parse_config(g_cases + "/couette.cfg");
        c.n_steps = 50;
        StaggeredGrid g = build_stretched_grid(c.domain, c.uniform, c.h_min, c.ratio);
        Stepper st(g, build_bodies(c), c.bc, c.nu, stepping_from(c));
        double worst_div = 0.0, worst_slip = 0.0;
        for (int k = 0; k < c.n_steps; ++k) {
            const StepReport rep = st.advance();
            expect(o, rep.ok, fmt("couette step %d", k));
            worst_div = std::max(worst_div, rep.div_residual);
            worst_slip = std::max(worst_slip, rep.noslip_residual);
        }
        o.detail = fmt("max divergence residual %.2e, max no-slip residual %.2e", worst_div, worst_slip);
        expect(o, worst_div <= 10.0 * c.solve2.params.rel_tol, "divergence residual <= 10 rel_tol");
        expect(o, worst_slip <= 10.0 * c.solve2.params.rel_tol, "no-slip residual <= 10 rel_tol");
    }
    {
        StaggeredGrid g = build_uniform_grid(Rect{-3.0, 3.0, -3.0, 3.0}, 0.1);
        LagrangianBody body = discretize_circle(0.0, 0.0, 1.0, 0.1);
        for (int order : {1, 3}) {
            OperatorSet ops = assemble_operators(g, {body}, 0.05, 0.025, order);
            expect(o, is_symmetric(ops.lhs2, 1e-12), fmt("lhs2 symmetric to 1e-12 (N=%d)", order));
        }
    }
    for (bool with_body : {true, false}) {
        StaggeredGrid g = build_uniform_grid(Rect{-0.6, 0.6, -0.6, 0.6}, 0.1);
        std::vector<LagrangianBody> bodies;
        if (with_body) bodies.push_back(discretize_circle(0.0, 0.0, 0.3, 0.1));
        OperatorSet ops = assemble_operators(g, bodies, 0.05, 0.02, 1);
        SparseMatrix raw = symmetrized(sliced_triple_product(ops.QT, ops.BN, ops.Q, ops.QT.rows()));
        const oracle::Dense d = oracle::to_dense(raw);
        const double tol = 1e-10 * oracle::spectral_bound(d);
        const int zeros = oracle::eigenvalues_below(d, tol) - oracle::eigenvalues_below(d, -tol);
        expect(o, zeros == 1, fmt("pre-pinning zero eigenvalues = 1 (%s body), got %d", with_body ? "with" : "no", zeros));
    }
    return o;
}

// criterion 7: sliced triple product against two plain products, and the slicing's peak bound
Outcome sliced_triple_product_oracle() {
    Outcome o;
    std::mt19937 rng(20240811);
    std::uniform_int_distribution<int> dim(5, 40);
    int compared = 0;
    double worst = 0.0;
    for (int trial = 0; trial < 50; ++trial) {
        const int m = dim(rng), k = dim(rng), l = dim(rng), n = dim(rng);
        SparseMatrix A = oracle::random_sparse(m, k, 0.25, 1000 + trial);
        SparseMatrix B = oracle::random_sparse(k, l, 0.25, 2000 + trial);
        SparseMatrix C = oracle::random_sparse(l, n, 0.25, 3000 + trial);
        SparseMatrix two_step = spmm(spmm(A, B), C);
        for (int slice : {1, 7, m}) {
            SparseMatrix D = sliced_triple_product(A, B, C, slice);
            const bool same = D.row_ptr() == two_step.row_ptr() && D.col_idx() == two_step.col_idx();
            expect(o, same, fmt("trial %d slice %d pattern", trial, slice));
            if (!same) continue;
            for (int e = 0; e < D.nnz(); ++e) {
                const double r = two_step.values()[(size_t)e];
                worst = std::max(worst, std::fabs(D.values()[(size_t)e] - r) / std::max(1.0, std::fabs(r)));
            }
            ++compared;
        }
    }
    expect(o, worst <= 1e-13, "entrywise relative agreement 1e-13");
    StaggeredGrid g = build_uniform_grid(Rect{-2.0, 2.0, -2.0, 2.0}, 0.1);
    LagrangianBody body = discretize_circle(0.0, 0.0, 1.0, 0.1);
    OperatorSet ops = assemble_operators(g, {body}, 0.05, 0.02, 1);
    TripleProductStats whole{}, eighth{};
    sliced_triple_product(ops.QT, ops.BN, ops.Q, ops.QT.rows(), &whole);
    sliced_triple_product(ops.QT, ops.BN, ops.Q, ops.QT.rows() / 8, &eighth);
    o.detail = fmt("%d sliced products vs two-step (worst rel diff %.2e); peak intermediate %zu < %zu", compared, worst,
                   eighth.peak_slice_nnz, whole.peak_slice_nnz);
    expect(o, eighth.peak_slice_nnz < whole.peak_slice_nnz, "peak intermediate strictly below full");
    return o;
}

// criterion 8: solver ordering on the 60x60 cylinder matrix
Outcome solver_ordering() {
    Outcome o;
    const Rect dom{-3.0, 3.0, -3.0, 3.0}, uni{-0.6, 0.6, -0.6, 0.6};
    const double ratio[4] = {1.17, 1.17, 1.17, 1.17};
    StaggeredGrid g = build_stretched_grid(dom, uni, 0.04, ratio);
    expect(o, g.nx == 60 && g.ny == 60, fmt("grid is 60x60 (got %dx%d)", g.nx, g.ny));
    LagrangianBody body = discretize_circle(0.0, 0.0, 1.0, 0.04);
    OperatorSet ops = assemble_operators(g, {body}, 0.02, 0.025, 1);
    SolverParams p;
    p.rel_tol = 1e-5;
    p.max_iters = 20000;
    SaOptions sa;
    sa.keep_fine_tail = 2 * ops.n_b;
    const std::vector<BenchRow> rows = solver_bench_matrix(ops.lhs2, 0, p, sa);
    print_bench(rows, stderr);
    int it_cg = 0, it_diag = 0, it_sa = 0;
    for (const auto& r : rows) {
        expect(o, r.converged, r.name + " converged to 1e-5");
        if (r.name == "cg") it_cg = r.iterations;
        if (r.name == "pcg-diag") it_diag = r.iterations;
        if (r.name == "pcg-sa") it_sa = r.iterations;
    }
    o.detail = fmt("iterations: pcg-sa %d < pcg-diag %d < cg %d (dim %d)", it_sa, it_diag, it_cg, ops.lhs2.rows());
    expect(o, it_sa < it_diag && it_diag < it_cg, "iteration ordering pcg-sa < pcg-diag < cg");
    return o;
}

// criterion 9: hierarchy reuse (n_pc 1/2/4) changes forces by less than 10 rel_tol; n_pc = 1 is
// field-identical to rebuilding every step
Outcome hierarchy_reuse() {
    Outcome o;
    CaseConfig base = parse_config(g_cases + "/flapping_smoke.cfg");
    base.n_steps = 50;
    struct Series {
        std::vector<double> fx, fy, q;
        long iters = 0;
    };
    auto run = [&](int n_pc, bool force_rebuild) {
        CaseConfig c = base;
        c.n_pc = n_pc;
        StaggeredGrid g = build_stretched_grid(c.domain, c.uniform, c.h_min, c.ratio);
        SteppingParams sp = stepping_from(c);
        sp.force_rebuild = force_rebuild;
        Stepper st(g, build_bodies(c), c.bc, c.nu, sp);
        Series s;
        for (int k = 0; k < c.n_steps; ++k) {
            const StepReport rep = st.advance();
            if (!rep.ok) throw std::runtime_error("flapping smoke: " + rep.message);
            const ForceRecord f = compute_force_coefficients(st.state().f_tilde, st.ops().n_b, st.state().t, 1.0, 1.0);
            s.fx.push_back(f.fx);
            s.fy.push_back(f.fy);
            s.iters += rep.solve2_iters;
        }
        s.q = st.state().q;
        return s;
    };
    const Series s1 = run(1, false), s2 = run(2, false), s4 = run(4, false), always = run(1, true);
    expect(o, s1.q == always.q, "n_pc=1 field-identical to the always-rebuild path");
    double scale = 1.0;
    for (double v : s1.fx) scale = std::max(scale, std::fabs(v));
    for (double v : s1.fy) scale = std::max(scale, std::fabs(v));
    const double tol = 10.0 * base.solve2.params.rel_tol * scale;
    double worst = 0.0;
    for (size_t k = 0; k < s1.fx.size(); ++k)
        for (const Series* s : {&s2, &s4})
            worst = std::max({worst, std::fabs(s->fx[k] - s1.fx[k]), std::fabs(s->fy[k] - s1.fy[k])});
    o.detail = fmt("force series n_pc {1,2,4}: worst pointwise diff %.3e (tol %.3e); solve-2 iterations %ld/%ld/%ld",
                   worst, tol, s1.iters, s2.iters, s4.iters);
    expect(o, worst <= tol, "force series agree within 10 rel_tol");
    expect(o, s2.iters >= s1.iters && s4.iters >= s1.iters, "stale hierarchies never cost fewer iterations");
    return o;
}

// the reference's extension points: a user Preconditioner subclass (krylov.hpp:39-43), spmv_into
// on host pointers (sparse.hpp:101), SaHierarchy's public levels (amg.hpp:41-52)
class UserJacobi final : public Preconditioner {
public:
    explicit UserJacobi(const SparseMatrix& A) : d_(A.diagonal_vector()) {}
    void apply(const std::vector<double>& r, std::vector<double>& z) const override {
        ++calls;
        z.resize(r.size());
        for (size_t i = 0; i < r.size(); ++i) z[i] = r[i] / d_[i];
    }
    mutable int calls = 0;

private:
    std::vector<double> d_;
};

Outcome extension_points() {
    Outcome o;
    StaggeredGrid g = build_uniform_grid(Rect{-2.0, 2.0, -2.0, 2.0}, 0.05);
    LagrangianBody body = discretize_circle(0.0, 0.0, 1.0, 0.05);
    OperatorSet ops = assemble_operators(g, {body}, 0.02, 0.02, 1);
    const SparseMatrix& A = ops.lhs2;
    std::vector<double> w((size_t)A.rows());
    for (size_t i = 0; i < w.size(); ++i) w[i] = std::sin(0.3 * (double)i);
    std::vector<double> b((size_t)A.rows());
    A.spmv_into(w.data(), b.data());  // host pointers, as the reference's signature
    const std::vector<double> b2 = A.spmv(w);
    expect(o, b == b2, "spmv_into(host) == spmv");
    SolverParams p;
    UserJacobi user(A);
    const SolveResult ru = pcg(A, b, {}, user, p);
    const SolveResult rd = pcg(A, b, {}, DiagonalPreconditioner(A), p);
    double dx = 0.0, xm = 0.0;
    for (size_t i = 0; i < w.size(); ++i) {
        dx = std::max(dx, std::fabs(ru.x[i] - rd.x[i]));
        xm = std::max(xm, std::fabs(rd.x[i]));
    }
    expect(o, ru.converged() && std::abs(ru.iterations - rd.iterations) <= 2, "user preconditioner converges like diag");
    expect(o, user.calls == ru.iterations + 1 || user.calls == ru.iterations, "user apply called once per iteration");
    expect(o, dx <= 1e-6 * xm, "user-preconditioned solution within 1e-6");
    SaOptions sa;
    sa.keep_fine_tail = 2 * ops.n_b;
    const SaHierarchy h = build_sa_hierarchy(A, sa);
    expect(o, !h.levels.empty() && h.levels[0].A.rows() == A.rows() && h.levels[0].omega > 0.0 &&
                  h.levels[0].P.rows() == A.rows() && h.levels[0].Pt.cols() == A.rows() &&
                  (int)h.levels[0].inv_diag.size() == A.rows(),
           "hierarchy levels readable");
    expect(o, h.coarse_A.rows() > 0 && h.finest_size() == A.rows(), "coarse_A and finest_size");
    const SolveResult rs = pcg(A, b, {}, SaPreconditioner(h), p);
    o.detail = fmt("user Jacobi %d its (%d applies) vs device diag %d; |dx| %.1e; SA levels %zu, coarse %d, pcg-sa %d its",
                   ru.iterations, user.calls, rd.iterations, dx, h.level_count(), h.coarse_A.rows(), rs.iterations);
    expect(o, rs.converged() && rs.iterations < rd.iterations, "pcg-sa beats pcg-diag");
    return o;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc > 1) g_cases = argv[1];
    struct Item {
        const char* id;
        Outcome (*f)();
    };
    const Item items[] = {{"5", step_invariants_and_symmetry},
                          {"7", sliced_triple_product_oracle},
                          {"8", solver_ordering},
                          {"9", hierarchy_reuse},
                          {"x", extension_points}};
    int failed = 0;
    for (const auto& it : items) {
        Outcome o;
        try {
            o = it.f();
        } catch (const std::exception& e) {
            o.pass = false;
            o.detail = std::string("exception: ") + e.what();
        }
        std::printf("%s criterion %s: %s\n", o.pass ? "PASS" : "FAIL", it.id, o.detail.c_str());
        std::fflush(stdout);
        failed += !o.pass;
    }
    return failed ? 1 : 0;
}
