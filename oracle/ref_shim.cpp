// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the *unmodified* reference headers (/root/reference/proj/include),
// compiled by oracle/Makefile with the reference's own flags (-std=c++20 -O3 -fopenmp,
// no -march: proj/CMakeLists.txt:9). Output: oracle/_ref/libibmref.so.
//
// Nothing here re-implements the reference: every entry point forwards to the
// reference function named in its comment. Used by tests/ (parity oracle, golden
// fixture generation) and by bench.py's reference arm / cpu_baseline leg.
#include <omp.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ibm/runner.hpp"

using namespace ibm;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

SparseMatrix from_csr(int rows, int cols, const int* rp, const int* ci, const double* v) {
    const int nnz = rp[rows];
    return SparseMatrix(rows, cols, std::vector<int>(rp, rp + rows + 1), std::vector<int>(ci, ci + nnz),
                        std::vector<double>(v, v + nnz));
}

struct RefCase {
    CaseConfig cfg;
    StaggeredGrid grid;
    std::unique_ptr<Stepper> st;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { omp_set_num_threads(n); }
int ref_max_threads() { return omp_get_max_threads(); }

// ---- matrices (opaque SparseMatrix*) ----
void* ref_mat_from_csr(int rows, int cols, const int* rp, const int* ci, const double* v) {
    return new SparseMatrix(from_csr(rows, cols, rp, ci, v));
}
// sparse.hpp:36 from_triplets (sort, sum duplicates, drop zeros)
void* ref_mat_from_triplets(int rows, int cols, int n, const int* r, const int* c, const double* v) {
    SparseMatrix* out = nullptr;
    if (guarded([&] {
            std::vector<Triplet> t(static_cast<size_t>(n));
            for (int k = 0; k < n; ++k) t[static_cast<size_t>(k)] = {r[k], c[k], v[k]};
            out = new SparseMatrix(SparseMatrix::from_triplets(rows, cols, std::move(t)));
        }))
        return nullptr;
    return out;
}
void ref_mat_free(void* m) { delete static_cast<SparseMatrix*>(m); }
void ref_mat_info(const void* m, int* rows, int* cols, int* nnz) {
    auto* A = static_cast<const SparseMatrix*>(m);
    *rows = A->rows();
    *cols = A->cols();
    *nnz = A->nnz();
}
void ref_mat_copy(const void* m, int* rp, int* ci, double* v) {
    auto* A = static_cast<const SparseMatrix*>(m);
    std::memcpy(rp, A->row_ptr().data(), sizeof(int) * A->row_ptr().size());
    if (A->nnz()) {
        std::memcpy(ci, A->col_idx().data(), sizeof(int) * static_cast<size_t>(A->nnz()));
        std::memcpy(v, A->values().data(), sizeof(double) * static_cast<size_t>(A->nnz()));
    }
}
// sparse.hpp:101
void ref_spmv(const void* m, const double* x, double* y) { static_cast<const SparseMatrix*>(m)->spmv_into(x, y); }
// sparse.hpp:120
void* ref_transpose(const void* m) { return new SparseMatrix(static_cast<const SparseMatrix*>(m)->transpose()); }
// sparse.hpp:270
void* ref_spmm(const void* a, const void* b) {
    SparseMatrix* out = nullptr;
    if (guarded([&] { out = new SparseMatrix(spmm(*static_cast<const SparseMatrix*>(a), *static_cast<const SparseMatrix*>(b))); }))
        return nullptr;
    return out;
}
// sparse.hpp:282
void* ref_triple(const void* a, const void* b, const void* c, int slice, long long* peak, int* slices) {
    SparseMatrix* out = nullptr;
    if (guarded([&] {
            TripleProductStats st;
            out = new SparseMatrix(sliced_triple_product(*static_cast<const SparseMatrix*>(a),
                                                         *static_cast<const SparseMatrix*>(b),
                                                         *static_cast<const SparseMatrix*>(c), slice, &st));
            if (peak) *peak = static_cast<long long>(st.peak_slice_nnz);
            if (slices) *slices = st.slices;
        }))
        return nullptr;
    return out;
}
// sparse.hpp:317
void* ref_add(double a, const void* A, double b, const void* B) {
    SparseMatrix* out = nullptr;
    if (guarded([&] { out = new SparseMatrix(add_sparse(a, *static_cast<const SparseMatrix*>(A), b, *static_cast<const SparseMatrix*>(B))); }))
        return nullptr;
    return out;
}
// sparse.hpp:351
void* ref_symmetrized(const void* A) { return new SparseMatrix(symmetrized(*static_cast<const SparseMatrix*>(A))); }
// operators.hpp:381
void* ref_pin(const void* A, int pin) { return new SparseMatrix(pin_row_col(*static_cast<const SparseMatrix*>(A), pin)); }
// sparse.hpp:331
int ref_is_symmetric(const void* A, double tol) { return is_symmetric(*static_cast<const SparseMatrix*>(A), tol) ? 1 : 0; }

// ---- solvers ----
// krylov.hpp:70 pcg; kind 0 identity, 1 diagonal, 2 SA (hier required)
int ref_pcg(const void* A, const double* b, const double* x0, int kind, const void* hier, double rel_tol,
            int max_iters, double* x_out, int* iters, double* rel_res, int* status, double* history, int hist_cap,
            int* hist_len) {
    return guarded([&] {
        const auto& M = *static_cast<const SparseMatrix*>(A);
        const size_t n = static_cast<size_t>(M.rows());
        std::vector<double> bb(b, b + n), xx;
        if (x0) xx.assign(x0, x0 + n);
        SolverParams p;
        p.rel_tol = rel_tol;
        p.max_iters = max_iters;
        p.record_history = history != nullptr;
        SolveResult r;
        if (kind == 0) {
            r = pcg(M, bb, xx, IdentityPreconditioner{}, p);
        } else if (kind == 1) {
            r = pcg(M, bb, xx, DiagonalPreconditioner(M), p);
        } else {
            r = pcg(M, bb, xx, SaPreconditioner(*static_cast<const SaHierarchy*>(hier)), p);
        }
        std::memcpy(x_out, r.x.data(), sizeof(double) * n);
        *iters = r.iterations;
        *rel_res = r.rel_residual;
        *status = static_cast<int>(r.status);
        if (history) {
            const int m = std::min<int>(hist_cap, static_cast<int>(r.history.size()));
            std::memcpy(history, r.history.data(), sizeof(double) * static_cast<size_t>(m));
            *hist_len = static_cast<int>(r.history.size());
        }
    });
}

// amg.hpp:127
void* ref_sa_build(const void* A, double theta, int max_coarse, int max_levels, int power_its, int tail) {
    SaHierarchy* out = nullptr;
    if (guarded([&] {
            SaOptions o;
            o.theta = theta;
            o.max_coarse = max_coarse;
            o.max_levels = max_levels;
            o.power_iterations = power_its;
            o.keep_fine_tail = tail;
            out = new SaHierarchy(build_sa_hierarchy(*static_cast<const SparseMatrix*>(A), o));
        }))
        return nullptr;
    return out;
}
void ref_sa_free(void* h) { delete static_cast<SaHierarchy*>(h); }
int ref_sa_levels(const void* h, int* stalled) {
    auto* H = static_cast<const SaHierarchy*>(h);
    if (stalled) *stalled = H->coarsening_stalled ? 1 : 0;
    return static_cast<int>(H->levels.size());
}
// borrowed pointers into the hierarchy: which 0 = A, 1 = P, 2 = Pt; lev == n_levels -> coarse_A
const void* ref_sa_level_mat(const void* h, int lev, int which, double* omega) {
    auto* H = static_cast<const SaHierarchy*>(h);
    if (lev == static_cast<int>(H->levels.size())) return &H->coarse_A;
    const SaLevel& L = H->levels[static_cast<size_t>(lev)];
    if (omega) *omega = L.omega;
    return which == 0 ? &L.A : which == 1 ? &L.P : &L.Pt;
}
// amg.hpp:231
void ref_sa_apply(const void* h, const double* r, int n, double* z) {
    std::vector<double> rr(r, r + n);
    auto zz = sa_apply(*static_cast<const SaHierarchy*>(h), rr);
    std::memcpy(z, zz.data(), sizeof(double) * static_cast<size_t>(n));
}
// amg.hpp:250
int ref_amg_solve(const void* A, const void* h, const double* b, double rel_tol, int max_iters, double* x_out,
                  int* iters, double* rel_res, int* status) {
    return guarded([&] {
        const auto& M = *static_cast<const SparseMatrix*>(A);
        const size_t n = static_cast<size_t>(M.rows());
        SolverParams p;
        p.rel_tol = rel_tol;
        p.max_iters = max_iters;
        auto r = amg_solve(M, *static_cast<const SaHierarchy*>(h), std::vector<double>(b, b + n), {}, p);
        std::memcpy(x_out, r.x.data(), sizeof(double) * n);
        *iters = r.iterations;
        *rel_res = r.rel_residual;
        *status = static_cast<int>(r.status);
    });
}
// amg.hpp:110 + :79 (strength graph on the core block, then greedy aggregation)
int ref_aggregate(const void* A, double theta, int n_core, int* agg) {
    SparseMatrix S = sa_detail::strength_graph(*static_cast<const SparseMatrix*>(A), theta, n_core);
    std::vector<int> a;
    const int n = sa_detail::aggregate(S, a);
    std::memcpy(agg, a.data(), sizeof(int) * a.size());
    return n;
}
void* ref_strength(const void* A, double theta, int n_core) {
    return new SparseMatrix(sa_detail::strength_graph(*static_cast<const SparseMatrix*>(A), theta, n_core));
}
// amg.hpp:58
double ref_rho(const void* A, int iters) {
    const auto& M = *static_cast<const SparseMatrix*>(A);
    auto d = M.diagonal_vector();
    for (double& x : d) x = 1.0 / x;
    return sa_detail::rho_dinv_a(M, d, iters);
}
// body.hpp:19
double ref_delta_roma(double r, double h) { return delta_roma(r, h); }

// ---- cases (config.hpp:236 parse_config, grid.hpp:134, stepper.hpp:171) ----
void* ref_case_open(const char* cfg_path, double h_min_override, double dt_override) {
    RefCase* rc = nullptr;
    if (guarded([&] {
            auto c = std::make_unique<RefCase>();
            c->cfg = parse_config(cfg_path);
            if (h_min_override > 0.0) c->cfg.h_min = h_min_override;
            if (dt_override > 0.0) c->cfg.dt = dt_override;
            c->grid = build_stretched_grid(c->cfg.domain, c->cfg.uniform, c->cfg.h_min, c->cfg.ratio);
            c->st = std::make_unique<Stepper>(c->grid, build_bodies(c->cfg), c->cfg.bc, c->cfg.nu,
                                              stepping_from(c->cfg), c->cfg.u0, c->cfg.v0);
            rc = c.release();
        }))
        return nullptr;
    return rc;
}
void ref_case_free(void* h) { delete static_cast<RefCase*>(h); }
void ref_case_dims(const void* h, int* out) {
    auto* c = static_cast<const RefCase*>(h);
    const auto& g = c->grid;
    out[0] = g.nx;
    out[1] = g.ny;
    out[2] = g.n_q();
    out[3] = g.n_p();
    out[4] = c->st->ops().n_b;
    out[5] = c->st->ops().n_lambda();
    out[6] = static_cast<int>(c->st->hierarchy().levels.size());
}
void ref_case_scalars(const void* h, double* out) {
    auto* c = static_cast<const RefCase*>(h);
    out[0] = c->cfg.dt;
    out[1] = c->cfg.nu;
    out[2] = c->grid.h_min;
    out[3] = c->cfg.u_inf;
    out[4] = c->cfg.ref_length;
}
// borrowed operator matrix by name
const void* ref_case_op(const void* h, const char* name) {
    const OperatorSet& o = static_cast<const RefCase*>(h)->st->ops();
    const std::string n(name);
    if (n == "L") return &o.L;
    if (n == "G") return &o.G;
    if (n == "E") return &o.E;
    if (n == "H") return &o.H;
    if (n == "A") return &o.A;
    if (n == "BN") return &o.BN;
    if (n == "Q") return &o.Q;
    if (n == "QT") return &o.QT;
    if (n == "lhs2") return &o.lhs2;
    return nullptr;
}
const void* ref_case_hier(const void* h) { return &static_cast<const RefCase*>(h)->st->hierarchy(); }
// grid arrays: which 0 x_faces,1 y_faces,2 dx,3 dy,4 x_c,5 y_c,6 del_x,7 del_y
int ref_case_grid(const void* h, int which, double* out) {
    const auto& g = static_cast<const RefCase*>(h)->grid;
    const std::vector<double>* v[] = {&g.x_faces, &g.y_faces, &g.dx, &g.dy, &g.x_c, &g.y_c, &g.del_x, &g.del_y};
    if (out) std::memcpy(out, v[which]->data(), sizeof(double) * v[which]->size());
    return static_cast<int>(v[which]->size());
}
void ref_case_uniform(const void* h, double* out) {
    const auto& g = static_cast<const RefCase*>(h)->grid;
    out[0] = g.uniform_region.x0;
    out[1] = g.uniform_region.x1;
    out[2] = g.uniform_region.y0;
    out[3] = g.uniform_region.y1;
}
// body points at the current state time: x, y, ub_x, ub_y, ds per point
void ref_case_bodies(const void* h, double* px, double* py, double* ubx, double* uby, double* ds) {
    int k = 0;
    for (const auto& b : static_cast<const RefCase*>(h)->st->bodies())
        for (int p = 0; p < b.n(); ++p, ++k) {
            px[k] = b.x[static_cast<size_t>(p)];
            py[k] = b.y[static_cast<size_t>(p)];
            ubx[k] = b.ub_x[static_cast<size_t>(p)];
            uby[k] = b.ub_y[static_cast<size_t>(p)];
            ds[k] = b.ds;
        }
}
// stepper.hpp:231 advance. rep: [ok, s1_it, s2_it, s1_res, s2_res, div, slip, rebuilt_h, rebuilt_ops,
//   t_assembly, t_precond, t_explicit, t_solve1, t_solve2, t_projection]
int ref_case_step(void* h, double* rep, char* msg, int msg_cap) {
    auto* c = static_cast<RefCase*>(h);
    StepReport r = c->st->advance();
    const double v[] = {r.ok ? 1.0 : 0.0, double(r.solve1_iters), double(r.solve2_iters), r.solve1_res, r.solve2_res,
                        r.div_residual, r.noslip_residual, r.rebuilt_hierarchy ? 1.0 : 0.0,
                        r.rebuilt_operators ? 1.0 : 0.0, r.t_assembly, r.t_precond, r.t_explicit, r.t_solve1,
                        r.t_solve2, r.t_projection};
    std::memcpy(rep, v, sizeof(v));
    if (msg && msg_cap > 0) {
        std::strncpy(msg, r.message.c_str(), static_cast<size_t>(msg_cap) - 1);
        msg[msg_cap - 1] = 0;
    }
    return r.ok ? 0 : 1;
}
// state vectors: which 0 q, 1 lambda, 2 conv_prev; returns length
int ref_case_state(const void* h, int which, double* out) {
    const FlowState& s = static_cast<const RefCase*>(h)->st->state();
    const std::vector<double>* v = which == 0 ? &s.q : which == 1 ? &s.lambda : &s.conv_prev;
    if (out) std::memcpy(out, v->data(), sizeof(double) * v->size());
    return static_cast<int>(v->size());
}
double ref_case_time(const void* h) { return static_cast<const RefCase*>(h)->st->state().t; }
// diagnostics.hpp:26 on the current f_tilde: out [fx, fy, cd, cl]
void ref_case_forces(const void* h, double* out) {
    auto* c = static_cast<const RefCase*>(h);
    auto f = compute_force_coefficients(c->st->state().f_tilde, c->st->ops().n_b, c->st->state().t, c->cfg.u_inf,
                                        c->cfg.ref_length);
    out[0] = f.fx;
    out[1] = f.fy;
    out[2] = f.cd;
    out[3] = f.cl;
}
// boundary arrays in BoundaryState order (boundary.hpp:37-40); returns total length written
int ref_case_boundary(const void* h, double* out) {
    const BoundaryState& b = static_cast<const RefCase*>(h)->st->boundary();
    size_t k = 0;
    for (const auto* v : {&b.left_u, &b.right_u, &b.left_v, &b.right_v, &b.bottom_v, &b.top_v, &b.bottom_u, &b.top_u}) {
        if (out) std::memcpy(out + k, v->data(), sizeof(double) * v->size());
        k += v->size();
    }
    return static_cast<int>(k);
}

// operators.hpp:27-33 BcCoupling list as (row, slot, idx, coeff) quadruples; returns the count
int ref_case_visc_bc(const void* h, double* out) {
    const auto& v = static_cast<const RefCase*>(h)->st->ops().visc_bc;
    if (out)
        for (size_t k = 0; k < v.size(); ++k) {
            out[4 * k] = v[k].row;
            out[4 * k + 1] = static_cast<double>(v[k].slot);
            out[4 * k + 2] = v[k].idx;
            out[4 * k + 3] = v[k].coeff;
        }
    return static_cast<int>(v.size());
}

// io.hpp:89-145 checkpoints (text, %.17g): 0 on success
int ref_case_write_checkpoint(const void* h, const char* path) {
    try {
        write_checkpoint(path, *static_cast<const RefCase*>(h)->st);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
int ref_case_read_checkpoint(void* h, const char* path) {
    try {
        read_checkpoint(path, *static_cast<RefCase*>(h)->st);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"
