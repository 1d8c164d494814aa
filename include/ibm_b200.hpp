// ibm_b200.hpp — header-only C++ shim that re-exposes the reference's operator interface
// (/root/reference/proj/include/ibm/{sparse,krylov,amg,operators,stepper}.hpp) on top of the
// B200 C ABI (ibmgpu.h). A caller of `ibm::SparseMatrix`, `ibm::pcg`, `ibm::build_sa_hierarchy`
// or `ibm::Stepper` switches by including this header and using namespace `ibm_b200`: same
// names, same argument meaning, same exception types (std::invalid_argument for bad
// arguments, std::runtime_error otherwise). Host std::vector in and out, exactly as the
// reference's value semantics; the device keeps its own copies.
#pragma once
#include <cstdio>
#include <fstream>
#include <memory>
#include <type_traits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ibmgpu.h"

namespace ibm_b200 {

class Context {
public:
    explicit Context(int device = 0) {
        ibmgpu_ctx_t c = nullptr;
        check(ibmgpu_init(device, 1, 0, nullptr, &c), nullptr);
        h_.reset(c);
    }
    static Context& get() {
        static Context ctx(0);
        return ctx;
    }
    ibmgpu_ctx_t h() const { return h_.get(); }
    static void check(int rc, ibmgpu_ctx_t c) {
        if (rc == IBMGPU_OK) return;
        const std::string msg = ibmgpu_last_error(c);
        if (rc == IBMGPU_EINVAL) throw std::invalid_argument(msg);
        throw std::runtime_error(msg);
    }

private:
    struct Del {
        void operator()(ibmgpu_ctx_t c) const { ibmgpu_destroy(c); }
    };
    std::unique_ptr<std::remove_pointer_t<ibmgpu_ctx_t>, Del> h_;
};

inline void check(int rc) { Context::check(rc, Context::get().h()); }

// Device buffer used for host<->device staging of std::vector arguments.
class DeviceVector {
public:
    explicit DeviceVector(size_t n) : n_(n) { check(ibmgpu_vec_alloc(Context::get().h(), n, &p_)); }
    explicit DeviceVector(const std::vector<double>& v) : DeviceVector(v.size()) { upload(v); }
    ~DeviceVector() { ibmgpu_vec_free(Context::get().h(), p_); }
    DeviceVector(const DeviceVector&) = delete;
    DeviceVector& operator=(const DeviceVector&) = delete;
    void upload(const std::vector<double>& v) { check(ibmgpu_h2d(Context::get().h(), p_, v.data(), v.size())); }
    std::vector<double> download() const {
        std::vector<double> out(n_);
        check(ibmgpu_d2h(Context::get().h(), out.data(), p_, n_));
        return out;
    }
    double* get() const { return p_; }

private:
    double* p_ = nullptr;
    size_t n_;
};

struct Triplet {
    int row;
    int col;
    double value;
};

// sparse.hpp:27-222
class SparseMatrix {
public:
    SparseMatrix() = default;
    SparseMatrix(int rows, int cols, const std::vector<int>& row_ptr, const std::vector<int>& col_idx,
                 const std::vector<double>& values) {
        ibmgpu_mat_t m = nullptr;
        check(ibmgpu_csr_upload(Context::get().h(), rows, cols, (int)col_idx.size(), row_ptr.data(), col_idx.data(),
                                values.data(), &m));
        adopt(m, true);
    }
    static SparseMatrix from_triplets(int rows, int cols, const std::vector<Triplet>& t) {
        std::vector<int> r(t.size()), c(t.size());
        std::vector<double> v(t.size());
        for (size_t k = 0; k < t.size(); ++k) r[k] = t[k].row, c[k] = t[k].col, v[k] = t[k].value;
        ibmgpu_mat_t m = nullptr;
        check(ibmgpu_csr_from_triplets(Context::get().h(), rows, cols, (int)t.size(), r.data(), c.data(), v.data(), &m));
        SparseMatrix out;
        out.adopt(m, true);
        return out;
    }
    static SparseMatrix borrowed(ibmgpu_mat_t m) {
        SparseMatrix out;
        out.adopt(m, false);
        return out;
    }
    int rows() const { return rows_; }
    int cols() const { return cols_; }
    int nnz() const { return nnz_; }
    ibmgpu_mat_t handle() const { return h_.get(); }

    std::vector<int> row_ptr() const { return download().rp; }
    std::vector<int> col_idx() const { return download().ci; }
    std::vector<double> values() const { return download().v; }

    // sparse.hpp:101 — device pointers
    void spmv_into(const double* x_dev, double* y_dev) const {
        check(ibmgpu_spmv(Context::get().h(), handle(), x_dev, y_dev));
    }
    // sparse.hpp:112
    std::vector<double> spmv(const std::vector<double>& x) const {
        if ((int)x.size() != cols_) throw std::invalid_argument("spmv: dimension mismatch");
        std::vector<double> y(rows_);
        check(ibmgpu_spmv_host(Context::get().h(), handle(), x.data(), y.data()));
        return y;
    }
    SparseMatrix transpose() const { return make([&](ibmgpu_mat_t* o) { return ibmgpu_transpose(ctx(), handle(), o); }); }
    SparseMatrix scaled(double a) const {
        return make([&](ibmgpu_mat_t* o) { return ibmgpu_scale(ctx(), handle(), 0, a, nullptr, o); });
    }
    SparseMatrix scaled_rows(const std::vector<double>& d) const {
        return make([&](ibmgpu_mat_t* o) { return ibmgpu_scale(ctx(), handle(), 1, 0.0, d.data(), o); });
    }
    SparseMatrix scaled_cols(const std::vector<double>& d) const {
        return make([&](ibmgpu_mat_t* o) { return ibmgpu_scale(ctx(), handle(), 2, 0.0, d.data(), o); });
    }

    template <class F>
    static SparseMatrix make(F&& f) {
        ibmgpu_mat_t m = nullptr;
        check(f(&m));
        SparseMatrix out;
        out.adopt(m, true);
        return out;
    }

private:
    struct Host {
        std::vector<int> rp, ci;
        std::vector<double> v;
    };
    Host download() const {
        Host h{std::vector<int>(rows_ + 1), std::vector<int>(nnz_), std::vector<double>(nnz_)};
        check(ibmgpu_csr_download(ctx(), handle(), h.rp.data(), h.ci.data(), h.v.data()));
        return h;
    }
    static ibmgpu_ctx_t ctx() { return Context::get().h(); }
    void adopt(ibmgpu_mat_t m, bool owned) {
        h_ = std::shared_ptr<ibmgpu_mat>(m, [owned](ibmgpu_mat_t p) {
            if (owned) ibmgpu_csr_destroy(Context::get().h(), p);
        });
        ibmgpu_csr_info(m, &rows_, &cols_, &nnz_);
    }
    std::shared_ptr<ibmgpu_mat> h_;
    int rows_ = 0, cols_ = 0, nnz_ = 0;
};

inline SparseMatrix spmm(const SparseMatrix& A, const SparseMatrix& B) {
    return SparseMatrix::make([&](ibmgpu_mat_t* o) { return ibmgpu_spmm(Context::get().h(), A.handle(), B.handle(), o); });
}
struct TripleProductStats {
    size_t peak_slice_nnz = 0;
    int slices = 0;
};
inline SparseMatrix sliced_triple_product(const SparseMatrix& A, const SparseMatrix& B, const SparseMatrix& C,
                                          int max_slice_rows, TripleProductStats* stats = nullptr) {
    long long peak = 0;
    int slices = 0;
    auto out = SparseMatrix::make([&](ibmgpu_mat_t* o) {
        return ibmgpu_triple_product(Context::get().h(), A.handle(), B.handle(), C.handle(), max_slice_rows, o, &peak,
                                     &slices);
    });
    if (stats) *stats = TripleProductStats{(size_t)peak, slices};
    return out;
}
inline SparseMatrix add_sparse(double a, const SparseMatrix& A, double b, const SparseMatrix& B) {
    return SparseMatrix::make(
        [&](ibmgpu_mat_t* o) { return ibmgpu_add(Context::get().h(), a, A.handle(), b, B.handle(), o); });
}
inline SparseMatrix symmetrized(const SparseMatrix& A) {
    return SparseMatrix::make([&](ibmgpu_mat_t* o) { return ibmgpu_symmetrized(Context::get().h(), A.handle(), o); });
}
inline SparseMatrix pin_row_col(const SparseMatrix& A, int pin) {
    return SparseMatrix::make([&](ibmgpu_mat_t* o) { return ibmgpu_pin(Context::get().h(), A.handle(), pin, o); });
}
inline bool is_symmetric(const SparseMatrix& A, double tol) {
    int r = 0;
    check(ibmgpu_is_symmetric(Context::get().h(), A.handle(), tol, &r));
    return r != 0;
}

// krylov.hpp:15-37
struct SolverParams {
    double rel_tol = 1e-5;
    int max_iters = 2000;
    bool record_history = false;
    bool check_symmetry = false;
    void validate() const {
        if (!(rel_tol > 0.0 && rel_tol < 1.0)) throw std::invalid_argument("solver: rel_tol must be in (0,1)");
        if (max_iters < 1) throw std::invalid_argument("solver: max_iters must be >= 1");
    }
};
enum class SolveStatus { converged, max_iterations, breakdown };
struct SolveResult {
    std::vector<double> x;
    int iterations = 0;
    double rel_residual = 0.0;
    SolveStatus status = SolveStatus::converged;
    std::vector<double> history;
    bool converged() const { return status == SolveStatus::converged; }
};

// amg.hpp:21-52
struct SaOptions {
    double theta = 0.25;
    int max_coarse = 64;
    int max_levels = 25;
    int power_iterations = 10;
    int keep_fine_tail = 0;
};
class SaHierarchy {
public:
    SaHierarchy() = default;
    explicit SaHierarchy(ibmgpu_hier_t h, bool owned = true)
        : h_(h, [owned](ibmgpu_hier_t p) {
              if (owned) ibmgpu_sa_destroy(Context::get().h(), p);
          }) {}
    ibmgpu_hier_t handle() const { return h_.get(); }
    size_t level_count() const {
        int n = 0;
        ibmgpu_hier_info(handle(), &n, nullptr, nullptr);
        return (size_t)n + 1;
    }
    bool coarsening_stalled() const {
        int s = 0;
        ibmgpu_hier_info(handle(), nullptr, &s, nullptr);
        return s != 0;
    }

private:
    std::shared_ptr<ibmgpu_hier> h_;
};
inline SaHierarchy build_sa_hierarchy(const SparseMatrix& A, const SaOptions& o = {}) {
    const ibm_sa_options c{o.theta, o.max_coarse, o.max_levels, o.power_iterations, o.keep_fine_tail};
    ibmgpu_hier_t h = nullptr;
    check(ibmgpu_sa_build(Context::get().h(), A.handle(), &c, &h));
    return SaHierarchy(h);
}
inline std::vector<double> sa_apply(const SaHierarchy& h, const std::vector<double>& r) {
    DeviceVector dr(r), dz(r.size());
    check(ibmgpu_sa_apply(Context::get().h(), h.handle(), dr.get(), dz.get()));
    return dz.download();
}

// krylov.hpp:40-66 / amg.hpp:237-246 — preconditioners select the device kernel set
struct Preconditioner {
    virtual ~Preconditioner() = default;
    virtual int kind() const = 0;
    virtual ibmgpu_hier_t hier() const { return nullptr; }
};
struct IdentityPreconditioner final : Preconditioner {
    int kind() const override { return IBMGPU_PC_IDENTITY; }
};
struct DiagonalPreconditioner final : Preconditioner {
    explicit DiagonalPreconditioner(const SparseMatrix&) {}
    int kind() const override { return IBMGPU_PC_DIAGONAL; }
};
class SaPreconditioner final : public Preconditioner {
public:
    explicit SaPreconditioner(const SaHierarchy& h) : h_(&h) {}  // non-owning (amg.hpp:245)
    int kind() const override { return IBMGPU_PC_SA; }
    ibmgpu_hier_t hier() const override { return h_->handle(); }

private:
    const SaHierarchy* h_;
};

// krylov.hpp:70-141
inline SolveResult pcg(const SparseMatrix& A, const std::vector<double>& b, const std::vector<double>& x0,
                       const Preconditioner& M, const SolverParams& p) {
    p.validate();
    if (A.rows() != A.cols() || (int)b.size() != A.rows()) throw std::invalid_argument("pcg: dimension mismatch");
    DeviceVector db(b), dx(x0.empty() ? std::vector<double>(b.size(), 0.0) : x0);
    const ibm_solver_params c{p.rel_tol, p.max_iters, p.record_history ? 1 : 0, p.check_symmetry ? 1 : 0};
    ibm_solve_result r{};
    std::vector<double> hist(p.record_history ? (size_t)p.max_iters + 1 : 0);
    check(ibmgpu_pcg(Context::get().h(), A.handle(), M.kind(), M.hier(), db.get(), dx.get(), &c, &r,
                     p.record_history ? hist.data() : nullptr));
    SolveResult out;
    out.x = dx.download();
    out.iterations = r.iterations;
    out.rel_residual = r.rel_residual;
    out.status = static_cast<SolveStatus>(r.status);
    if (p.record_history) out.history.assign(hist.begin(), hist.begin() + r.history_len);
    return out;
}
inline SolveResult cg(const SparseMatrix& A, const std::vector<double>& b, const std::vector<double>& x0,
                      const SolverParams& p) {
    return pcg(A, b, x0, IdentityPreconditioner{}, p);
}

// stepper.hpp:128-145 / :169-356
struct StepReport {
    bool ok = true;
    std::string message;
    int solve1_iters = 0, solve2_iters = 0;
    double solve1_res = 0, solve2_res = 0, div_residual = 0, noslip_residual = 0;
    bool rebuilt_hierarchy = false, rebuilt_operators = false;
    double bc_cfl = 0, t_assembly = 0, t_precond = 0, t_explicit = 0, t_solve1 = 0, t_solve2 = 0, t_projection = 0;
};
class Stepper {
public:
    explicit Stepper(const std::string& cfg_path, const ibm_case_overrides& ov = ibm_case_overrides{}) {
        ibmgpu_stepper_t s = nullptr;
        check(ibmgpu_stepper_create(Context::get().h(), cfg_path.c_str(), &ov, &s));
        h_.reset(s);
    }
    StepReport advance() {
        ibm_step_report r{};
        check(ibmgpu_stepper_advance(h_.get(), &r));
        StepReport o;
        o.ok = r.ok != 0;
        o.message = r.message;
        o.solve1_iters = r.solve1_iters;
        o.solve2_iters = r.solve2_iters;
        o.solve1_res = r.solve1_res;
        o.solve2_res = r.solve2_res;
        o.div_residual = r.div_residual;
        o.noslip_residual = r.noslip_residual;
        o.rebuilt_hierarchy = r.rebuilt_hierarchy != 0;
        o.rebuilt_operators = r.rebuilt_operators != 0;
        o.bc_cfl = r.bc_cfl;
        o.t_assembly = r.t_assembly;
        o.t_precond = r.t_precond;
        o.t_explicit = r.t_explicit;
        o.t_solve1 = r.t_solve1;
        o.t_solve2 = r.t_solve2;
        o.t_projection = r.t_projection;
        return o;
    }
    // FlowState fields (stepper.hpp:99-108)
    std::vector<double> q() const { return get(0); }
    std::vector<double> lambda() const { return get(1); }
    std::vector<double> f_tilde() const { return get(5); }
    // compute_force_coefficients (diagnostics.hpp:26-38): {fx, fy, cd, cl}
    std::vector<double> forces() const {
        std::vector<double> f(4);
        check(ibmgpu_stepper_forces(h_.get(), f.data()));
        return f;
    }
    SparseMatrix op(const std::string& name) const {
        ibmgpu_mat_t m = nullptr;
        check(ibmgpu_stepper_op(h_.get(), name.c_str(), &m));
        return SparseMatrix::borrowed(m);
    }

    // raw state access (ibmgpu_stepper_get/set codes: 0 q, 1 lambda, 2 conv_prev, 3 boundary,
    // 4 {t, step, have_conv}, 5 f~) — what write_checkpoint / read_checkpoint below use
    std::vector<double> get(int which) const {
        int n = 0;
        check(ibmgpu_stepper_get(h_.get(), which, nullptr, &n));
        std::vector<double> v(n);
        check(ibmgpu_stepper_get(h_.get(), which, v.data(), &n));
        return v;
    }
    void set(int which, const std::vector<double>& v) {
        check(ibmgpu_stepper_set(h_.get(), which, v.data(), static_cast<int>(v.size())));
    }
    std::pair<int, int> grid_dims() const {
        int d[8];
        check(ibmgpu_stepper_dims(h_.get(), d));
        return {d[0], d[1]};
    }

private:
    struct Del {
        void operator()(ibmgpu_stepper_t s) const { ibmgpu_stepper_destroy(s); }
    };
    std::unique_ptr<ibmgpu_stepper, Del> h_;
};

// io.hpp:89-110 write_checkpoint: "ibmcfd-checkpoint 1", every double as %.17g
inline void write_checkpoint(const std::string& path, const Stepper& st) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::runtime_error("cannot open " + path);
    const auto sc = st.get(4);
    auto block = [&](const char* name, const double* v, size_t n) {
        std::fprintf(f, "%s %zu\n", name, n);
        for (size_t i = 0; i < n; ++i) std::fprintf(f, "%.17g\n", v[i]);
    };
    std::fprintf(f, "ibmcfd-checkpoint 1\n");
    std::fprintf(f, "t %.17g\n", sc[0]);
    std::fprintf(f, "step %d\n", static_cast<int>(sc[1]));
    std::fprintf(f, "have_conv %d\n", sc[2] != 0.0 ? 1 : 0);
    const auto q = st.get(0), cp = st.get(2), lam = st.get(1), bnd = st.get(3);
    block("q", q.data(), q.size());
    block("conv_prev", cp.data(), cp.size());
    block("lambda", lam.data(), lam.size());
    const auto [nx, ny] = st.grid_dims();
    const char* names[8] = {"left_u", "right_u", "left_v", "right_v", "bottom_v", "top_v", "bottom_u", "top_u"};
    const size_t sizes[8] = {size_t(ny), size_t(ny), size_t(ny - 1), size_t(ny - 1),
                             size_t(nx), size_t(nx), size_t(nx - 1), size_t(nx - 1)};
    size_t o = 0;
    for (int k = 0; k < 8; ++k) {
        block(names[k], bnd.data() + o, sizes[k]);
        o += sizes[k];
    }
    std::fclose(f);
}

// io.hpp:112-145 read_checkpoint (bodies follow the restored time, as sync_bodies_to_time)
inline void read_checkpoint(const std::string& path, Stepper& st) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::string magic, key;
    int version = 0;
    if (!(in >> magic >> version) || magic != "ibmcfd-checkpoint" || version != 1)
        throw std::runtime_error("checkpoint: bad header in " + path);
    double t = 0;
    int step = 0, have = 0;
    if (!(in >> key >> t) || key != "t") throw std::runtime_error("checkpoint: missing t");
    if (!(in >> key >> step) || key != "step") throw std::runtime_error("checkpoint: missing step");
    if (!(in >> key >> have) || key != "have_conv") throw std::runtime_error("checkpoint: missing have_conv");
    auto block = [&](const std::string& expect) {
        std::string name;
        size_t n = 0;
        if (!(in >> name >> n) || name != expect)
            throw std::runtime_error("checkpoint: expected block '" + expect + "', found '" + name + "'");
        std::vector<double> v(n);
        for (auto& x : v)
            if (!(in >> x)) throw std::runtime_error("checkpoint: truncated block " + expect);
        return v;
    };
    const auto q = block("q"), cp = block("conv_prev"), lam = block("lambda");
    std::vector<double> bnd;
    for (const char* n : {"left_u", "right_u", "left_v", "right_v", "bottom_v", "top_v", "bottom_u", "top_u"}) {
        const auto b = block(n);
        bnd.insert(bnd.end(), b.begin(), b.end());
    }
    st.set(0, q);
    st.set(2, cp);
    st.set(1, lam);
    st.set(3, bnd);
    st.set(4, {t, double(step), double(have)});
}

}  // namespace ibm_b200
