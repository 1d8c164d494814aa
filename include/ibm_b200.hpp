// ibm_b200.hpp — header-only C++ shim that re-exposes the reference's operator interface
// (/root/reference/proj/include/ibm/{sparse,krylov,amg,operators,stepper}.hpp) on top of the
// B200 C ABI (ibmgpu.h). A caller of `ibm::SparseMatrix`, `ibm::pcg`, `ibm::build_sa_hierarchy`
// or `ibm::Stepper` switches by including this header and using namespace `ibm_b200`: same
// names, same argument meaning, same exception types (std::invalid_argument for bad
// arguments, std::runtime_error otherwise). Host std::vector in and out, exactly as the
// reference's value semantics; the device keeps its own copies.
#pragma once
#include <algorithm>
#include <cmath>
#include <chrono>
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

// sparse.hpp:27-222. The CSR lives on the device; row_ptr()/col_idx()/values() return host
// copies made once on first use (a matrix is immutable after construction, as in the reference).
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
    // sparse.hpp:69-82
    static SparseMatrix identity(int n) { return diagonal(std::vector<double>((size_t)n, 1.0)); }
    static SparseMatrix diagonal(const std::vector<double>& d) {
        std::vector<Triplet> t;
        for (int i = 0; i < (int)d.size(); ++i) t.push_back({i, i, d[(size_t)i]});
        return from_triplets((int)d.size(), (int)d.size(), t);
    }
    // a matrix owned elsewhere (a stepper's operator, a hierarchy level); `keep` holds its owner
    static SparseMatrix borrowed(ibmgpu_mat_t m, std::shared_ptr<void> keep = {}) {
        SparseMatrix out;
        out.adopt(m, false);
        out.keep_ = std::move(keep);
        return out;
    }
    int rows() const { return rows_; }
    int cols() const { return cols_; }
    int nnz() const { return nnz_; }
    ibmgpu_mat_t handle() const { return h_.get(); }

    const std::vector<int>& row_ptr() const { return host().rp; }
    const std::vector<int>& col_idx() const { return host().ci; }
    const std::vector<double>& values() const { return host().v; }
    // operator()(i, j) (sparse.hpp:93-98)
    double operator()(int i, int j) const {
        const auto& H = host();
        const auto b = H.ci.begin() + H.rp[(size_t)i], e = H.ci.begin() + H.rp[(size_t)i + 1];
        const auto p = std::lower_bound(b, e, j);
        return (p != e && *p == j) ? H.v[(size_t)(p - H.ci.begin())] : 0.0;
    }
    std::vector<double> diagonal_vector() const {  // sparse.hpp:163-167
        std::vector<double> d((size_t)std::min(rows_, cols_));
        for (int i = 0; i < (int)d.size(); ++i) d[(size_t)i] = (*this)(i, i);
        return d;
    }
    double inf_norm() const {  // sparse.hpp:176-185: max row sum of |a_ij|
        const auto& H = host();
        double m = 0.0;
        for (int i = 0; i < rows_; ++i) {
            double s = 0.0;
            for (int k = H.rp[(size_t)i]; k < H.rp[(size_t)i + 1]; ++k) s += std::fabs(H.v[(size_t)k]);
            m = std::max(m, s);
        }
        return m;
    }

    // sparse.hpp:101 — y = A x on HOST pointers (x length cols, y length rows, caller-allocated),
    // exactly the reference's signature and meaning; the product runs on the device
    void spmv_into(const double* x, double* y) const {
        check(ibmgpu_spmv_host(Context::get().h(), handle(), x, y));
    }
    // the same on device pointers (no host transfer)
    void spmv_into_device(const double* x_dev, double* y_dev) const {
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
    const Host& host() const {
        if (!cache_) {
            auto h = std::make_shared<Host>(Host{std::vector<int>(rows_ + 1), std::vector<int>(nnz_),
                                                 std::vector<double>(nnz_)});
            check(ibmgpu_csr_download(ctx(), handle(), h->rp.data(), h->ci.data(), h->v.data()));
            cache_ = h;
        }
        return *cache_;
    }
    static ibmgpu_ctx_t ctx() { return Context::get().h(); }
    void adopt(ibmgpu_mat_t m, bool owned) {
        h_ = std::shared_ptr<ibmgpu_mat>(m, [owned](ibmgpu_mat_t p) {
            if (owned) ibmgpu_csr_destroy(Context::get().h(), p);
        });
        ibmgpu_csr_info(m, &rows_, &cols_, &nnz_);
    }
    std::shared_ptr<ibmgpu_mat> h_;
    std::shared_ptr<void> keep_;
    mutable std::shared_ptr<Host> cache_;
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
// sparse.hpp:357-373 vector helpers
inline double dot(const std::vector<double>& a, const std::vector<double>& b) {
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}
inline double norm2(const std::vector<double>& a) { return std::sqrt(dot(a, a)); }

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

// amg.hpp:21-52. A hierarchy built on the device; `levels[l].A/P/Pt` are that level's device
// matrices (host copies on first use), `inv_diag` and `omega` as the reference stores them.
struct SaOptions {
    double theta = 0.25;
    int max_coarse = 64;
    int max_levels = 25;
    int power_iterations = 10;
    int keep_fine_tail = 0;
};
struct SaLevel {
    SparseMatrix A, P, Pt;
    std::vector<double> inv_diag;
    double omega = 0.0;
};
class SaHierarchy {
public:
    std::vector<SaLevel> levels;  // levels[l].P maps level l+1 -> level l
    SparseMatrix coarse_A;
    int built_at_step = -1;
    bool coarsening_stalled = false;

    SaHierarchy() = default;
    // wrap a device hierarchy; owned: destroyed with the last copy of this object
    explicit SaHierarchy(ibmgpu_hier_t h, bool owned = true) {
        h_ = std::shared_ptr<ibmgpu_hier>(h, [owned](ibmgpu_hier_t p) {
            if (owned) ibmgpu_sa_destroy(Context::get().h(), p);
        });
        int nl = 0, st = 0, nc = 0;
        check(ibmgpu_hier_info(h, &nl, &st, &nc));
        coarsening_stalled = st != 0;
        for (int l = 0; l <= nl; ++l) {
            ibmgpu_mat_t A = nullptr, P = nullptr, Pt = nullptr;
            double om = 0.0;
            check(ibmgpu_hier_level(h, l, &A, &P, &Pt, &om));
            if (l == nl) {
                coarse_A = SparseMatrix::borrowed(A, h_);
                break;
            }
            SaLevel L;
            L.A = SparseMatrix::borrowed(A, h_);
            L.P = SparseMatrix::borrowed(P, h_);
            L.Pt = SparseMatrix::borrowed(Pt, h_);
            L.omega = om;
            L.inv_diag = L.A.diagonal_vector();
            for (double& d : L.inv_diag) d = 1.0 / d;
            levels.push_back(std::move(L));
        }
    }
    ibmgpu_hier_t handle() const { return h_.get(); }
    size_t level_count() const { return levels.size() + 1; }
    int finest_size() const { return levels.empty() ? coarse_A.rows() : levels.front().A.rows(); }

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

// krylov.hpp:39-66 / amg.hpp:237-246. The reference's one polymorphic extension point: any
// subclass overriding apply() is honoured (pcg calls it every iteration through the C ABI's
// callback solve). The built-in preconditioners also name the device kernel set that applies
// them inside the one-graph solve (device_kind), so they never leave the GPU.
class Preconditioner {
public:
    virtual ~Preconditioner() = default;
    virtual void apply(const std::vector<double>& r, std::vector<double>& z) const = 0;
    virtual int device_kind() const { return -1; }  // -1: user preconditioner (host apply)
    virtual ibmgpu_hier_t device_hier() const { return nullptr; }
};
class IdentityPreconditioner final : public Preconditioner {
public:
    void apply(const std::vector<double>& r, std::vector<double>& z) const override { z = r; }
    int device_kind() const override { return IBMGPU_PC_IDENTITY; }
};
class DiagonalPreconditioner final : public Preconditioner {
public:
    explicit DiagonalPreconditioner(const SparseMatrix& A) : inv_diag_(A.diagonal_vector()) {
        for (double& d : inv_diag_) {
            if (d == 0.0) throw std::invalid_argument("diagonal preconditioner: zero diagonal entry");
            d = 1.0 / d;
        }
    }
    void apply(const std::vector<double>& r, std::vector<double>& z) const override {
        z.resize(r.size());
        for (size_t i = 0; i < r.size(); ++i) z[i] = r[i] * inv_diag_[i];
    }
    int device_kind() const override { return IBMGPU_PC_DIAGONAL; }

private:
    std::vector<double> inv_diag_;
};
class SaPreconditioner final : public Preconditioner {
public:
    explicit SaPreconditioner(const SaHierarchy& h) : h_(&h) {}  // non-owning (amg.hpp:245)
    void apply(const std::vector<double>& r, std::vector<double>& z) const override { z = sa_apply(*h_, r); }
    int device_kind() const override { return IBMGPU_PC_SA; }
    ibmgpu_hier_t device_hier() const override { return h_->handle(); }

private:
    const SaHierarchy* h_;
};

namespace detail {
// C-ABI callback -> Preconditioner::apply on host vectors
struct ApplyCtx {
    const Preconditioner* M;
    std::vector<double> r, z;
    std::string error;
};
inline int apply_trampoline(void* user, int n, const double* r_dev, double* z_dev) {
    auto* a = static_cast<ApplyCtx*>(user);
    try {
        a->r.resize((size_t)n);
        check(ibmgpu_d2h(Context::get().h(), a->r.data(), r_dev, (size_t)n));
        a->M->apply(a->r, a->z);
        if ((int)a->z.size() != n) throw std::invalid_argument("preconditioner: apply returned a wrong size");
        check(ibmgpu_h2d(Context::get().h(), z_dev, a->z.data(), (size_t)n));
        return 0;
    } catch (const std::exception& e) {
        a->error = e.what();
        return 1;
    }
}
}  // namespace detail

// krylov.hpp:70-141
inline SolveResult pcg(const SparseMatrix& A, const std::vector<double>& b, const std::vector<double>& x0,
                       const Preconditioner& M, const SolverParams& p) {
    p.validate();
    if (A.rows() != A.cols() || (int)b.size() != A.rows()) throw std::invalid_argument("pcg: dimension mismatch");
    if (!x0.empty() && x0.size() != b.size()) throw std::invalid_argument("pcg: bad initial guess size");
    DeviceVector db(b), dx(x0.empty() ? std::vector<double>(b.size(), 0.0) : x0);
    const ibm_solver_params c{p.rel_tol, p.max_iters, p.record_history ? 1 : 0, p.check_symmetry ? 1 : 0};
    ibm_solve_result r{};
    std::vector<double> hist(p.record_history ? (size_t)p.max_iters + 1 : 0);
    double* hp = p.record_history ? hist.data() : nullptr;
    if (M.device_kind() >= 0) {
        check(ibmgpu_pcg(Context::get().h(), A.handle(), M.device_kind(), M.device_hier(), db.get(), dx.get(), &c, &r,
                         hp));
    } else {
        detail::ApplyCtx a{&M, {}, {}, {}};
        const int rc = ibmgpu_pcg_callback(Context::get().h(), A.handle(), detail::apply_trampoline, &a, db.get(),
                                           dx.get(), &c, &r, hp);
        if (rc != IBMGPU_OK && !a.error.empty()) throw std::invalid_argument(a.error);
        check(rc);
    }
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
// amg.hpp:250-280
inline SolveResult amg_solve(const SparseMatrix& A, const SaHierarchy& h, const std::vector<double>& b,
                             const std::vector<double>& x0, const SolverParams& p) {
    p.validate();
    if (A.rows() != A.cols() || (int)b.size() != A.rows()) throw std::invalid_argument("amg: dimension mismatch");
    DeviceVector db(b), dx(x0.empty() ? std::vector<double>(b.size(), 0.0) : x0);
    const ibm_solver_params c{p.rel_tol, p.max_iters, 0, 0};
    ibm_solve_result r{};
    check(ibmgpu_amg_solve(Context::get().h(), A.handle(), h.handle(), db.get(), dx.get(), &c, &r));
    SolveResult out;
    out.x = dx.download();
    out.iterations = r.iterations;
    out.rel_residual = r.rel_residual;
    out.status = static_cast<SolveStatus>(r.status);
    return out;
}

// ---------------------------------------------------------------- grid, bodies, boundary, config
// The reference's host types (grid.hpp, body.hpp, boundary.hpp, config.hpp). Builders run the
// library's host code (bit-identical coordinates, ibmgpu_host_*).
namespace detail {
inline void host_check(int rc, const char* err) {
    if (rc == IBMGPU_OK) return;
    if (rc == IBMGPU_EINVAL) throw std::invalid_argument(err);
    throw std::runtime_error(err);
}
}  // namespace detail

struct Rect {  // grid.hpp:13-25
    double x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
    double width() const { return x1 - x0; }
    double height() const { return y1 - y0; }
};

struct StaggeredGrid {  // grid.hpp:27-78
    int nx = 0, ny = 0;
    std::vector<double> x_faces, y_faces, dx, dy, x_c, y_c, del_x, del_y;
    Rect domain, uniform_region;
    double h_min = 0.0;
    int n_u() const { return (nx - 1) * ny; }
    int n_v() const { return nx * (ny - 1); }
    int n_q() const { return n_u() + n_v(); }
    int n_p() const { return nx * ny; }
    int u_id(int i_f, int j) const { return (i_f - 1) + j * (nx - 1); }
    int v_id(int i, int j_f) const { return n_u() + i + (j_f - 1) * nx; }
    int p_id(int i, int j) const { return i + j * nx; }
    ibm_grid_desc desc() const {
        return ibm_grid_desc{nx, ny, x_faces.data(), y_faces.data(), dx.data(), dy.data(), x_c.data(), y_c.data(),
                             del_x.data(), del_y.data(), h_min,
                             {uniform_region.x0, uniform_region.x1, uniform_region.y0, uniform_region.y1}};
    }
};

inline StaggeredGrid build_stretched_grid(const Rect& domain, const Rect& uniform_region, double h_min,
                                          const double ratio[4]) {
    const double d[4] = {domain.x0, domain.x1, domain.y0, domain.y1};
    const double u[4] = {uniform_region.x0, uniform_region.x1, uniform_region.y0, uniform_region.y1};
    char err[256] = {0};
    StaggeredGrid g;
    detail::host_check(ibmgpu_host_grid(d, u, h_min, ratio, &g.nx, &g.ny, nullptr, nullptr, err, sizeof err), err);
    std::vector<double> packed((size_t)(6 * (g.nx + g.ny)));
    double u4[4];
    detail::host_check(ibmgpu_host_grid(d, u, h_min, ratio, &g.nx, &g.ny, packed.data(), u4, err, sizeof err), err);
    const double* p = packed.data();
    auto take = [&](std::vector<double>& v, int n) {
        v.assign(p, p + n);
        p += n;
    };
    take(g.x_faces, g.nx + 1), take(g.y_faces, g.ny + 1), take(g.dx, g.nx), take(g.dy, g.ny);
    take(g.x_c, g.nx), take(g.y_c, g.ny), take(g.del_x, g.nx - 1), take(g.del_y, g.ny - 1);
    g.domain = domain;
    g.uniform_region = Rect{u4[0], u4[1], u4[2], u4[3]};
    g.h_min = h_min;
    return g;
}
inline StaggeredGrid build_uniform_grid(const Rect& domain, double h) {  // grid.hpp:196-199
    const double r[4] = {1.0, 1.0, 1.0, 1.0};
    return build_stretched_grid(domain, domain, h, r);
}

enum class MotionKind { stationary, rotating, heaving, flapping };
struct MotionParams {  // body.hpp:32-52
    MotionKind kind = MotionKind::stationary;
    double omega = 0.0;
    double k = 0.0, kh = 0.0;
    double heave_omega = 0.0, heave_amp = 0.0;
    double A0 = 0.0, f = 0.0, alpha0 = 0.0, beta = 0.0, phase = 0.0;
};

// body.hpp:85-148. Positions follow move_to on the device side of the stepper; x, y hold the
// positions at construction time (t = 0) here.
struct LagrangianBody {
    std::vector<double> ref_x, ref_y;
    std::vector<double> x, y;
    std::vector<double> ub_x, ub_y;
    double center_x = 0.0, center_y = 0.0;
    double ds = 0.0;
    MotionParams motion;
    bool shape_rotation_invariant = false;
    double preamble_offset = 0.0, preamble_duration = 0.0;
    int n() const { return static_cast<int>(ref_x.size()); }
    ibm_body_desc desc() const {
        const auto& m = motion;
        return ibm_body_desc{n(),        ref_x.data(), ref_y.data(), center_x, center_y, ds, (int)m.kind,
                             m.omega,    m.k,          m.kh,         m.heave_omega, m.heave_amp, m.A0, m.f,
                             m.alpha0,   m.beta,       m.phase,      shape_rotation_invariant ? 1 : 0,
                             preamble_offset, preamble_duration};
    }
};
namespace detail {
inline LagrangianBody body_from(int n, std::vector<double> rx, std::vector<double> ry, double cx, double cy,
                                double ds) {
    LagrangianBody b;
    b.ref_x = std::move(rx);
    b.ref_y = std::move(ry);
    b.center_x = cx, b.center_y = cy, b.ds = ds;
    b.x = b.ref_x, b.y = b.ref_y;
    for (double& v : b.x) v += cx;
    for (double& v : b.y) v += cy;
    b.ub_x.assign((size_t)n, 0.0);
    b.ub_y.assign((size_t)n, 0.0);
    return b;
}
inline std::vector<ibm_body_desc> descs(const std::vector<LagrangianBody>& bodies) {
    std::vector<ibm_body_desc> d;
    for (const auto& b : bodies) d.push_back(b.desc());
    return d;
}
}  // namespace detail
inline LagrangianBody discretize_circle(double cx, double cy, double diameter, double h) {  // body.hpp:151-173
    char err[256] = {0};
    int n = 0;
    double ds = 0.0;
    detail::host_check(ibmgpu_host_circle(cx, cy, diameter, h, &n, nullptr, nullptr, nullptr, err, sizeof err), err);
    std::vector<double> rx((size_t)n), ry((size_t)n);
    detail::host_check(ibmgpu_host_circle(cx, cy, diameter, h, &n, rx.data(), ry.data(), &ds, err, sizeof err), err);
    LagrangianBody b = detail::body_from(n, std::move(rx), std::move(ry), cx, cy, ds);
    b.shape_rotation_invariant = true;
    return b;
}
inline LagrangianBody discretize_ellipse(double cx, double cy, double chord, double thickness_ratio, double h,
                                         int n_override = 0) {  // body.hpp:213-261
    char err[256] = {0};
    int n = 0;
    double ds = 0.0;
    detail::host_check(ibmgpu_host_ellipse(cx, cy, chord, thickness_ratio, h, n_override, &n, nullptr, nullptr,
                                           nullptr, err, sizeof err),
                       err);
    std::vector<double> rx((size_t)n), ry((size_t)n);
    detail::host_check(ibmgpu_host_ellipse(cx, cy, chord, thickness_ratio, h, n_override, &n, rx.data(), ry.data(),
                                           &ds, err, sizeof err),
                       err);
    return detail::body_from(n, std::move(rx), std::move(ry), cx, cy, ds);
}

enum class BcKind { dirichlet, convective };
struct EdgeBc {  // boundary.hpp:17-21
    BcKind kind = BcKind::dirichlet;
    double u = 0.0, v = 0.0;
};
struct BcSpec {  // boundary.hpp:23-32
    EdgeBc left, right, bottom, top;
    double u_inf = 1.0;
    bool any_convective() const {
        return left.kind == BcKind::convective || right.kind == BcKind::convective ||
               bottom.kind == BcKind::convective || top.kind == BcKind::convective;
    }
    ibm_bc_spec desc() const {
        auto e = [](const EdgeBc& x) { return ibm_edge_bc{x.kind == BcKind::convective ? 1 : 0, x.u, x.v}; };
        return ibm_bc_spec{e(left), e(right), e(bottom), e(top), u_inf};
    }
};

enum class SolverKind { cg, pcg_diag, pcg_sa, amg };
struct SolverConfig {  // config.hpp:33-37
    SolverKind kind = SolverKind::pcg_sa;
    SolverParams params;
    SaOptions sa;
};
// config.hpp:54-95 (bodies kept as the case file describes them; build_bodies re-reads them)
struct CaseConfig {
    Rect domain, uniform;
    double h_min = 0.0;
    double ratio[4] = {1.0, 1.0, 1.0, 1.0};
    double nu = 0.0, re = 0.0, u_inf = 1.0, ref_length = 1.0, u0 = 0.0, v0 = 0.0;
    double dt = 0.0;
    int n_steps = 0, n_out = 0, checkpoint_every = 0;
    int n_bodies = 0;
    BcSpec bc;
    SolverConfig solve1, solve2;
    int n_pc = 2, n_order = 1, slice_rows = 0;
    std::string output_dir = "out";
    std::string source;  // the file parse_config read
};
inline CaseConfig parse_config(const std::string& path) {  // config.hpp:236-355
    ibm_case_config c{};
    char err[512] = {0};
    detail::host_check(ibmgpu_host_case_config(path.c_str(), &c, err, sizeof err), err);
    CaseConfig o;
    o.domain = Rect{c.domain[0], c.domain[1], c.domain[2], c.domain[3]};
    o.uniform = Rect{c.uniform[0], c.uniform[1], c.uniform[2], c.uniform[3]};
    o.h_min = c.h_min;
    std::copy(c.ratio, c.ratio + 4, o.ratio);
    o.nu = c.nu, o.re = c.re, o.u_inf = c.u_inf, o.ref_length = c.ref_length, o.u0 = c.u0, o.v0 = c.v0;
    o.dt = c.dt;
    o.n_steps = c.n_steps, o.n_out = c.n_out, o.checkpoint_every = c.checkpoint_every;
    o.n_bodies = c.n_bodies;
    auto edge = [](const ibm_edge_bc& e) { return EdgeBc{e.kind == 1 ? BcKind::convective : BcKind::dirichlet, e.u, e.v}; };
    o.bc = BcSpec{edge(c.bc.left), edge(c.bc.right), edge(c.bc.bottom), edge(c.bc.top), c.bc.u_inf};
    auto solver = [](const ibm_solver_config& s) {
        SolverConfig r;
        r.kind = static_cast<SolverKind>(s.kind);
        r.params.rel_tol = s.rel_tol;
        r.params.max_iters = s.max_iters;
        r.sa.theta = s.sa_theta;
        r.sa.max_coarse = s.sa_max_coarse;
        return r;
    };
    o.solve1 = solver(c.solve1);
    o.solve2 = solver(c.solve2);
    o.n_pc = c.n_pc, o.n_order = c.n_order, o.slice_rows = c.slice_rows;
    o.output_dir = c.out_dir;
    o.source = path;
    return o;
}
inline std::vector<LagrangianBody> build_bodies(const CaseConfig& c) {  // config.hpp:358-385
    char err[512] = {0};
    int nb = 0, np = 0;
    detail::host_check(ibmgpu_host_case_bodies(c.source.c_str(), &nb, &np, nullptr, nullptr, err, sizeof err), err);
    std::vector<ibm_body_desc> d((size_t)nb);
    std::vector<double> xy((size_t)2 * np + 1);
    detail::host_check(ibmgpu_host_case_bodies(c.source.c_str(), &nb, &np, d.data(), xy.data(), err, sizeof err), err);
    std::vector<LagrangianBody> out;
    for (const auto& e : d) {
        LagrangianBody b = detail::body_from(e.n_points, std::vector<double>(e.ref_x, e.ref_x + e.n_points),
                                             std::vector<double>(e.ref_y, e.ref_y + e.n_points), e.center_x,
                                             e.center_y, e.ds);
        b.motion = MotionParams{static_cast<MotionKind>(e.motion), e.omega, e.k, e.kh, e.heave_omega, e.heave_amp,
                                e.A0, e.f, e.alpha0, e.beta, e.phase};
        b.shape_rotation_invariant = e.shape_rotation_invariant != 0;
        b.preamble_offset = e.preamble_offset;
        b.preamble_duration = e.preamble_duration;
        out.push_back(std::move(b));
    }
    return out;
}

// ---------------------------------------------------------------- operators + stepper
struct SteppingParams {  // stepper.hpp:110-125
    double dt = 0.0;
    int n_order = 1;
    int n_pc = 2;
    bool force_rebuild = false;
    int slice_rows = 0;
    SolverParams solve1, solve2;
    SaOptions sa;
    void validate() const {
        if (dt <= 0.0) throw std::invalid_argument("stepping: dt must be positive");
        if (n_pc < 1) throw std::invalid_argument("stepping: n_pc must be >= 1");
        solve1.validate();
        solve2.validate();
    }
    ibm_stepping_params desc() const {
        auto sp = [](const SolverParams& p) {
            return ibm_solver_params{p.rel_tol, p.max_iters, p.record_history ? 1 : 0, p.check_symmetry ? 1 : 0};
        };
        return ibm_stepping_params{dt, n_order, n_pc, force_rebuild ? 1 : 0, slice_rows, sp(solve1), sp(solve2),
                                   ibm_sa_options{sa.theta, sa.max_coarse, sa.max_levels, sa.power_iterations,
                                                  sa.keep_fine_tail}};
    }
};
inline SteppingParams stepping_from(const CaseConfig& c) {  // runner.hpp:63-73
    SteppingParams p;
    p.dt = c.dt;
    p.n_order = c.n_order;
    p.n_pc = c.n_pc;
    p.slice_rows = c.slice_rows;
    p.solve1 = c.solve1.params;
    p.solve2 = c.solve2.params;
    p.sa = c.solve2.sa;
    return p;
}

// operators.hpp:49-69 — the device operator set of a stepper (or of assemble_operators)
struct OperatorSet {
    double dt = 0.0, nu = 0.0;
    int n_order = 1, n_b = 0, pin_index = 0, slice_rows = 0;
    SparseMatrix L, G, E, H, A, BN, Q, QT, lhs2;
    int n_lambda() const { return G.cols() + 2 * n_b; }
};

namespace detail {
struct StepperHandle {
    ibmgpu_stepper_t h = nullptr;
    explicit StepperHandle(ibmgpu_stepper_t s) : h(s) {}
    ~StepperHandle() {
        if (h) ibmgpu_stepper_destroy(h);
    }
};
inline SparseMatrix stepper_op(const std::shared_ptr<StepperHandle>& s, const char* name) {
    ibmgpu_mat_t m = nullptr;
    check(ibmgpu_stepper_op(s->h, name, &m));
    return SparseMatrix::borrowed(m, s);
}
inline void fill_ops(OperatorSet& o, const std::shared_ptr<StepperHandle>& s) {
    for (auto [name, m] : {std::pair<const char*, SparseMatrix*>{"L", &o.L}, {"G", &o.G}, {"E", &o.E}, {"H", &o.H},
                           {"A", &o.A}, {"BN", &o.BN}, {"Q", &o.Q}, {"QT", &o.QT}, {"lhs2", &o.lhs2}})
        *m = stepper_op(s, name);
}
}  // namespace detail

// operators.hpp:420-442
inline OperatorSet assemble_operators(const StaggeredGrid& g, const std::vector<LagrangianBody>& bodies, double dt,
                                      double nu, int n_order, int pin_index = 0, int slice_rows = 0) {
    const ibm_grid_desc gd = g.desc();
    const auto bd = detail::descs(bodies);
    ibmgpu_stepper_t s = nullptr;
    check(ibmgpu_operators_create(Context::get().h(), &gd, (int)bd.size(), bd.data(), dt, nu, n_order, pin_index,
                                  slice_rows, &s));
    auto h = std::make_shared<detail::StepperHandle>(s);
    OperatorSet o;
    o.dt = dt, o.nu = nu, o.n_order = n_order, o.pin_index = pin_index, o.slice_rows = slice_rows;
    for (const auto& b : bodies) o.n_b += b.n();
    detail::fill_ops(o, h);
    return o;
}

// stepper.hpp:128-145 / :99-108
struct StepReport {
    bool ok = true;
    std::string message;
    int solve1_iters = 0, solve2_iters = 0;
    double solve1_res = 0, solve2_res = 0, div_residual = 0, noslip_residual = 0;
    bool rebuilt_hierarchy = false, rebuilt_operators = false;
    double bc_cfl = 0, t_assembly = 0, t_precond = 0, t_explicit = 0, t_solve1 = 0, t_solve2 = 0, t_projection = 0;
    // converts to the reference's own StepReport (same members), so code written against
    // ibm::StepReport (`StepReport rep = st.advance();` in runner.hpp:102) keeps compiling
    template <class T, class = decltype(std::declval<T&>().t_projection), class = decltype(std::declval<T&>().message)>
    operator T() const {
        T t;
        t.ok = ok, t.message = message, t.solve1_iters = solve1_iters, t.solve2_iters = solve2_iters;
        t.solve1_res = solve1_res, t.solve2_res = solve2_res, t.div_residual = div_residual;
        t.noslip_residual = noslip_residual, t.rebuilt_hierarchy = rebuilt_hierarchy;
        t.rebuilt_operators = rebuilt_operators, t.bc_cfl = bc_cfl, t.t_assembly = t_assembly;
        t.t_precond = t_precond, t.t_explicit = t_explicit, t.t_solve1 = t_solve1, t.t_solve2 = t_solve2;
        t.t_projection = t_projection;
        return t;
    }
};
struct FlowState {
    std::vector<double> q, conv_prev, phi, f_tilde, lambda;
    double t = 0.0;
    int step_index = 0;
    bool have_conv_prev = false;
};

// stepper.hpp:169-370. Every field stays in HBM; state(), ops() and hierarchy() are host views
// refreshed on demand after each advance().
class Stepper {
public:
    // Stepper(grid, bodies, bc, nu, params, u0, v0) (stepper.hpp:171-195)
    Stepper(const StaggeredGrid& grid, std::vector<LagrangianBody> bodies, BcSpec bc, double nu,
            SteppingParams params, double u0 = 0.0, double v0 = 0.0) {
        params.validate();
        const ibm_grid_desc gd = grid.desc();
        const auto bd = detail::descs(bodies);
        const ibm_bc_spec bs = bc.desc();
        const ibm_stepping_params sp = params.desc();
        ibmgpu_stepper_t s = nullptr;
        check(ibmgpu_stepper_create_from(Context::get().h(), &gd, (int)bd.size(), bd.data(), &bs, nu, &sp, u0, v0, &s));
        init(s, grid, params.dt, nu, params.n_order, params.slice_rows, bc.u_inf);
    }
    // The same constructor taking the REFERENCE's own objects (ibm::StaggeredGrid, ibm::LagrangianBody,
    // ibm::BcSpec, ibm::SteppingParams — any types with the reference's member names): the
    // reference's run_case (runner.hpp:86-88) switches to the device path by changing only the
    // declared type of `st` (INTEGRATION.md shows the diff; oracle/Makefile builds it).
    template <class Grid, class Body, class Bc, class Params>
    Stepper(const Grid& grid, const std::vector<Body>& bodies, const Bc& bc, double nu, const Params& params,
            double u0 = 0.0, double v0 = 0.0) {
        StaggeredGrid g;
        g.nx = grid.nx, g.ny = grid.ny;
        g.x_faces = grid.x_faces, g.y_faces = grid.y_faces, g.dx = grid.dx, g.dy = grid.dy;
        g.x_c = grid.x_c, g.y_c = grid.y_c, g.del_x = grid.del_x, g.del_y = grid.del_y;
        g.domain = Rect{grid.domain.x0, grid.domain.x1, grid.domain.y0, grid.domain.y1};
        g.uniform_region = Rect{grid.uniform_region.x0, grid.uniform_region.x1, grid.uniform_region.y0,
                                grid.uniform_region.y1};
        g.h_min = grid.h_min;
        std::vector<LagrangianBody> bs;
        for (const auto& b : bodies) {
            LagrangianBody o;
            o.ref_x = b.ref_x, o.ref_y = b.ref_y, o.x = b.x, o.y = b.y, o.ub_x = b.ub_x, o.ub_y = b.ub_y;
            o.center_x = b.center_x, o.center_y = b.center_y, o.ds = b.ds;
            const auto& m = b.motion;
            o.motion = MotionParams{static_cast<MotionKind>(static_cast<int>(m.kind)), m.omega, m.k, m.kh,
                                    m.heave_omega, m.heave_amp, m.A0, m.f, m.alpha0, m.beta, m.phase};
            o.shape_rotation_invariant = b.shape_rotation_invariant;
            o.preamble_offset = b.preamble_offset, o.preamble_duration = b.preamble_duration;
            bs.push_back(std::move(o));
        }
        auto edge = [](const auto& e) {
            return EdgeBc{static_cast<int>(e.kind) == 1 ? BcKind::convective : BcKind::dirichlet, e.u, e.v};
        };
        const BcSpec b2{edge(bc.left), edge(bc.right), edge(bc.bottom), edge(bc.top), bc.u_inf};
        SteppingParams p;
        p.dt = params.dt, p.n_order = params.n_order, p.n_pc = params.n_pc;
        p.force_rebuild = params.force_rebuild, p.slice_rows = params.slice_rows;
        auto sp = [](const auto& s) {
            SolverParams r;
            r.rel_tol = s.rel_tol, r.max_iters = s.max_iters;
            r.record_history = s.record_history, r.check_symmetry = s.check_symmetry;
            return r;
        };
        p.solve1 = sp(params.solve1), p.solve2 = sp(params.solve2);
        p.sa = SaOptions{params.sa.theta, params.sa.max_coarse, params.sa.max_levels, params.sa.power_iterations,
                         params.sa.keep_fine_tail};
        *this = Stepper(g, std::move(bs), b2, nu, p, u0, v0);
    }
    // from a case file (what run_case constructs, runner.hpp:77-88)
    explicit Stepper(const std::string& cfg_path, const ibm_case_overrides& ov = ibm_case_overrides{}) {
        ibmgpu_stepper_t s = nullptr;
        check(ibmgpu_stepper_create(Context::get().h(), cfg_path.c_str(), &ov, &s));
        double sc[6];
        check(ibmgpu_stepper_scalars(s, sc));
        init(s, StaggeredGrid{}, sc[0], sc[1], 1, 0, sc[3]);
    }

    StepReport advance() {
        ibm_step_report r{};
        check(ibmgpu_stepper_advance(h_->h, &r));
        ++epoch_;
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

    const FlowState& state() const {
        if (state_epoch_ != epoch_) {
            FlowState s;
            s.q = get(0);
            s.lambda = get(1);
            s.conv_prev = get(2);
            s.f_tilde = get(5);
            s.phi.assign(s.lambda.begin(), s.lambda.begin() + (s.lambda.size() - s.f_tilde.size()));
            const auto sc = get(4);
            s.t = sc[0];
            s.step_index = static_cast<int>(sc[1]);
            s.have_conv_prev = sc[2] != 0.0;
            state_ = std::move(s);
            state_epoch_ = epoch_;
        }
        return state_;
    }
    const OperatorSet& ops() const {  // moving bodies replace E, H, Q, QT, lhs2 every step
        if (ops_epoch_ != epoch_) {
            detail::fill_ops(ops_, h_);
            ops_epoch_ = epoch_;
        }
        return ops_;
    }
    const SaHierarchy& hierarchy() const {
        if (hier_epoch_ != epoch_) {
            ibmgpu_hier_t hh = nullptr;
            check(ibmgpu_stepper_hier(h_->h, &hh));
            hier_ = SaHierarchy(hh, false);
            hier_epoch_ = epoch_;
        }
        return hier_;
    }
    const StaggeredGrid& grid() const { return grid_; }
    // BoundaryState (boundary.hpp:34-40): the stored edge values in the reference's layout, as
    // any struct with its member names (e.g. ibm::BoundaryState for couette_profile_error)
    template <class BS>
    BS boundary_as() const {
        const auto v = get(3);
        const auto [nx, ny] = grid_dims();
        BS out;
        size_t o = 0;
        auto take = [&](std::vector<double>& dst, int n) {
            dst.assign(v.begin() + (long)o, v.begin() + (long)o + n);
            o += (size_t)n;
        };
        take(out.left_u, ny), take(out.right_u, ny), take(out.left_v, ny - 1), take(out.right_v, ny - 1);
        take(out.bottom_v, nx), take(out.top_v, nx), take(out.bottom_u, nx - 1), take(out.top_u, nx - 1);
        return out;
    }
    struct BoundaryState {
        std::vector<double> left_u, right_u, left_v, right_v, bottom_v, top_v, bottom_u, top_u;
    };
    BoundaryState boundary() const { return boundary_as<BoundaryState>(); }
    // compute_force_coefficients on the device copy of f~ (diagnostics.hpp:26-38): {fx, fy, cd, cl}
    std::vector<double> forces() const {
        std::vector<double> f(4);
        check(ibmgpu_stepper_forces(h_->h, f.data()));
        return f;
    }
    SparseMatrix op(const std::string& name) const { return detail::stepper_op(h_, name.c_str()); }

    // raw state access (ibmgpu_stepper_get/set codes: 0 q, 1 lambda, 2 conv_prev, 3 boundary,
    // 4 {t, step, have_conv}, 5 f~) — what write_checkpoint / read_checkpoint below use
    std::vector<double> get(int which) const {
        int n = 0;
        check(ibmgpu_stepper_get(h_->h, which, nullptr, &n));
        std::vector<double> v(n);
        check(ibmgpu_stepper_get(h_->h, which, v.data(), &n));
        return v;
    }
    void set(int which, const std::vector<double>& v) {
        check(ibmgpu_stepper_set(h_->h, which, v.data(), static_cast<int>(v.size())));
        ++epoch_;
    }
    std::pair<int, int> grid_dims() const {
        int d[8];
        check(ibmgpu_stepper_dims(h_->h, d));
        return {d[0], d[1]};
    }

private:
    void init(ibmgpu_stepper_t s, const StaggeredGrid& g, double dt, double nu, int n_order, int slice_rows,
              double u_inf) {
        h_ = std::make_shared<detail::StepperHandle>(s);
        int d[8];
        check(ibmgpu_stepper_dims(s, d));
        grid_ = g;
        if (grid_.nx == 0) {  // case-file construction: the grid from the device stepper
            grid_.nx = d[0], grid_.ny = d[1];
            std::vector<double>* arrs[8] = {&grid_.x_faces, &grid_.y_faces, &grid_.dx,    &grid_.dy,
                                            &grid_.x_c,     &grid_.y_c,     &grid_.del_x, &grid_.del_y};
            for (int k = 0; k < 8; ++k) {
                int n = 0;
                check(ibmgpu_stepper_grid(s, k, nullptr, &n));
                arrs[k]->resize((size_t)n);
                check(ibmgpu_stepper_grid(s, k, arrs[k]->data(), &n));
            }
        }
        ops_.dt = dt, ops_.nu = nu, ops_.n_order = n_order, ops_.slice_rows = slice_rows;
        ops_.n_b = d[4];
        u_inf_ = u_inf;
    }
    std::shared_ptr<detail::StepperHandle> h_;
    StaggeredGrid grid_;
    double u_inf_ = 1.0;
    long long epoch_ = 0;
    mutable long long state_epoch_ = -1, ops_epoch_ = -1, hier_epoch_ = -1;
    mutable FlowState state_;
    mutable OperatorSet ops_;
    mutable SaHierarchy hier_;
};

// diagnostics.hpp:17-38
struct ForceRecord {
    double t = 0.0, fx = 0.0, fy = 0.0, cd = 0.0, cl = 0.0;
};
inline ForceRecord compute_force_coefficients(const std::vector<double>& f_tilde, int n_b, double t, double u_inf,
                                              double ref_length) {
    ForceRecord r;
    r.t = t;
    for (int k = 0; k < n_b; ++k) {
        r.fx += f_tilde[static_cast<size_t>(k)];
        r.fy += f_tilde[static_cast<size_t>(n_b + k)];
    }
    const double denom = 0.5 * u_inf * u_inf * ref_length;
    r.cd = r.fx / denom;
    r.cl = r.fy / denom;
    return r;
}

// runner.hpp:165-232 solver bench on the device
struct BenchRow {
    std::string name;
    int iterations = 0;
    double seconds = 0.0;
    double rel_residual = 0.0;
    bool converged = false;
};
inline std::vector<BenchRow> solver_bench_matrix(const SparseMatrix& lhs2, int pin_index, const SolverParams& params,
                                                 const SaOptions& sa) {
    using clock = std::chrono::steady_clock;
    std::vector<double> w(static_cast<size_t>(lhs2.rows()));
    for (size_t i = 0; i < w.size(); ++i) w[i] = std::sin(0.7 * static_cast<double>(i) + 0.3);
    if (pin_index >= 0) w[static_cast<size_t>(pin_index)] = 0.0;
    const double wn = norm2(w);
    for (double& x : w) x /= wn;
    const std::vector<double> b = lhs2.spmv(w);
    std::vector<BenchRow> rows;
    auto push = [&](const std::string& name, const SolveResult& r, double secs) {
        rows.push_back({name, r.iterations, secs, r.rel_residual, r.converged()});
    };
    {
        auto t0 = clock::now();
        auto r = cg(lhs2, b, {}, params);
        push("cg", r, std::chrono::duration<double>(clock::now() - t0).count());
    }
    {
        auto t0 = clock::now();
        DiagonalPreconditioner pc(lhs2);
        auto r = pcg(lhs2, b, {}, pc, params);
        push("pcg-diag", r, std::chrono::duration<double>(clock::now() - t0).count());
    }
    {
        auto t0 = clock::now();
        auto h = build_sa_hierarchy(lhs2, sa);
        SaPreconditioner pc(h);
        auto r = pcg(lhs2, b, {}, pc, params);
        push("pcg-sa", r, std::chrono::duration<double>(clock::now() - t0).count());
    }
    {
        auto t0 = clock::now();
        auto h = build_sa_hierarchy(lhs2, sa);
        auto r = amg_solve(lhs2, h, b, {}, params);
        push("amg", r, std::chrono::duration<double>(clock::now() - t0).count());
    }
    return rows;
}
inline void print_bench(const std::vector<BenchRow>& rows, std::FILE* f) {
    std::fprintf(f, "%-10s %12s %12s %14s %10s\n", "solver", "iterations", "time [s]", "rel residual", "status");
    for (const auto& r : rows)
        std::fprintf(f, "%-10s %12d %12.4f %14.3e %10s\n", r.name.c_str(), r.iterations, r.seconds, r.rel_residual,
                     r.converged ? "ok" : "FAILED");
}

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
