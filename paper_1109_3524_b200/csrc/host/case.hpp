// case.hpp — host-side case setup kept from the reference's interface: config parsing
// (config.hpp:236-385), the stretched staggered grid (grid.hpp:85-190), Lagrangian bodies and
// their kinematics (body.hpp:30-294), boundary values (boundary.hpp:15-62) and the grid
// operators assembled once on the host (metric M, diffusion L + boundary couplings, gradient G;
// operators.hpp:75-228). Everything here is O(nx+ny+n_b) or one pass over the grid and is
// compiled with -ffp-contract=off so that grid coordinates and body points — which feed the
// device E/H assembly — are bit-identical to the reference's.
#pragma once
#include <limits>
#include <string>
#include <memory>
#include <utility>
#include <vector>

namespace ibmhost {

struct Rect {
    double x0 = 0, x1 = 0, y0 = 0, y1 = 0;
    double width() const { return x1 - x0; }
    double height() const { return y1 - y0; }
    bool contains(const Rect& r) const {
        return r.x0 >= x0 - 1e-12 && r.x1 <= x1 + 1e-12 && r.y0 >= y0 - 1e-12 && r.y1 <= y1 + 1e-12;
    }
};

struct Grid {
    int nx = 0, ny = 0;
    std::vector<double> x_faces, y_faces, dx, dy, x_c, y_c, del_x, del_y;
    Rect domain, uniform_region;
    double h_min = 0;
    int n_u() const { return (nx - 1) * ny; }
    int n_v() const { return nx * (ny - 1); }
    int n_p() const { return nx * ny; }
    int n_q() const { return n_u() + n_v(); }
    int u_id(int i_f, int j) const { return (i_f - 1) + j * (nx - 1); }
    int v_id(int i, int j_f) const { return n_u() + i + (j_f - 1) * nx; }
    int p_id(int i, int j) const { return i + j * nx; }
};

Grid build_grid(const Rect& domain, const Rect& uniform, double h_min, const double ratio[4]);

enum class Motion { stationary, rotating, heaving, flapping };

struct MotionParams {
    Motion kind = Motion::stationary;
    double omega = 0, k = 0, kh = 0, heave_omega = 0, heave_amp = 0;
    double A0 = 0, f = 0, alpha0 = 0, beta = 0, phase = 0;
    void finalize(double u_ref, double chord);
};

struct Body {
    std::vector<double> ref_x, ref_y, x, y, ub_x, ub_y;
    double center_x = 0, center_y = 0, ds = 0;
    MotionParams motion;
    bool rotation_invariant = false;
    double preamble_offset = 0, preamble_duration = 0;
    int n() const { return (int)ref_x.size(); }
    bool base_static() const;
    bool geometry_static() const;
    double static_after() const;
    void move_to(double t);
};

Body circle_body(double cx, double cy, double diameter, double h);
Body ellipse_body(double cx, double cy, double chord, double thickness, double h, int n_override);
Body point_file_body(const std::string& path);

enum class Edge { dirichlet, convective };
struct EdgeBc {
    Edge kind = Edge::dirichlet;
    double u = 0, v = 0;
};
struct BcSpec {
    EdgeBc left, right, bottom, top;
    double u_inf = 1.0;
};

// BoundaryState arrays in the reference order (boundary.hpp:37-40)
struct Boundary {
    std::vector<double> left_u, right_u, left_v, right_v, bottom_v, top_v, bottom_u, top_u;
    static Boundary initial(const Grid& g, const BcSpec& bc);
    std::vector<double> packed() const;
};

struct BodyCfg {
    enum Shape { circle, ellipse, points } shape = circle;
    double cx = 0, cy = 0, diameter = 1.0, chord = 1.0, thickness_ratio = 0.12;
    int n_points = 0;
    std::string points_file;
    MotionParams motion;
    double preamble_offset = 0, preamble_duration = 0;
};

struct SolverCfg {
    std::string type;
    double rel_tol = 1e-5;
    int max_iters = 2000;
    double sa_theta = 0.25;
    int sa_max_coarse = 64;
};

struct Case {
    Rect domain, uniform;
    double h_min = 0;
    double ratio[4] = {1, 1, 1, 1};
    double nu = 0, re = 0, u_inf = 1.0, ref_length = 1.0, u0 = 0, v0 = 0;
    double dt = 0;
    int n_steps = 0, n_out = 0, checkpoint_every = 0;
    std::vector<BodyCfg> bodies;
    BcSpec bc;
    SolverCfg solve1{"pcg-diag"}, solve2{"pcg-sa"};
    int n_pc = 2, n_order = 1, slice_rows = 0;
    std::string out_dir = "out";
    void validate();
};

// config.hpp:236-355; throws std::invalid_argument with the reference's messages
Case parse_case(const std::string& path);
std::vector<Body> build_bodies(const Case& c);

// ---- grid operators (host CSR) ----
// Default-initialising allocator: resize() leaves the storage untouched, so the parallel fill
// below is the first touch (a 64M-cell L is 8 GB; zeroing it first on one thread doubled setup).
template <class T>
struct UninitAlloc : std::allocator<T> {
    using std::allocator<T>::allocator;
    template <class U>
    struct rebind {
        using other = UninitAlloc<U>;
    };
    template <class U>
    void construct(U* p) noexcept {
        ::new (static_cast<void*>(p)) U;
    }
    template <class U, class... Args>
    void construct(U* p, Args&&... args) {
        ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
    }
};

struct Csr {
    int rows = 0, cols = 0;
    std::vector<int, UninitAlloc<int>> rp, ci;
    std::vector<double, UninitAlloc<double>> v;
};

enum Slot { LU, RU, LV, RV, BV, TV, BU, TU };
struct BcCoupling {
    int row;
    Slot slot;
    int idx;
    double coeff;
};

std::vector<double> metric(const Grid& g);                                  // operators.hpp:75-84
Csr diffusion(const Grid& g, std::vector<BcCoupling>& bc);                 // operators.hpp:94-194
Csr gradient(const Grid& g);                                               // operators.hpp:210-226

}  // namespace ibmhost
