// reference_api.cpp — host-only C entry points for the reference-shaped C++ shim (ibm_b200.hpp):
// build_stretched_grid, discretize_circle/ellipse, parse_config and build_bodies (grid.hpp,
// body.hpp, config.hpp) over case.cpp. No CUDA calls.
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../../../include/ibmgpu.h"
#include "case.hpp"

namespace {

void put_err(char* err, int cap, const std::string& m) {
    if (err && cap > 0) {
        std::strncpy(err, m.c_str(), (size_t)cap - 1);
        err[cap - 1] = 0;
    }
}

template <class F>
int host_guard(char* err, int cap, F&& f) {
    try {
        f();
        return IBMGPU_OK;
    } catch (const std::invalid_argument& e) {
        put_err(err, cap, e.what());
        return IBMGPU_EINVAL;
    } catch (const std::exception& e) {
        put_err(err, cap, e.what());
        return IBMGPU_ESUPPORT;
    }
}

ibmhost::Rect rect(const double r[4]) { return ibmhost::Rect{r[0], r[1], r[2], r[3]}; }

void body_out(const ibmhost::Body& b, int* n, double* rx, double* ry, double* ds) {
    *n = b.n();
    if (rx) std::copy(b.ref_x.begin(), b.ref_x.end(), rx);
    if (ry) std::copy(b.ref_y.begin(), b.ref_y.end(), ry);
    if (ds) *ds = b.ds;
}

ibm_edge_bc edge_out(const ibmhost::EdgeBc& e) {
    return ibm_edge_bc{e.kind == ibmhost::Edge::convective ? 1 : 0, e.u, e.v};
}

int solver_kind(const std::string& t) {
    return t == "cg" ? 0 : t == "pcg-diag" ? 1 : t == "pcg-sa" ? 2 : t == "amg" ? 3 : -1;
}

}  // namespace

extern "C" {

int ibmgpu_host_grid(const double domain[4], const double uniform[4], double h_min, const double ratio[4], int* nx,
                     int* ny, double* packed, double* uniform4, char* err, int err_cap) {
    return host_guard(err, err_cap, [&] {
        if (!domain || !uniform || !ratio || !nx || !ny) throw std::invalid_argument("grid: null argument");
        const ibmhost::Grid g = ibmhost::build_grid(rect(domain), rect(uniform), h_min, ratio);
        *nx = g.nx;
        *ny = g.ny;
        if (packed) {
            double* o = packed;
            for (const auto* a : {&g.x_faces, &g.y_faces, &g.dx, &g.dy, &g.x_c, &g.y_c, &g.del_x, &g.del_y})
                o = std::copy(a->begin(), a->end(), o);
        }
        if (uniform4) {
            uniform4[0] = g.uniform_region.x0;
            uniform4[1] = g.uniform_region.x1;
            uniform4[2] = g.uniform_region.y0;
            uniform4[3] = g.uniform_region.y1;
        }
    });
}

int ibmgpu_host_circle(double cx, double cy, double diameter, double h, int* n, double* ref_x, double* ref_y,
                       double* ds, char* err, int err_cap) {
    return host_guard(err, err_cap, [&] { body_out(ibmhost::circle_body(cx, cy, diameter, h), n, ref_x, ref_y, ds); });
}

int ibmgpu_host_ellipse(double cx, double cy, double chord, double thickness_ratio, double h, int n_override, int* n,
                        double* ref_x, double* ref_y, double* ds, char* err, int err_cap) {
    return host_guard(err, err_cap, [&] {
        body_out(ibmhost::ellipse_body(cx, cy, chord, thickness_ratio, h, n_override), n, ref_x, ref_y, ds);
    });
}

int ibmgpu_host_case_config(const char* cfg_path, ibm_case_config* out, char* err, int err_cap) {
    return host_guard(err, err_cap, [&] {
        if (!cfg_path || !out) throw std::invalid_argument("config: null argument");
        const ibmhost::Case c = ibmhost::parse_case(cfg_path);
        ibm_case_config o{};
        const ibmhost::Rect* rs[2] = {&c.domain, &c.uniform};
        double* ds[2] = {o.domain, o.uniform};
        for (int k = 0; k < 2; ++k) {
            ds[k][0] = rs[k]->x0, ds[k][1] = rs[k]->x1, ds[k][2] = rs[k]->y0, ds[k][3] = rs[k]->y1;
        }
        o.h_min = c.h_min;
        std::copy(c.ratio, c.ratio + 4, o.ratio);
        o.nu = c.nu, o.re = c.re, o.u_inf = c.u_inf, o.ref_length = c.ref_length, o.u0 = c.u0, o.v0 = c.v0;
        o.dt = c.dt;
        o.n_steps = c.n_steps, o.n_out = c.n_out, o.checkpoint_every = c.checkpoint_every;
        o.n_pc = c.n_pc, o.n_order = c.n_order, o.slice_rows = c.slice_rows;
        o.n_bodies = (int)c.bodies.size();
        o.bc = ibm_bc_spec{edge_out(c.bc.left), edge_out(c.bc.right), edge_out(c.bc.bottom), edge_out(c.bc.top),
                           c.bc.u_inf};
        o.solve1 = ibm_solver_config{solver_kind(c.solve1.type), c.solve1.rel_tol, c.solve1.max_iters,
                                     c.solve1.sa_theta, c.solve1.sa_max_coarse};
        o.solve2 = ibm_solver_config{solver_kind(c.solve2.type), c.solve2.rel_tol, c.solve2.max_iters,
                                     c.solve2.sa_theta, c.solve2.sa_max_coarse};
        std::strncpy(o.out_dir, c.out_dir.c_str(), sizeof(o.out_dir) - 1);
        *out = o;
    });
}

int ibmgpu_host_case_bodies(const char* cfg_path, int* n_bodies, int* n_points_total, ibm_body_desc* descs, double* xy,
                            char* err, int err_cap) {
    return host_guard(err, err_cap, [&] {
        if (!cfg_path || !n_bodies || !n_points_total) throw std::invalid_argument("config: null argument");
        const ibmhost::Case c = ibmhost::parse_case(cfg_path);
        const std::vector<ibmhost::Body> bodies = ibmhost::build_bodies(c);
        int total = 0;
        for (const auto& b : bodies) total += b.n();
        *n_bodies = (int)bodies.size();
        *n_points_total = total;
        if (!descs || !xy) return;
        int off = 0;
        for (size_t k = 0; k < bodies.size(); ++k) {
            const auto& b = bodies[k];
            double* px = xy + 2 * off;
            double* py = px + b.n();
            std::copy(b.ref_x.begin(), b.ref_x.end(), px);
            std::copy(b.ref_y.begin(), b.ref_y.end(), py);
            const auto& m = b.motion;
            descs[k] = ibm_body_desc{b.n(),       px,        py,          b.center_x, b.center_y, b.ds,
                                     (int)m.kind, m.omega,   m.k,         m.kh,       m.heave_omega,
                                     m.heave_amp, m.A0,      m.f,         m.alpha0,   m.beta,
                                     m.phase,     b.rotation_invariant ? 1 : 0, b.preamble_offset,
                                     b.preamble_duration};
            off += b.n();
        }
    });
}

}  // extern "C"
