// hostcase_capi.cpp — host-only C entry points over the case setup (no CUDA): lets the CPU test
// suite pin grid / bodies / M / L / G against the reference without a GPU.
#include <cstring>
#include <stdexcept>
#include <string>

#include "../../../include/ibmgpu.h"
#include "case.hpp"

struct ibmgpu_hostcase {
    ibmhost::Case cfg;
    ibmhost::Grid g;
    std::vector<ibmhost::Body> bodies;
    std::vector<double> M;
    ibmhost::Csr L, G;
    std::vector<ibmhost::BcCoupling> vbc;
};

namespace {
void put_err(char* err, int cap, const std::string& m) {
    if (err && cap > 0) {
        std::strncpy(err, m.c_str(), (size_t)cap - 1);
        err[cap - 1] = 0;
    }
}
}  // namespace

extern "C" {

int ibmgpu_hostcase_open(const char* path, const ibm_case_overrides* ov, ibmgpu_hostcase_t* out, int* dims8, char* err,
                         int err_cap) {
    auto* h = new ibmgpu_hostcase();
    try {
        h->cfg = ibmhost::parse_case(path);
        if (ov) {
            if (ov->h_min > 0) h->cfg.h_min = ov->h_min;
            if (ov->dt > 0) h->cfg.dt = ov->dt;
        }
        h->g = ibmhost::build_grid(h->cfg.domain, h->cfg.uniform, h->cfg.h_min, h->cfg.ratio);
        h->bodies = ibmhost::build_bodies(h->cfg);
        for (auto& b : h->bodies) b.move_to(0.0);
        h->M = ibmhost::metric(h->g);
        h->L = ibmhost::diffusion(h->g, h->vbc);
        h->G = ibmhost::gradient(h->g);
    } catch (const std::invalid_argument& e) {
        put_err(err, err_cap, e.what());
        delete h;
        return IBMGPU_EINVAL;
    } catch (const std::exception& e) {
        put_err(err, err_cap, e.what());
        delete h;
        return IBMGPU_ESUPPORT;
    }
    int n_b = 0;
    for (const auto& b : h->bodies) n_b += b.n();
    if (dims8) {
        const int d[8] = {h->g.nx, h->g.ny, h->g.n_q(), h->g.n_p(), n_b, h->g.n_p() + 2 * n_b, 0, 0};
        std::memcpy(dims8, d, sizeof d);
    }
    *out = h;
    return 0;
}

int ibmgpu_hostcase_array(ibmgpu_hostcase_t h, const char* name, double* out, int* n) {
    const std::string k(name);
    const auto& g = h->g;
    std::vector<double> tmp;
    const std::vector<double>* v = nullptr;
    if (k == "x_faces") v = &g.x_faces;
    else if (k == "y_faces") v = &g.y_faces;
    else if (k == "dx") v = &g.dx;
    else if (k == "dy") v = &g.dy;
    else if (k == "x_c") v = &g.x_c;
    else if (k == "y_c") v = &g.y_c;
    else if (k == "del_x") v = &g.del_x;
    else if (k == "del_y") v = &g.del_y;
    else if (k == "M") v = &h->M;
    else if (k == "uniform") {
        tmp = {g.uniform_region.x0, g.uniform_region.x1, g.uniform_region.y0, g.uniform_region.y1};
        v = &tmp;
    } else if (k.rfind("body_", 0) == 0) {
        for (const auto& b : h->bodies)
            for (int p = 0; p < b.n(); ++p) {
                if (k == "body_x") tmp.push_back(b.x[p]);
                else if (k == "body_y") tmp.push_back(b.y[p]);
                else if (k == "body_ub_x") tmp.push_back(b.ub_x[p]);
                else if (k == "body_ub_y") tmp.push_back(b.ub_y[p]);
                else if (k == "body_ds") tmp.push_back(b.ds);
                else return IBMGPU_EINVAL;
            }
        v = &tmp;
    } else if (k == "visc_bc") {
        for (const auto& c : h->vbc) {
            tmp.push_back(c.row);
            tmp.push_back((double)c.slot);
            tmp.push_back(c.idx);
            tmp.push_back(c.coeff);
        }
        v = &tmp;
    } else if (k == "boundary") {
        tmp = ibmhost::Boundary::initial(g, h->cfg.bc).packed();
        v = &tmp;
    } else {
        return IBMGPU_EINVAL;
    }
    if (n) *n = (int)v->size();
    if (out) std::memcpy(out, v->data(), sizeof(double) * v->size());
    return 0;
}

int ibmgpu_hostcase_csr(ibmgpu_hostcase_t h, const char* name, int* rows, int* cols, int* nnz, int* rp, int* ci,
                        double* v) {
    const std::string k(name);
    const ibmhost::Csr* m = k == "L" ? &h->L : k == "G" ? &h->G : nullptr;
    if (!m) return IBMGPU_EINVAL;
    if (rows) *rows = m->rows;
    if (cols) *cols = m->cols;
    if (nnz) *nnz = (int)m->ci.size();
    if (rp) std::memcpy(rp, m->rp.data(), sizeof(int) * m->rp.size());
    if (ci) std::memcpy(ci, m->ci.data(), sizeof(int) * m->ci.size());
    if (v) std::memcpy(v, m->v.data(), sizeof(double) * m->v.size());
    return 0;
}

int ibmgpu_hostcase_move(ibmgpu_hostcase_t h, double t) {
    for (auto& b : h->bodies) b.move_to(t);
    return 0;
}

int ibmgpu_hostcase_free(ibmgpu_hostcase_t h) {
    delete h;
    return 0;
}

}  // extern "C"
