// stepper.cu — Stepper::advance (stepper.hpp:231-356) with every field and operator in HBM.
//
// Setup: the case is parsed and the grid / bodies / M, L, G are assembled on the host
// (csrc/host/case.cpp, the reference's interface kept); A, B^N, E, H, Q, Q^T, lhs2 and the SA
// hierarchy are built on the device. Per step, host<->device traffic is O(n_b): body positions
// and velocities go up, the step report (and on request f~) come down.
//
// Per step (all kernels on the context stream):
//   bc update (boundary.hpp:82-173)      one block; serial mass-balance sum => bit-exact
//   convection (stepper.hpp:23-97)        thread per velocity unknown
//   viscous bc (operators.hpp:198-202)    thread per coupled boundary row, list order
//   rhs1 (stepper.hpp:150-165)            fused into the L SpMV epilogue (also seeds x0 = q)
//   solve 1  pcg(A, r1, q, diag)          one graph launch (pcg.cu)
//   rhs2 (stepper.hpp:295-301)            fused into the Q^T SpMV epilogue (bc2 on the fly, pin)
//   solve 2  pcg(lhs2, rhs2, lambda, SA)  one graph launch
//   projection (stepper.hpp:315-320)      Q SpMV with B^N (diagonal) applied in the epilogue
//   invariants (stepper.hpp:323-345)      Q^T SpMV + fused div/slip/NaN reductions
// This file is compiled with --fmad=false: every expression rounds like the reference's.
#include <chrono>
#include <condition_variable>
#include <deque>
#include <climits>
#include <map>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>

#include "amg.cuh"
#include "dist.cuh"
#include "host/dist_plan.hpp"
#include "host/case.hpp"
#include "internal.cuh"
#include "kern.cuh"
#include "pcg.cuh"
#include "refresh.cuh"
#include "assemble.cuh"

#include <nvtx3/nvToolsExt.h>

namespace ibmgpu {
struct GridDev;
GridDev* grid_dev_new(Ctx* c, const ibm_grid_desc& g);
void grid_dev_free(GridDev* g);
void assemble_eh_dev(Ctx* c, const GridDev& gd, int n_b, const double* px, const double* py, const double* ds,
                     Mat** E, Mat** H);
void coupled_system(Ctx* c, const Mat* G, const Mat* E, const Mat* BN, int pin_idx, int slice_rows, Mat** Q,
                    Mat** QT, Mat** lhs2, long long* peak);
void check_support(const double uniform[4], double h_min, int n_b, const double* px, const double* py);
void ctx_free_extras(Ctx*) {}
}  // namespace ibmgpu

using namespace ibmgpu;

namespace {

// packed boundary arrays (boundary.hpp:37-40 order)
struct BndLayout {
    int nx, ny;
    int lu, ru, lv, rv, bv, tv, bu, tu, total;
    void init(int nx_, int ny_) {
        nx = nx_, ny = ny_;
        lu = 0;
        ru = lu + ny;
        lv = ru + ny;
        rv = lv + ny - 1;
        bv = rv + ny - 1;
        tv = bv + nx;
        bu = tv + nx;
        tu = bu + nx - 1;
        total = tu + nx - 1;
    }
};

struct GridArrays {
    const double *dx, *dy, *del_x, *del_y;
};

struct EdgeKinds {
    int kind[4];  // left, right, bottom, top: 0 dirichlet, 1 convective
    double u[4], v[4];
    double u_inf, dt;
    double width, height;
};

// ---------------------------------------------------------------- boundary update
__global__ void k_bc_update(BndLayout L, GridArrays g, EdgeKinds e, const double* __restrict__ q,
                            double* __restrict__ bnd, double* __restrict__ bnd_n, int* __restrict__ err) {
    const int t = threadIdx.x, nt = blockDim.x;
    const int nx = L.nx, ny = L.ny;
    const int n_u = (nx - 1) * ny;
    for (int k = t; k < L.total; k += nt) bnd_n[k] = bnd[k];
    __syncthreads();
    auto uq = [&](int i_f, int j) { return q[(i_f - 1) + j * (nx - 1)] / g.dy[j]; };
    auto vq = [&](int i, int j_f) { return q[n_u + i + (j_f - 1) * nx] / g.dx[i]; };
    // Dirichlet resets
    if (e.kind[0] == 0) {
        for (int k = t; k < ny; k += nt) bnd[L.lu + k] = e.u[0];
        for (int k = t; k < ny - 1; k += nt) bnd[L.lv + k] = e.v[0];
    }
    if (e.kind[1] == 0) {
        for (int k = t; k < ny; k += nt) bnd[L.ru + k] = e.u[1];
        for (int k = t; k < ny - 1; k += nt) bnd[L.rv + k] = e.v[1];
    }
    if (e.kind[2] == 0) {
        for (int k = t; k < nx; k += nt) bnd[L.bv + k] = e.v[2];
        for (int k = t; k < nx - 1; k += nt) bnd[L.bu + k] = e.u[2];
    }
    if (e.kind[3] == 0) {
        for (int k = t; k < nx; k += nt) bnd[L.tv + k] = e.v[3];
        for (int k = t; k < nx - 1; k += nt) bnd[L.tu + k] = e.u[3];
    }
    // convective edges: b -= c (b - interior)
    if (e.kind[1] == 1) {
        const double c = e.u_inf * e.dt / g.dx[nx - 1];
        for (int j = t; j < ny; j += nt) bnd[L.ru + j] -= c * (bnd[L.ru + j] - uq(nx - 1, j));
        for (int jf = 1 + t; jf < ny; jf += nt) bnd[L.rv + jf - 1] -= c * (bnd[L.rv + jf - 1] - vq(nx - 1, jf));
    }
    if (e.kind[0] == 1) {
        const double c = e.u_inf * e.dt / g.dx[0];
        for (int j = t; j < ny; j += nt) bnd[L.lu + j] -= c * (bnd[L.lu + j] - uq(1, j));
        for (int jf = 1 + t; jf < ny; jf += nt) bnd[L.lv + jf - 1] -= c * (bnd[L.lv + jf - 1] - vq(0, jf));
    }
    if (e.kind[3] == 1) {
        const double c = e.u_inf * e.dt / g.dy[ny - 1];
        for (int i = t; i < nx; i += nt) bnd[L.tv + i] -= c * (bnd[L.tv + i] - vq(i, ny - 1));
        for (int i_f = 1 + t; i_f < nx; i_f += nt) bnd[L.tu + i_f - 1] -= c * (bnd[L.tu + i_f - 1] - uq(i_f, ny - 1));
    }
    if (e.kind[2] == 1) {
        const double c = e.u_inf * e.dt / g.dy[0];
        for (int i = t; i < nx; i += nt) bnd[L.bv + i] -= c * (bnd[L.bv + i] - vq(i, 1));
        for (int i_f = 1 + t; i_f < nx; i_f += nt) bnd[L.bu + i_f - 1] -= c * (bnd[L.bu + i_f - 1] - uq(i_f, 0));
    }
    __syncthreads();
    // global mass balance, summed serially in the reference's order (bit-exact)
    __shared__ double corr_sh;
    __shared__ int have_corr;
    if (t == 0) {
        double net = 0.0, conv_len = 0.0;
        for (int j = 0; j < ny; ++j) net += (bnd[L.ru + j] - bnd[L.lu + j]) * g.dy[j];
        for (int i = 0; i < nx; ++i) net += (bnd[L.tv + i] - bnd[L.bv + i]) * g.dx[i];
        if (e.kind[0] == 1) conv_len += e.height;
        if (e.kind[1] == 1) conv_len += e.height;
        if (e.kind[3] == 1) conv_len += e.width;
        if (e.kind[2] == 1) conv_len += e.width;
        have_corr = conv_len > 0.0;
        corr_sh = have_corr ? net / conv_len : 0.0;
        if (!have_corr && fabs(net) > 1e-9 * fmax(1.0, e.width + e.height)) *err = 1;
    }
    __syncthreads();
    if (have_corr) {
        const double corr = corr_sh;
        if (e.kind[1] == 1)
            for (int j = t; j < ny; j += nt) bnd[L.ru + j] -= corr;
        if (e.kind[0] == 1)
            for (int j = t; j < ny; j += nt) bnd[L.lu + j] += corr;
        if (e.kind[3] == 1)
            for (int i = t; i < nx; i += nt) bnd[L.tv + i] -= corr;
        if (e.kind[2] == 1)
            for (int i = t; i < nx; i += nt) bnd[L.bv + i] += corr;
    }
}

// ---------------------------------------------------------------- convection (stepper.hpp:23-97)
__global__ void k_convection(BndLayout L, GridArrays g, const double* __restrict__ q, const double* __restrict__ s,
                             double* __restrict__ conv) {
    const int nx = L.nx, ny = L.ny;
    const int n_u = (nx - 1) * ny, n_q = n_u + nx * (ny - 1);
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n_q) return;
    auto u_at = [&](int i_f, int j) -> double {
        if (i_f == 0) return s[L.lu + j];
        if (i_f == nx) return s[L.ru + j];
        return q[(i_f - 1) + j * (nx - 1)] / g.dy[j];
    };
    auto v_at = [&](int i, int j_f) -> double {
        if (j_f == 0) return s[L.bv + i];
        if (j_f == ny) return s[L.tv + i];
        return q[n_u + i + (j_f - 1) * nx] / g.dx[i];
    };
    if (row < n_u) {
        const int i_f = row % (nx - 1) + 1, j = row / (nx - 1);
        const double uc_w = 0.5 * (u_at(i_f - 1, j) + u_at(i_f, j));
        const double uc_e = 0.5 * (u_at(i_f, j) + u_at(i_f + 1, j));
        const double ddx = (uc_e * uc_e - uc_w * uc_w) / g.del_x[i_f - 1];
        auto corner = [&](int jf) {
            double u_cor, v_cor;
            const double wx = 0.5 * g.dx[i_f - 1] / g.del_x[i_f - 1];
            if (jf == 0) {
                u_cor = s[L.bu + i_f - 1];
                v_cor = (1.0 - wx) * s[L.bv + i_f - 1] + wx * s[L.bv + i_f];
            } else if (jf == ny) {
                u_cor = s[L.tu + i_f - 1];
                v_cor = (1.0 - wx) * s[L.tv + i_f - 1] + wx * s[L.tv + i_f];
            } else {
                const double wy = 0.5 * g.dy[jf - 1] / g.del_y[jf - 1];
                u_cor = (1.0 - wy) * u_at(i_f, jf - 1) + wy * u_at(i_f, jf);
                v_cor = (1.0 - wx) * v_at(i_f - 1, jf) + wx * v_at(i_f, jf);
            }
            return u_cor * v_cor;
        };
        const double ddy = (corner(j + 1) - corner(j)) / g.dy[j];
        conv[row] = g.del_x[i_f - 1] * (ddx + ddy);
    } else {
        const int k = row - n_u;
        const int i = k % nx, j_f = k / nx + 1;
        const double vc_s = 0.5 * (v_at(i, j_f - 1) + v_at(i, j_f));
        const double vc_n = 0.5 * (v_at(i, j_f) + v_at(i, j_f + 1));
        const double ddy = (vc_n * vc_n - vc_s * vc_s) / g.del_y[j_f - 1];
        auto corner = [&](int ic) {
            double u_cor, v_cor;
            const double wy = 0.5 * g.dy[j_f - 1] / g.del_y[j_f - 1];
            if (ic == 0) {
                v_cor = s[L.lv + j_f - 1];
                u_cor = (1.0 - wy) * s[L.lu + j_f - 1] + wy * s[L.lu + j_f];
            } else if (ic == nx) {
                v_cor = s[L.rv + j_f - 1];
                u_cor = (1.0 - wy) * s[L.ru + j_f - 1] + wy * s[L.ru + j_f];
            } else {
                const double wx = 0.5 * g.dx[ic - 1] / g.del_x[ic - 1];
                v_cor = (1.0 - wx) * v_at(ic - 1, j_f) + wx * v_at(ic, j_f);
                u_cor = (1.0 - wy) * u_at(ic, j_f - 1) + wy * u_at(ic, j_f);
            }
            return u_cor * v_cor;
        };
        const double ddx = (corner(i + 1) - corner(i)) / g.dx[i];
        conv[row] = g.del_y[j_f - 1] * (ddx + ddy);
    }
}

// ---------------------------------------------------------------- viscous bc (operators.hpp:198-202)
__global__ void k_visc_bc(int n_rows, const int* __restrict__ rows, const int* __restrict__ off,
                          const int* __restrict__ pos, const double* __restrict__ coeff, const double* __restrict__ s_n,
                          const double* __restrict__ s_np1, double* __restrict__ bcn, double* __restrict__ bcnp1) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n_rows) return;
    double a = 0.0, b = 0.0;
    for (int k = off[u]; k < off[u + 1]; ++k) {
        a += coeff[k] * s_n[pos[k]];
        b += coeff[k] * s_np1[pos[k]];
    }
    bcn[rows[u]] = a;
    bcnp1[rows[u]] = b;
}

// ---------------------------------------------------------------- fused SpMV epilogues
struct EpiRhs1 {  // r1 = (M/dt) q + (nu/2)(L q + bc_n + bc_np1) - c1 conv (+ c2 conv_prev); x0 = q
    static constexpr int NR = 0;
    const double *mdt, *q, *bcn, *bcnp1, *conv, *conv_prev;
    double half_nu, c1, c2;
    double *r1, *x0;
    __device__ bool skip() const { return false; }
    __device__ void row(int i, double s, double*) const {
        const double qi = q[i];
        double r = mdt[i] * qi + half_nu * (s + bcn[i] + bcnp1[i]) - c1 * conv[i];
        if (c2 != 0.0) r += c2 * conv_prev[i];
        r1[i] = r;
        x0[i] = qi;
    }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

struct Bc2 {  // boundary.hpp:177-188, evaluated per cell
    BndLayout L;
    const double *bnd, *dx, *dy;
    __device__ double operator()(int p) const {
        const int i = p % L.nx, j = p / L.nx;
        double v = 0.0;
        if (i == 0) v += bnd[L.lu + j] * dy[j];
        if (i == L.nx - 1) v -= bnd[L.ru + j] * dy[j];
        if (j == 0) v += bnd[L.bv + i] * dx[i];
        if (j == L.ny - 1) v -= bnd[L.tv + i] * dx[i];
        return v;
    }
};

struct EpiRhs2 {  // rhs2 = QT q* + [bc2; -u_B], rhs2[pin] = 0
    static constexpr int NR = 0;
    Bc2 bc2;
    int n_p, pin;
    const double* ub;
    double* rhs;
    __device__ bool skip() const { return false; }
    __device__ void row(int i, double s, double*) const {
        double v = i < n_p ? s + bc2(i) : s - ub[i - n_p];
        if (i == pin) v = 0.0;
        rhs[i] = v;
    }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

struct EpiProjectDiag {  // q_new = q* - bn .* (Q lambda); non-finite flag
    static constexpr int NR = 0;
    const double *qs, *bn;
    double* qn;
    int* nonfinite;
    __device__ bool skip() const { return false; }
    __device__ void row(int i, double s, double*) const {
        const double v = qs[i] - bn[i] * s;
        qn[i] = v;
        if (!isfinite(v)) *nonfinite = 1;
    }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

struct EpiProjectGen {  // q_new = q* - (BN y)
    static constexpr int NR = 0;
    const double* qs;
    double* qn;
    int* nonfinite;
    __device__ bool skip() const { return false; }
    __device__ void row(int i, double s, double*) const {
        const double v = qs[i] - s;
        qn[i] = v;
        if (!isfinite(v)) *nonfinite = 1;
    }
    __device__ RedSlot slot() const { return {}; }
    __device__ void fin(double*) const {}
};

struct StepDev {
    double div2, bc2n;
    unsigned long long slip_bits, ubmax_bits;
    int nonfinite, bc_err;
};

struct EpiInvariants {  // QT q_new -> ||-div - bc2||^2, ||bc2||^2, max|slip|, max|u_B|
    static constexpr int NR = 2;
    Bc2 bc2;
    int n_p;
    const double* ub;
    RedSlot rs;
    StepDev* sd;
    __device__ bool skip() const { return false; }
    __device__ void row(int i, double s, double* acc) const {
        if (i < n_p) {
            const double b = bc2(i);
            const double r = -s - b;
            acc[0] += r * r;
            acc[1] += b * b;
        } else {
            const double u = ub[i - n_p];
            const double sl = fabs(s - u);
            atomicMax(&sd->slip_bits, (unsigned long long)__double_as_longlong(sl));
            atomicMax(&sd->ubmax_bits, (unsigned long long)__double_as_longlong(fabs(u)));
        }
    }
    __device__ RedSlot slot() const { return rs; }
    __device__ void fin(double* tot) const {
        sd->div2 = tot[0];
        sd->bc2n = tot[1];
    }
};

struct BodyForces {  // diagnostics.hpp:26-38: F = sum f~ per component
    static constexpr int NR = 2;
    const double* f;
    int n_b;
    RedSlot rs;
    double* out;
    __device__ bool skip() const { return false; }
    __device__ void row(int k, double* acc) const {
        acc[0] += f[k];
        acc[1] += f[n_b + k];
    }
    __device__ RedSlot slot() const { return rs; }
    __device__ void fin(double* tot) const {
        out[0] = tot[0];
        out[1] = tot[1];
    }
};

inline int blocks(long long n, int b = 256) { return (int)((n + b - 1) / b); }

double host_from_bits(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, sizeof d);
    return d;
}

}  // namespace

namespace {
// operators.hpp:350-374 diagonal terms: M/dt, 1/M, dt * (1/M)
__global__ void k_metric_terms(long long n, const double* __restrict__ M, double dt, double* __restrict__ mdt,
                               double* __restrict__ minv, double* __restrict__ d) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double m = M[i];
    mdt[i] = __ddiv_rn(m, dt);
    const double mi = __ddiv_rn(1.0, m);
    minv[i] = mi;
    d[i] = __dmul_rn(dt, mi);
}
__global__ void k_fill(long long n, double v, double* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = v;
}
}  // namespace

namespace {
// compute_vorticity (diagnostics.hpp:42-56): omega = dv/dx - du/dy at the interior vertices,
// row-major in j, same operation order (bit-exact)
__global__ void k_vorticity(int nx, int ny, const double* __restrict__ dx, const double* __restrict__ dy,
                            const double* __restrict__ del_x, const double* __restrict__ del_y,
                            const double* __restrict__ q, double* __restrict__ w) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long m = (long long)(nx - 1) * (ny - 1);
    if (t >= m) return;
    const int i = 1 + (int)(t % (nx - 1)), j = 1 + (int)(t / (nx - 1));
    const long long n_u = (long long)(nx - 1) * ny;
    auto u_id = [&](int i_f, int jj) { return (long long)(i_f - 1) + (long long)jj * (nx - 1); };
    auto v_id = [&](int ii, int j_f) { return n_u + ii + (long long)(j_f - 1) * nx; };
    const double dvdx = __ddiv_rn(__dsub_rn(__ddiv_rn(q[v_id(i, j)], dx[i]), __ddiv_rn(q[v_id(i - 1, j)], dx[i - 1])),
                                  del_x[i - 1]);
    const double dudy = __ddiv_rn(__dsub_rn(__ddiv_rn(q[u_id(i, j)], dy[j]), __ddiv_rn(q[u_id(i, j - 1)], dy[j - 1])),
                                  del_y[j - 1]);
    w[t] = __dsub_rn(dvdx, dudy);
}
}  // namespace

namespace ibmgpu {
struct OpsPipeline;
void pipeline_free(OpsPipeline* p);
}  // namespace ibmgpu

struct ibmgpu_stepper {
    Ctx* c = nullptr;
    // moving bodies: the operators of the next steps (E, Q, Q^T, lhs2 and, on the policy steps, the
    // SA hierarchy) are prepared ahead on a worker stream — they depend only on the prescribed
    // kinematics, never on the flow state (stepper.cu OpsPipeline)
    ibmgpu::OpsPipeline* pipe = nullptr;
    bool pipe_on = false;
    ibmhost::Case cfg;
    ibmhost::Grid g;
    std::vector<ibmhost::Body> bodies;
    double dt = 0, nu = 0;
    int n_order = 1, n_pc = 2, slice_rows = 0;
    bool force_rebuild = false;
    ibm_solver_params p1{}, p2{};
    ibm_sa_options sa{};
    int n_b = 0, n_q = 0, n_p = 0, n_lambda = 0;
    double geom_static_after = 0.0;
    BndLayout bl{};
    EdgeKinds ek{};
    double max_cfl = 0.0;

    // operators
    Mat *L = nullptr, *G = nullptr, *A = nullptr, *BN = nullptr, *E = nullptr, *H = nullptr;
    Mat *Q = nullptr, *QT = nullptr, *lhs2 = nullptr;
    Hier* hier = nullptr;
    bool bn_diagonal = true;
    GridDev* gd = nullptr;
    RefreshCache rcache;  // moving bodies: G^T and the invariant pressure block (refresh.cu)
    bool check_refresh = false;
    int pin = 0;             // pressure cell pinned in lhs2 (stepper.hpp:176)
    bool ops_only = false;   // ibmgpu_operators_create: the operator set only
    bool sa_given = false;   // SaOptions came with SteppingParams (create_from)
    AggCache agg_cache;   // moving bodies: aggregates reused when the strength graph repeats

    // device vectors
    DBuf<double> dx, dy, del_x, del_y, mdt, bn_diag;
    DBuf<double> px, py, pds, ub;
    DBuf<double> q, q_new, conv, conv_prev, lambda, y;
    DBuf<double> bnd, bnd_n, bcn, bcnp1;
    DBuf<int> vb_rows, vb_off, vb_pos;
    DBuf<double> vb_coeff;
    int vb_n = 0;
    DBuf<StepDev> sd;
    DBuf<double> red_part;
    DBuf<unsigned> red_cnt;
    DBuf<double> forces;
    StepDev* sd_host = nullptr;

    // state
    double t = 0.0;
    int step = 0;
    bool have_conv = false;
    cudaEvent_t ev[8] = {};
    float phase_ms[6] = {};

    // row-slab solve 2 (dist.cu): enabled by ibmgpu_stepper_distribute
    int dist_ranks = 0, dist_min_rows = 0;
    Dist* dist = nullptr;   // solve 2 (SA)
    Dist* dist1 = nullptr;  // solve 1 (diagonal); A never changes, so planned once
    bool dist_stale = true;
    DBuf<double> b2, x2, b1, x1;

    ~ibmgpu_stepper() {
        pipeline_free(pipe);
        pipe = nullptr;
        if (c) cudaStreamSynchronize(c->stream);
        dist_destroy(dist);
        dist_destroy(dist1);
        if (c) {
            pcg_forget(c, A, nullptr);
            pcg_forget(c, lhs2, hier);
        }
        for (Mat* m : {L, G, A, BN, E, H, Q, QT, lhs2}) delete m;
        delete hier;
        if (gd) grid_dev_free(gd);
        if (sd_host) cudaFreeHost(sd_host);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
    }

    void upload_bodies() {
        std::vector<double> hx, hy, hds, hub;
        for (const auto& b : bodies)
            for (int p = 0; p < b.n(); ++p) {
                hx.push_back(b.x[p]);
                hy.push_back(b.y[p]);
                hds.push_back(b.ds);
            }
        hub.resize(2 * (size_t)n_b);
        int k = 0;
        for (const auto& b : bodies)
            for (int p = 0; p < b.n(); ++p, ++k) {
                hub[k] = b.ub_x[p];
                hub[n_b + k] = b.ub_y[p];
            }
        h2d(c, px.p, hx.data(), hx.size());
        h2d(c, py.p, hy.data(), hy.size());
        h2d(c, pds.p, hds.data(), hds.size());
        h2d(c, ub.p, hub.data(), hub.size());
    }

    void host_points(std::vector<double>& hx, std::vector<double>& hy) const {
        for (const auto& b : bodies)
            for (int p = 0; p < b.n(); ++p) {
                hx.push_back(b.x[p]);
                hy.push_back(b.y[p]);
            }
    }

    // refresh_body_operators (operators.hpp:445-450) on the device
    void refresh_body_operators() {
        static const bool prof = std::getenv("IBMGPU_SETUP_PROFILE") != nullptr;
        auto t0 = std::chrono::steady_clock::now();
        auto lap = [&](const char* what) {
            if (!prof) return;
            sync(c);
            const auto t1 = std::chrono::steady_clock::now();
            std::fprintf(stderr, "[refresh] %-14s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
            t0 = t1;
        };
        dist_stale = true;
        std::vector<double> hx, hy;
        host_points(hx, hy);
        const double uni[4] = {g.uniform_region.x0, g.uniform_region.x1, g.uniform_region.y0, g.uniform_region.y1};
        check_support(uni, g.h_min, n_b, hx.data(), hy.data());
        upload_bodies();
        Mat* En = nullptr;
        // H (operators.hpp:304-342) is assembled with E by the reference but never applied in a
        // step; it is built from the same uploaded points when first asked for (ensure_H)
        assemble_eh_dev(c, *gd, n_b, px.p, py.p, pds.p, &En, nullptr);
        delete E;
        delete H;
        E = En;
        H = nullptr;
        lap("E, H");
        Mat *Qn, *QTn, *L2n;
        if (rcache.ready()) {
            coupled_refresh(c, rcache, G, E, BN, &Qn, &QTn, &L2n);
            if (check_refresh) {  // IBMGPU_CHECK_REFRESH=1: compare with the full assembly
                Mat *Qf, *QTf, *L2f;
                coupled_system(c, G, E, BN, pin, slice_rows, &Qf, &QTf, &L2f, nullptr);
                const bool same = mat_equal(c, Qn, Qf) && mat_equal(c, QTn, QTf) && mat_equal(c, L2n, L2f);
                delete Qf;
                delete QTf;
                delete L2f;
                if (!same) fail(IBMGPU_ECUDA, "incremental refresh differs from the full assembly");
            }
        } else {
            coupled_system(c, G, E, BN, pin, slice_rows, &Qn, &QTn, &L2n, nullptr);
        }
        lap("Q, QT, lhs2");
        pcg_forget(c, lhs2, nullptr);
        delete Q;
        delete QT;
        delete lhs2;
        Q = Qn;
        QT = QTn;
        lhs2 = L2n;
        lap("free");
        mat_plan(c, Q);
        lap("plan Q");
        mat_plan(c, QT);
        lap("plan QT");
        mat_plan(c, lhs2);
        lap("plan lhs2");
    }

    Mat* ensure_H() {
        if (!H) {
            Mat* En = nullptr;
            assemble_eh_dev(c, *gd, n_b, px.p, py.p, pds.p, &En, &H);
            delete En;
        }
        return H;
    }

    // row owners of lambda: pressure j-slabs, force rows with the slab of their point's cell
    std::vector<int> lambda_owner(int R) const {
        std::vector<int> cj;
        for (const auto& b : bodies)
            for (int p = 0; p < b.n(); ++p) {
                const int j = (int)(std::upper_bound(g.y_faces.begin(), g.y_faces.end(), b.y[p]) - g.y_faces.begin()) - 1;
                cj.push_back(std::clamp(j, 0, g.ny - 1));
            }
        return ibmhost::partition_lambda(g.nx, g.ny, n_b, cj.data(), R);
    }

    // row owners of q: u(i_f, j) with the slab of cell row j, v(i, j_f) with the slab of j_f
    std::vector<int> q_owner(int R) const {
        std::vector<int> own((size_t)n_q);
        auto slab = [&](int j) { return static_cast<int>((static_cast<long long>(std::clamp(j, 0, g.ny - 1)) * R) / g.ny); };
        for (int j = 0; j < g.ny; ++j)
            for (int i_f = 1; i_f < g.nx; ++i_f) own[(size_t)g.u_id(i_f, j)] = slab(j);
        for (int j_f = 1; j_f < g.ny; ++j_f)
            for (int i = 0; i < g.nx; ++i) own[(size_t)g.v_id(i, j_f)] = slab(j_f);
        return own;
    }

    // one process per GPU over NCCL; otherwise virtual ranks on this GPU (loopback, with a
    // one-rank NCCL communicator moving the halos by NCCL send/recv to self)
    bool multi_rank() const { return c->nccl && c->nranks > 1; }

    void ensure_dist1() {
        if (dist1) return;
        const int R = multi_rank() ? c->nranks : dist_ranks;
        const auto own = q_owner(R);
        dist1 = dist_create(c, A, IBMGPU_PC_DIAGONAL, nullptr, own.data(), multi_rank() ? 1 : dist_ranks, 0);
        b1.alloc(c, (size_t)n_q);
        x1.alloc(c, (size_t)n_q);
    }

    void ensure_dist() {
        if (!dist_stale && dist) return;
        dist_destroy(dist);
        dist = nullptr;
        const int R = multi_rank() ? c->nranks : dist_ranks;
        const auto own = lambda_owner(R);
        dist = dist_create(c, lhs2, IBMGPU_PC_SA, hier, own.data(), multi_rank() ? 1 : dist_ranks, dist_min_rows);
        if (b2.n != (size_t)n_lambda) {
            b2.alloc(c, (size_t)n_lambda);
            x2.alloc(c, (size_t)n_lambda);
        }
        dist_stale = false;
    }

    void rebuild_hierarchy() {
        dist_stale = true;
        Hier* h = sa_build(c, lhs2, sa, rcache.ready() ? &agg_cache : nullptr);
        if (hier) {
            pcg_forget(c, nullptr, hier);
            delete hier;
        }
        hier = h;
        hier->built_at_step = step;
    }
};

namespace {

void stepper_setup(ibmgpu_stepper* S, const char* path, const ibm_case_overrides* ov) {
    Ctx* c = S->c;
    // IBMGPU_SETUP_PROFILE=1: wall time of each setup phase on stderr
    const bool prof = std::getenv("IBMGPU_SETUP_PROFILE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!prof) return;
        sync(c);
        const auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[setup] %-22s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    };
    if (path) {  // ibmgpu_stepper_create: a case file (runner.hpp:77-88 run_case's construction)
        S->cfg = ibmhost::parse_case(path);
        auto& cfg = S->cfg;
        if (ov) {
            if (ov->h_min > 0) cfg.h_min = ov->h_min;
            if (ov->dt > 0) cfg.dt = ov->dt;
            if (ov->n_pc > 0) cfg.n_pc = ov->n_pc;
            if (ov->slice_rows > 0) cfg.slice_rows = ov->slice_rows;
            S->force_rebuild = ov->force_rebuild != 0;
        }
        S->g = ibmhost::build_grid(cfg.domain, cfg.uniform, cfg.h_min, cfg.ratio);
        S->bodies = ibmhost::build_bodies(cfg);
    }  // else ibmgpu_stepper_create_from filled cfg, g and bodies (stepper.hpp:171-173)
    auto& cfg = S->cfg;
    require(cfg.dt > 0.0, "stepping: dt must be positive");
    require(cfg.n_pc >= 1, "stepping: n_pc must be >= 1");
    S->dt = cfg.dt;
    S->nu = cfg.nu;
    S->n_order = cfg.n_order;
    S->n_pc = cfg.n_pc;
    S->slice_rows = cfg.slice_rows;
    // runner.hpp:63-73 stepping_from: solve 1 is always PCG-diag, solve 2 PCG-SA (stepper.hpp:282, :303)
    S->p1 = ibm_solver_params{cfg.solve1.rel_tol, cfg.solve1.max_iters, 0, 0};
    S->p2 = ibm_solver_params{cfg.solve2.rel_tol, cfg.solve2.max_iters, 0, 0};
    if (!S->sa_given) S->sa = ibm_sa_options{cfg.solve2.sa_theta, cfg.solve2.sa_max_coarse, 25, 10, 0};

    const auto& g = S->g;
    for (auto& b : S->bodies) b.move_to(0.0);
    S->n_b = 0;
    for (const auto& b : S->bodies) S->n_b += b.n();
    S->n_q = g.n_q();
    S->n_p = g.n_p();
    S->n_lambda = S->n_p + 2 * S->n_b;
    for (const auto& b : S->bodies) S->geom_static_after = std::max(S->geom_static_after, b.static_after());

    // grid arrays on the device
    auto up = [&](DBuf<double>& d, const std::vector<double>& h) {
        d.alloc(c, h.size());
        h2d(c, d.p, h.data(), h.size());
    };
    up(S->dx, g.dx);
    up(S->dy, g.dy);
    up(S->del_x, g.del_x);
    up(S->del_y, g.del_y);
    // M, L (with its wall couplings) and G assembled on the device (assemble.cu, operators.hpp:75-228)
    S->bl.init(g.nx, g.ny);
    const int slot_off[8] = {S->bl.lu, S->bl.ru, S->bl.lv, S->bl.rv, S->bl.bv, S->bl.tv, S->bl.bu, S->bl.tu};
    GridOps gops = assemble_grid_ops(c, g.nx, g.ny, S->dx.p, S->dy.p, S->del_x.p, S->del_y.p, slot_off);
    S->L = gops.L;
    S->G = gops.G;
    lap("device M, L, G");

    // A = M/dt - (nu/2) L ; B^N (operators.hpp:350-374) on the device; M/dt, 1/M and dt/M are
    // formed from M on the device with the reference's rounding (one IEEE op each)
    const size_t nq = (size_t)S->n_q;
    require(S->dt > 0.0, "operators: dt must be positive");
    require(S->n_order >= 1 && S->n_order <= 3, "operators: B^N order must be 1, 2 or 3");
    DBuf<double> dd(c, nq), mi(c, nq);
    {
        const DBuf<double>& Md = gops.M;
        S->mdt.alloc(c, nq);
        k_metric_terms<<<blocks((long long)nq), 256, 0, c->stream>>>((long long)nq, Md.p, S->dt, S->mdt.p, mi.p, dd.p);
        CK_LAUNCH(c);
        Mat* Dm = diag_matrix(c, S->n_q, S->mdt.p);
        S->A = add(c, 1.0, Dm, -0.5 * S->nu, S->L);
        delete Dm;
    }
    {
        if (S->n_order == 1) {
            S->BN = diag_matrix(c, S->n_q, dd.p);
        } else {
            Mat* Xc = scale(c, S->L, 2, 0.0, mi.p);
            Mat* X = scale(c, Xc, 0, 0.5 * S->nu * S->dt, nullptr);
            delete Xc;
            DBuf<double> on(c, nq);
            k_fill<<<blocks((long long)nq), 256, 0, c->stream>>>((long long)nq, 1.0, on.p);
            CK_LAUNCH(c);
            Mat* I = diag_matrix(c, S->n_q, on.p);
            Mat* series = add(c, 1.0, I, 1.0, X);
            delete I;
            if (S->n_order == 3) {
                Mat* XX = spmm_rows(c, X, 0, X->rows, X);
                Mat* s3 = add(c, 1.0, series, 1.0, XX);
                delete XX;
                delete series;
                series = s3;
            }
            delete X;
            S->BN = scale(c, series, 1, 0.0, dd.p);
            delete series;
        }
    }
    S->bn_diagonal = S->n_order == 1 && S->BN->nnz == S->n_q;
    S->bn_diag.alloc(c, nq);
    diag_of(c, S->BN, S->bn_diag.p);
    lap("A, B^N");

    // body operators + coupled system
    S->px.alloc(c, (size_t)std::max(S->n_b, 1));
    S->py.alloc(c, (size_t)std::max(S->n_b, 1));
    S->pds.alloc(c, (size_t)std::max(S->n_b, 1));
    S->ub.alloc(c, (size_t)std::max(2 * S->n_b, 1));
    const ibm_grid_desc gdsc{g.nx,       g.ny,          g.x_faces.data(), g.y_faces.data(), g.dx.data(),
                             g.dy.data(), g.x_c.data(), g.y_c.data(),     g.del_x.data(),   g.del_y.data(),
                             g.h_min,
                             {g.uniform_region.x0, g.uniform_region.x1, g.uniform_region.y0, g.uniform_region.y1}};
    S->gd = grid_dev_new(c, gdsc);
    S->refresh_body_operators();
    // a moving body re-assembles only the body coupling from here on (refresh.cu)
    S->check_refresh = std::getenv("IBMGPU_CHECK_REFRESH") != nullptr;
    if (S->n_b > 0 && S->geom_static_after > 0.0 && !std::getenv("IBMGPU_FULL_REFRESH"))
        S->rcache.init(c, S->G, S->BN, S->lhs2, S->n_p, S->pin, S->n_order);
    {
        const char* e = std::getenv("IBMGPU_PIPELINE");  // IBMGPU_PIPELINE=0: operators built in line
        S->pipe_on = S->rcache.ready() && !(e && e[0] == '0');
    }
    lap("E, H, Q, Q^T, lhs2");
    for (Mat* m : {S->L, S->A, S->BN, S->G}) mat_plan(c, m);
    lap("SpMV plans");
    if (S->ops_only) {  // assemble_operators (operators.hpp:420-442) stops here
        sync(c);
        return;
    }

    // SA hierarchy with the force rows carried to the coarse level (stepper.hpp:179-181)
    S->sa.keep_fine_tail = 2 * S->n_b;
    S->rebuild_hierarchy();
    S->hier->built_at_step = 0;
    lap("SA hierarchy");

    // boundary + state
    const ibmhost::Boundary b0 = ibmhost::Boundary::initial(g, cfg.bc);
    up(S->bnd, b0.packed());
    S->bnd_n.alloc(c, (size_t)S->bl.total);
    const ibmhost::EdgeBc* edges[4] = {&cfg.bc.left, &cfg.bc.right, &cfg.bc.bottom, &cfg.bc.top};
    for (int e = 0; e < 4; ++e) {
        S->ek.kind[e] = edges[e]->kind == ibmhost::Edge::convective ? 1 : 0;
        S->ek.u[e] = edges[e]->u;
        S->ek.v[e] = edges[e]->v;
    }
    S->ek.u_inf = cfg.bc.u_inf;
    S->ek.dt = S->dt;
    S->ek.width = g.domain.width();
    S->ek.height = g.domain.height();
    // BcUpdateReport::max_cfl (boundary.hpp:108-143) depends only on dt and the edge widths
    if (S->ek.kind[1]) S->max_cfl = std::max(S->max_cfl, cfg.bc.u_inf * S->dt / g.dx[g.nx - 1]);
    if (S->ek.kind[0]) S->max_cfl = std::max(S->max_cfl, cfg.bc.u_inf * S->dt / g.dx[0]);
    if (S->ek.kind[3]) S->max_cfl = std::max(S->max_cfl, cfg.bc.u_inf * S->dt / g.dy[g.ny - 1]);
    if (S->ek.kind[2]) S->max_cfl = std::max(S->max_cfl, cfg.bc.u_inf * S->dt / g.dy[0]);

    // viscous boundary couplings grouped by row in list order (assembled with L on the device)
    S->vb_n = gops.n_wall_rows;
    S->vb_rows = std::move(gops.wall_rows);
    S->vb_off = std::move(gops.wall_off);
    S->vb_pos = std::move(gops.wall_pos);
    S->vb_coeff = std::move(gops.wall_coeff);
    S->bcn.alloc(c, nq);
    S->bcnp1.alloc(c, nq);
    CK(cudaMemsetAsync(S->bcn.p, 0, sizeof(double) * nq, c->stream));
    CK(cudaMemsetAsync(S->bcnp1.p, 0, sizeof(double) * nq, c->stream));

    // initial state (stepper.hpp:183-194)
    std::vector<double> q0(nq, 0.0);
    for (int j = 0; j < g.ny; ++j)
        for (int i_f = 1; i_f < g.nx; ++i_f) q0[g.u_id(i_f, j)] = cfg.u0 * g.dy[j];
    for (int j_f = 1; j_f < g.ny; ++j_f)
        for (int i = 0; i < g.nx; ++i) q0[g.v_id(i, j_f)] = cfg.v0 * g.dx[i];
    up(S->q, q0);
    S->q_new.alloc(c, nq);
    S->conv.alloc(c, nq);
    S->conv_prev.alloc(c, nq);
    CK(cudaMemsetAsync(S->conv_prev.p, 0, sizeof(double) * nq, c->stream));
    S->lambda.alloc(c, (size_t)S->n_lambda);
    CK(cudaMemsetAsync(S->lambda.p, 0, sizeof(double) * S->n_lambda, c->stream));
    S->y.alloc(c, nq);
    S->sd.alloc(c, 1);
    S->red_part.alloc(c, (size_t)std::max(spmv_grid(S->QT), 64) * 2 + 2 * 4096);
    S->red_cnt.alloc(c, 1);
    CK(cudaMemsetAsync(S->red_cnt.p, 0, sizeof(unsigned), c->stream));
    S->forces.alloc(c, 2);
    CK(cudaMallocHost(&S->sd_host, sizeof(StepDev)));
    for (auto& e : S->ev) CK(cudaEventCreate(&e));
    sync(c);
}

void set_err(ibm_step_report* rep, const std::string& m) {
    rep->ok = 0;
    std::strncpy(rep->message, m.c_str(), sizeof(rep->message) - 1);
    rep->message[sizeof(rep->message) - 1] = 0;
}

std::string fmt_res(double r) { return std::to_string(r); }

// Stepper::advance (stepper.hpp:231-356)
}  // namespace

namespace ibmgpu {

// ---------------------------------------------------------------- operator pipeline
// refresh_body_operators (operators.hpp:445-450) and the policy rebuilds of build_sa_hierarchy
// (stepper.hpp:257-265) for the coming steps, computed by a worker thread on its own stream while
// the main stream runs the current step's solves. Inputs: the prescribed body positions at each
// step's t_new (the same sequence of t + dt additions as the stepper), G, B^N and the refresh
// cache — all constant — so every prepared operator is bit-identical to the in-line one; the
// main thread only installs them. The workers run a bounded number of steps ahead (OpsPipeline::run).
struct Prepared {
    int step = -1;
    double t_new = 0.0;
    bool moving = false, rebuild = false;
    std::vector<ibmhost::Body> bodies;  // positions at t_new
    Mat *E = nullptr, *Q = nullptr, *QT = nullptr, *lhs2 = nullptr;
    Hier* hier = nullptr;
    int err_code = 0;
    std::string err;
    long long launches = 0;
    double worker_ms = 0.0;
    ~Prepared() {
        for (Mat* m : {E, Q, QT, lhs2}) delete m;
        delete hier;
    }
};

// Workers build the operators of the next steps concurrently: each owns a stream, an aggregate
// cache and its body positions, and claims the next unclaimed step (rebuild steps and cheap
// refresh-only steps interleave, so two workers overlap two hierarchy builds). A build is a chain
// of small, latency-bound kernels with host round trips, so concurrent builds share the GPU
// well. IBMGPU_PIPE_WORKERS sets the count (default 3).
struct OpsPipeline {
    struct Worker {
        Ctx wc;  // own stream, the stepper context's pool
        std::thread th;
        std::vector<ibmhost::Body> bodies;
        DBuf<double> px, py, pds;
        AggCache agg;
    };
    ibmgpu_stepper* S = nullptr;
    std::vector<std::unique_ptr<Worker>> workers;
    std::mutex mu;
    std::condition_variable cv;
    std::map<int, std::unique_ptr<Prepared>> ready;
    int first_step = 0;
    int next_step = 0;        // next step to claim
    double t_prev = 0.0;      // time before next_step
    int in_flight = 0;
    int finish_step = INT_MAX;  // first step that was not moving (or failed): nothing after it
    int taken_upto = INT_MIN;   // last step handed to the stepper
    bool stop = false;

    static int worker_count() {
        static const int n = [] {
            const char* e = std::getenv("IBMGPU_PIPE_WORKERS");
            return e ? std::max(1, std::min(4, std::atoi(e))) : 3;  // 3: flapping 96-97 -> 100 steps/s vs 2
        }();
        return n;
    }

    OpsPipeline(ibmgpu_stepper* st, int step, double t) : S(st), first_step(step), next_step(step), t_prev(t) {
        CK(cudaStreamSynchronize(S->c->stream));
        const int nw = worker_count();
        for (int w = 0; w < nw; ++w) {
            auto W = std::make_unique<Worker>();
            W->wc.device = S->c->device;
            W->wc.num_sms = S->c->num_sms;
            W->wc.pool = S->c->pool;
            W->wc.eager = S->c->eager;
            int lo = 0, hi = 0;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CK(cudaStreamCreateWithPriority(&W->wc.stream, cudaStreamNonBlocking, lo));
            W->bodies = S->bodies;
            if (w == 0) {
                W->agg = std::move(S->agg_cache);  // worker 0 owns the stepper's aggregate cache
                W->agg.rehome(W->wc.stream);
            }
            workers.push_back(std::move(W));
        }
        for (auto& W : workers) {
            Worker* wp = W.get();
            wp->th = std::thread([this, wp] { run(*wp); });
        }
    }
    ~OpsPipeline() {
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
        cv.notify_all();
        for (auto& W : workers)
            if (W->th.joinable()) W->th.join();
        ready.clear();
        for (auto& W : workers) {
            W->px.release(), W->py.release(), W->pds.release();
            zero_scratch_free(&W->wc);
            cudaStreamSynchronize(W->wc.stream);
        }
        workers[0]->agg.rehome(S->c->stream);
        S->agg_cache = std::move(workers[0]->agg);
        for (size_t w = 1; w < workers.size(); ++w) workers[w]->agg = AggCache{};  // freed on its stream
        for (auto& W : workers) cudaStreamDestroy(W->wc.stream);
    }

    std::unique_ptr<Prepared> produce(Worker& W, int step, double tp) {
        auto P = std::make_unique<Prepared>();
        const auto t0 = std::chrono::steady_clock::now();
        P->step = step;
        P->t_new = tp + S->dt;
        P->moving = tp < S->geom_static_after;
        if (!P->moving) return P;
        for (auto& b : W.bodies) b.move_to(P->t_new);
        P->bodies = W.bodies;
        Ctx* c = &W.wc;
        try {
            std::vector<double> hx, hy, hds;
            for (const auto& b : W.bodies)
                for (int p = 0; p < b.n(); ++p) {
                    hx.push_back(b.x[p]);
                    hy.push_back(b.y[p]);
                    hds.push_back(b.ds);
                }
            const auto& g = S->g;
            const double uni[4] = {g.uniform_region.x0, g.uniform_region.x1, g.uniform_region.y0, g.uniform_region.y1};
            check_support(uni, g.h_min, S->n_b, hx.data(), hy.data());
            const size_t nb = (size_t)std::max(S->n_b, 1);
            if (W.px.n != nb) W.px.alloc(c, nb), W.py.alloc(c, nb), W.pds.alloc(c, nb);
            h2d(c, W.px.p, hx.data(), hx.size());
            h2d(c, W.py.p, hy.data(), hy.size());
            h2d(c, W.pds.p, hds.data(), hds.size());
            assemble_eh_dev(c, *S->gd, S->n_b, W.px.p, W.py.p, W.pds.p, &P->E, nullptr);
            coupled_refresh(c, S->rcache, S->G, P->E, S->BN, &P->Q, &P->QT, &P->lhs2);
            for (Mat* m : {P->Q, P->QT, P->lhs2}) mat_plan(c, m);
            const bool freezing = P->t_new >= S->geom_static_after;
            P->rebuild = S->force_rebuild || freezing || step % S->n_pc == 0;
            if (P->rebuild) P->hier = sa_build(c, P->lhs2, S->sa, &W.agg);
            sync(c);
        } catch (const Error& e) {
            cudaStreamSynchronize(W.wc.stream);
            P->err_code = e.code;
            P->err = e.what();
        } catch (const std::exception& e) {
            cudaStreamSynchronize(W.wc.stream);
            P->err_code = IBMGPU_ECUDA;
            P->err = e.what();
        }
        P->launches = W.wc.launches;
        W.wc.launches = 0;
        P->worker_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        return P;
    }

    void run(Worker& W) {
        cudaSetDevice(W.wc.device);
        // prepared-but-not-installed steps are bounded (each holds a lhs2 and maybe a hierarchy):
        // one in flight per worker plus IBMGPU_PIPE_AHEAD ready ahead. Default 3 (flapping, three
        // workers: 99.6-100 steps/s; 1 ahead: 97.4); large moving cases can lower it for memory
        static const int ahead = [] {
            const char* e = std::getenv("IBMGPU_PIPE_AHEAD");
            return e ? std::max(0, std::atoi(e)) : 3;
        }();
        const int cap = (int)workers.size() + ahead;
        for (;;) {
            int step;
            double tp;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return stop || (next_step < finish_step && (int)ready.size() + in_flight < cap); });
                if (stop) return;
                step = next_step++;
                tp = t_prev;
                t_prev = tp + S->dt;  // the same sum the main timeline forms (P->t_new)
                ++in_flight;
            }
            auto P = produce(W, step, tp);
            {
                std::lock_guard<std::mutex> lk(mu);
                if (!P->moving || P->err_code) finish_step = std::min(finish_step, step + 1);
                --in_flight;
                ready[step] = std::move(P);
            }
            cv.notify_all();
        }
    }

    // the prepared operators of `step` (waits for them); nullptr if the pipeline cannot produce it
    std::unique_ptr<Prepared> take(int step) {
        std::unique_lock<std::mutex> lk(mu);
        // a step before the timeline, or one already taken (a failed step being repeated)
        if (step < first_step || step <= taken_upto) return nullptr;
        cv.wait(lk, [&] { return ready.count(step) || step >= finish_step; });
        auto it = ready.find(step);
        if (it == ready.end()) return nullptr;
        auto P = std::move(it->second);
        ready.erase(it);
        taken_upto = step;
        lk.unlock();
        cv.notify_all();
        return P;
    }
};

void pipeline_free(OpsPipeline* p) { delete p; }

}  // namespace ibmgpu

namespace {

// NVTX range per phase of Stepper::advance (stepper.hpp:232-321): visible in any CUDA profiler
// timeline (nsys / ncu --nvtx); the ranges cover the host enqueue of each phase
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

void advance(ibmgpu_stepper* S, ibm_step_report* rep) {
    NvtxRange step_range("ibm.advance");
    require(!S->ops_only, "stepper: this handle holds an operator set only (ibmgpu_operators_create)");
    Ctx* c = S->c;
    using clk = std::chrono::steady_clock;
    std::memset(rep, 0, sizeof(*rep));
    rep->ok = 1;
    const double t_new = S->t + S->dt;
    const bool moving = S->t < S->geom_static_after;
    auto tic = clk::now();
    if (moving && S->pipe_on && S->rcache.ready() && !S->dist && S->dist_ranks == 0 && !c->nccl) {
        NvtxRange r("install prepared operators");
        std::unique_ptr<Prepared> P;
        for (int attempt = 0; attempt < 2 && !P; ++attempt) {
            if (!S->pipe) S->pipe = new OpsPipeline(S, S->step, S->t);
            P = S->pipe->take(S->step);
            if (!P) {  // the pipeline ran on another timeline (a failed step was repeated, a restore)
                pipeline_free(S->pipe);
                S->pipe = nullptr;
            }
        }
        require(P != nullptr, "stepper: operator pipeline out of step");
        if (P->err_code) {
            pipeline_free(S->pipe);
            S->pipe = nullptr;
            if (P->err_code == IBMGPU_ESUPPORT) {
                set_err(rep, P->err);
                return;
            }
            fail(P->err_code, P->err);
        }
        // install: the worker synchronised its stream, so the operators are complete; their
        // buffers are handed to the main stream
        for (Mat* m : {P->E, P->Q, P->QT, P->lhs2}) mat_rehome(m, c->stream);
        pcg_forget(c, S->lhs2, nullptr);
        delete S->E;
        delete S->H;
        delete S->Q;
        delete S->QT;
        delete S->lhs2;
        S->E = P->E, S->H = nullptr, S->Q = P->Q, S->QT = P->QT, S->lhs2 = P->lhs2;
        P->E = P->Q = P->QT = P->lhs2 = nullptr;
        S->bodies = P->bodies;
        S->upload_bodies();
        S->dist_stale = true;
        c->launches += P->launches;
        rep->rebuilt_operators = 1;
        if (P->rebuild) {
            hier_rehome(P->hier, c->stream);
            pcg_forget(c, nullptr, S->hier);
            delete S->hier;
            S->hier = P->hier;
            P->hier = nullptr;
            S->hier->built_at_step = S->step;
            rep->rebuilt_hierarchy = 1;
        }
        rep->t_assembly = std::chrono::duration<double>(clk::now() - tic).count();  // wait + install
    } else if (moving) {
        for (auto& b : S->bodies) b.move_to(t_new);
        try {
            NvtxRange r("refresh_body_operators");
            S->refresh_body_operators();
        } catch (const Error& e) {
            if (e.code == IBMGPU_ESUPPORT) {
                set_err(rep, e.what());
                return;
            }
            throw;
        }
        sync(c);
        rep->rebuilt_operators = 1;
        rep->t_assembly = std::chrono::duration<double>(clk::now() - tic).count();
        tic = clk::now();
        const bool freezing = t_new >= S->geom_static_after;
        if (S->force_rebuild || freezing || S->step % S->n_pc == 0) {
            NvtxRange r("build_sa_hierarchy");
            S->rebuild_hierarchy();
            S->hier->built_at_step = S->step;
            rep->rebuilt_hierarchy = 1;
            rep->t_precond = std::chrono::duration<double>(clk::now() - tic).count();
        }
    } else if (S->n_b) {
        for (auto& b : S->bodies) b.move_to(t_new);
        // geometry fixed, velocities may still change (e.g. rotating circle): refresh u_B only
        S->upload_bodies();
    }
    cudaStream_t s = c->stream;
    const int n_q = S->n_q, n_p = S->n_p;
    CK(cudaEventRecord(S->ev[0], s));
    CK(cudaMemsetAsync(S->sd.p, 0, sizeof(StepDev), s));
    // explicit terms
    nvtxRangePushA("explicit terms + rhs1");
    const GridArrays ga{S->dx.p, S->dy.p, S->del_x.p, S->del_y.p};
    k_bc_update<<<1, 1024, 0, s>>>(S->bl, ga, S->ek, S->q.p, S->bnd.p, S->bnd_n.p, &S->sd.p->bc_err);
    CK_LAUNCH(c);
    k_convection<<<blocks(n_q), 256, 0, s>>>(S->bl, ga, S->q.p, S->bnd_n.p, S->conv.p);
    CK_LAUNCH(c);
    if (S->vb_n) {
        k_visc_bc<<<blocks(S->vb_n), 256, 0, s>>>(S->vb_n, S->vb_rows.p, S->vb_off.p, S->vb_pos.p, S->vb_coeff.p,
                                                   S->bnd_n.p, S->bnd.p, S->bcn.p, S->bcnp1.p);
        CK_LAUNCH(c);
    }
    // stage 1 (single GPU: one graph launch; distributed: row-slab PCG-diag over q slabs)
    const bool distributed = S->dist_ranks > 0 || c->nccl != nullptr;
    if (distributed) S->ensure_dist1();
    PcgPlan* P1 = distributed ? nullptr : pcg_plan(c, S->A, IBMGPU_PC_DIAGONAL, nullptr);
    double* b1 = distributed ? S->b1.p : P1->b.p;
    double* qs = distributed ? S->x1.p : P1->x.p;  // q* after the solve (full on every rank)
    const double c1 = S->have_conv ? 1.5 : 1.0, c2 = S->have_conv ? 0.5 : 0.0;
    launch_spmv(c, S->L, XPlain{S->q.p},
                EpiRhs1{S->mdt.p, S->q.p, S->bcn.p, S->bcnp1.p, S->conv.p, S->conv_prev.p, 0.5 * S->nu, c1, c2, b1,
                        qs},
                s);
    CK(cudaEventRecord(S->ev[1], s));
    nvtxRangePop();
    nvtxRangePushA("solve 1 (pcg-diag)");
    ibm_solve_result r1{};
    // Single GPU: solve 1's outcome (and the boundary flux check) is read after the step's one
    // final synchronisation. Solve 2 and the projection are queued behind it right away, and the
    // host builds solve 2's plan while the GPU runs solve 1; on a failure the step reports
    // exactly what the in-order checks would and leaves the state untouched (stepper.hpp:266-276).
    const auto check_solve1 = [&] {
        if (S->sd_host->bc_err)
            fail(IBMGPU_ECUDA,
                 "boundary: prescribed velocities have nonzero net flux and no convective edge to absorb it");
        rep->solve1_iters = r1.iterations;
        rep->solve1_res = r1.rel_residual;
        rep->bc_cfl = S->max_cfl;
        if (r1.status != 0) {
            // as in the reference, the boundary state has already advanced (stepper.hpp:271)
            set_err(rep, "momentum solve did not converge (rel residual " + fmt_res(r1.rel_residual) + ")");
            return false;
        }
        return true;
    };
    if (distributed) {
        dist_solve(S->dist1, b1, qs, S->p1, &r1, nullptr);
        CK(cudaEventRecord(S->ev[2], s));
        CK(cudaMemcpyAsync(S->sd_host, S->sd.p, sizeof(StepDev), cudaMemcpyDeviceToHost, s));
        sync(c);
        nvtxRangePop();
        if (!check_solve1()) return;
    } else {
        P1->run(c, S->p1, nullptr);
        CK(cudaEventRecord(S->ev[2], s));
        nvtxRangePop();
    }
    // stage 2 (single GPU: one graph launch; distributed: row-slab PCG, dist.cu)
    nvtxRangePushA("solve 2 (rhs2 + pcg-sa)");
    if (distributed) S->ensure_dist();
    static const bool prof = std::getenv("IBMGPU_SETUP_PROFILE") != nullptr;
    const auto tp0 = clk::now();
    PcgPlan* P2 = distributed ? nullptr : pcg_plan(c, S->lhs2, IBMGPU_PC_SA, S->hier);
    if (prof)
        std::fprintf(stderr, "[step] solve-2 plan %8.3f ms\n",
                     std::chrono::duration<double, std::milli>(clk::now() - tp0).count());
    double* b2 = distributed ? S->b2.p : P2->b.p;
    double* lam = distributed ? S->x2.p : P2->x.p;
    const Bc2 bc2{S->bl, S->bnd.p, S->dx.p, S->dy.p};
    launch_spmv(c, S->QT, XPlain{qs}, EpiRhs2{bc2, n_p, 0, S->ub.p, b2}, s);
    d2d(c, lam, S->lambda.p, (size_t)S->n_lambda);
    CK(cudaEventRecord(S->ev[3], s));
    ibm_solve_result r2{};
    if (distributed) {
        dist_solve(S->dist, b2, lam, S->p2, &r2, nullptr);
        CK(cudaEventRecord(S->ev[4], s));
    } else {
        P2->run(c, S->p2, nullptr);
        CK(cudaEventRecord(S->ev[4], s));
    }
    nvtxRangePop();
    // stage 3: projection q = q* - B^N (Q lambda)
    NvtxRange proj_range("projection + invariants");
    if (S->bn_diagonal) {
        launch_spmv(c, S->Q, XPlain{lam}, EpiProjectDiag{qs, S->bn_diag.p, S->q_new.p, &S->sd.p->nonfinite}, s);
    } else {
        launch_spmv(c, S->Q, XPlain{lam}, EpiStore{S->y.p}, s);
        launch_spmv(c, S->BN, XPlain{S->y.p}, EpiProjectGen{qs, S->q_new.p, &S->sd.p->nonfinite}, s);
    }
    CK(cudaEventRecord(S->ev[5], s));
    launch_spmv(c, S->QT, XPlain{S->q_new.p},
                EpiInvariants{bc2, n_p, S->ub.p, RedSlot{S->red_part.p, S->red_cnt.p}, S->sd.p}, s);
    CK(cudaEventRecord(S->ev[6], s));
    CK(cudaMemcpyAsync(S->sd_host, S->sd.p, sizeof(StepDev), cudaMemcpyDeviceToHost, s));
    sync(c);
    if (!distributed) {
        P1->finish(c, &r1);  // already complete: reads the solve's pinned state
        P2->finish(c, &r2);
        if (!check_solve1()) return;
    }
    rep->solve2_iters = r2.iterations;
    rep->solve2_res = r2.rel_residual;
    if (r2.status != 0) {
        set_err(rep, "coupled solve did not converge (rel residual " + fmt_res(r2.rel_residual) + ")");
        return;
    }
    const StepDev& sd = *S->sd_host;
    float ms[6];
    CK(cudaEventElapsedTime(&ms[0], S->ev[0], S->ev[1]));  // explicit
    CK(cudaEventElapsedTime(&ms[1], S->ev[1], S->ev[2]));  // solve 1
    CK(cudaEventElapsedTime(&ms[2], S->ev[3], S->ev[4]));  // solve 2
    CK(cudaEventElapsedTime(&ms[3], S->ev[4], S->ev[6]));  // projection + invariants
    rep->t_explicit = ms[0] * 1e-3;
    rep->t_solve1 = ms[1] * 1e-3;
    rep->t_solve2 = ms[2] * 1e-3;
    rep->t_projection = ms[3] * 1e-3;
    S->phase_ms[0] = (float)(rep->t_assembly * 1e3);
    S->phase_ms[1] = (float)(rep->t_precond * 1e3);
    S->phase_ms[2] = ms[0];
    S->phase_ms[3] = ms[1];
    S->phase_ms[4] = ms[2];
    S->phase_ms[5] = ms[3];
    if (sd.nonfinite) {
        set_err(rep, "NaN/Inf detected in the velocity field");
        return;
    }
    rep->div_residual = std::sqrt(sd.div2) / std::max(1.0, std::sqrt(sd.bc2n));
    rep->noslip_residual = host_from_bits(sd.slip_bits) / std::max(1.0, host_from_bits(sd.ubmax_bits));
    // state update (stepper.hpp:347-355)
    std::swap(S->q, S->q_new);
    std::swap(S->conv_prev, S->conv);
    S->have_conv = true;
    d2d(c, S->lambda.p, lam, (size_t)S->n_lambda);
    S->t = t_new;
    ++S->step;
}

template <class F>
int sguard(ibmgpu_stepper* S, F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        if (S && S->c) S->c->err = e.what();
        return e.code;
    } catch (const std::invalid_argument& e) {
        if (S && S->c) S->c->err = e.what();
        return IBMGPU_EINVAL;
    } catch (const std::exception& e) {
        if (S && S->c) S->c->err = e.what();
        return IBMGPU_ECUDA;
    }
}

}  // namespace

extern "C" {

int ibmgpu_stepper_create(ibmgpu_ctx_t c, const char* cfg_path, const ibm_case_overrides* ov, ibmgpu_stepper_t* out) {
    auto* S = new ibmgpu_stepper();
    S->c = c;
    const int rc = sguard(S, [&] { stepper_setup(S, cfg_path, ov); });
    if (rc) {
        delete S;
        *out = nullptr;
        return rc;
    }
    *out = S;
    return 0;
}

}  // extern "C"

namespace {
// grid + bodies of a stepper from the reference-shaped descriptors
void desc_setup(ibmgpu_stepper* S, const ibm_grid_desc* gd, int n_bodies, const ibm_body_desc* bd) {
    require(gd && gd->nx >= 2 && gd->ny >= 2, "grid: need at least 2 cells per direction");
    require(n_bodies == 0 || bd, "stepper: null body descriptors");
    auto& g = S->g;
    g.nx = gd->nx;
    g.ny = gd->ny;
    auto take = [](const double* p, int n) {
        require(p != nullptr, "grid: null array");
        return std::vector<double>(p, p + n);
    };
    g.x_faces = take(gd->x_faces, g.nx + 1);
    g.y_faces = take(gd->y_faces, g.ny + 1);
    g.dx = take(gd->dx, g.nx);
    g.dy = take(gd->dy, g.ny);
    g.x_c = take(gd->x_c, g.nx);
    g.y_c = take(gd->y_c, g.ny);
    g.del_x = take(gd->del_x, g.nx - 1);
    g.del_y = take(gd->del_y, g.ny - 1);
    g.h_min = gd->h_min;
    g.domain = ibmhost::Rect{g.x_faces.front(), g.x_faces.back(), g.y_faces.front(), g.y_faces.back()};
    g.uniform_region = ibmhost::Rect{gd->uniform[0], gd->uniform[1], gd->uniform[2], gd->uniform[3]};
    S->cfg.domain = g.domain;
    S->cfg.uniform = g.uniform_region;
    S->cfg.h_min = g.h_min;
    S->bodies.clear();
    for (int k = 0; k < n_bodies; ++k) {
        const ibm_body_desc& d = bd[k];
        require(d.n_points > 0 && d.ref_x && d.ref_y, "body: empty point set");
        require(d.motion >= 0 && d.motion <= 3, "motion: unknown kind");
        ibmhost::Body b;
        b.ref_x.assign(d.ref_x, d.ref_x + d.n_points);
        b.ref_y.assign(d.ref_y, d.ref_y + d.n_points);
        b.x = b.ref_x;
        b.y = b.ref_y;
        b.ub_x.assign(d.n_points, 0.0);
        b.ub_y.assign(d.n_points, 0.0);
        b.center_x = d.center_x;
        b.center_y = d.center_y;
        b.ds = d.ds;
        b.motion.kind = static_cast<ibmhost::Motion>(d.motion);
        b.motion.omega = d.omega, b.motion.k = d.k, b.motion.kh = d.kh;
        b.motion.heave_omega = d.heave_omega, b.motion.heave_amp = d.heave_amp;
        b.motion.A0 = d.A0, b.motion.f = d.f, b.motion.alpha0 = d.alpha0, b.motion.beta = d.beta;
        b.motion.phase = d.phase;
        b.rotation_invariant = d.shape_rotation_invariant != 0;
        b.preamble_offset = d.preamble_offset;
        b.preamble_duration = d.preamble_duration;
        S->bodies.push_back(std::move(b));
    }
}

ibmhost::EdgeBc edge_in(const ibm_edge_bc& e) {
    ibmhost::EdgeBc o;
    o.kind = e.kind == 1 ? ibmhost::Edge::convective : ibmhost::Edge::dirichlet;
    o.u = e.u;
    o.v = e.v;
    return o;
}
}  // namespace

extern "C" {

int ibmgpu_stepper_create_from(ibmgpu_ctx_t c, const ibm_grid_desc* grid, int n_bodies, const ibm_body_desc* bodies,
                               const ibm_bc_spec* bc, double nu, const ibm_stepping_params* p, double u0, double v0,
                               ibmgpu_stepper_t* out) {
    auto* S = new ibmgpu_stepper();
    S->c = c;
    const int rc = sguard(S, [&] {
        require(bc && p && out, "stepper: null argument");
        // SteppingParams::validate (stepper.hpp:119-124)
        require(p->dt > 0.0, "stepping: dt must be positive");
        require(p->n_pc >= 1, "stepping: n_pc must be >= 1");
        validate_params(p->solve1);
        validate_params(p->solve2);
        desc_setup(S, grid, n_bodies, bodies);
        auto& cfg = S->cfg;
        cfg.bc.left = edge_in(bc->left), cfg.bc.right = edge_in(bc->right);
        cfg.bc.bottom = edge_in(bc->bottom), cfg.bc.top = edge_in(bc->top);
        cfg.bc.u_inf = bc->u_inf;
        cfg.u_inf = bc->u_inf;
        cfg.nu = nu;
        cfg.dt = p->dt;
        cfg.n_order = p->n_order;
        cfg.n_pc = p->n_pc;
        cfg.slice_rows = p->slice_rows;
        cfg.solve1.rel_tol = p->solve1.rel_tol, cfg.solve1.max_iters = p->solve1.max_iters;
        cfg.solve2.rel_tol = p->solve2.rel_tol, cfg.solve2.max_iters = p->solve2.max_iters;
        cfg.solve2.sa_theta = p->sa.theta, cfg.solve2.sa_max_coarse = p->sa.max_coarse;
        cfg.u0 = u0;
        cfg.v0 = v0;
        S->force_rebuild = p->force_rebuild != 0;
        S->sa = ibm_sa_options{p->sa.theta, p->sa.max_coarse, p->sa.max_levels > 0 ? p->sa.max_levels : 25,
                               p->sa.power_iterations >= 0 ? p->sa.power_iterations : 10, 0};
        S->sa_given = true;
        stepper_setup(S, nullptr, nullptr);
    });
    if (rc) {
        delete S;
        if (out) *out = nullptr;
        return rc;
    }
    *out = S;
    return 0;
}

int ibmgpu_operators_create(ibmgpu_ctx_t c, const ibm_grid_desc* grid, int n_bodies, const ibm_body_desc* bodies,
                            double dt, double nu, int n_order, int pin, int slice_rows, ibmgpu_stepper_t* out) {
    auto* S = new ibmgpu_stepper();
    S->c = c;
    const int rc = sguard(S, [&] {
        require(out != nullptr, "operators: null argument");
        desc_setup(S, grid, n_bodies, bodies);
        require(pin >= 0 && pin < S->g.nx * S->g.ny, "pin_row_col: bad pin index");
        S->cfg.dt = dt;
        S->cfg.nu = nu;
        S->cfg.n_order = n_order;
        S->cfg.slice_rows = slice_rows;
        S->pin = pin;
        S->ops_only = true;
        stepper_setup(S, nullptr, nullptr);
    });
    if (rc) {
        delete S;
        if (out) *out = nullptr;
        return rc;
    }
    *out = S;
    return 0;
}

int ibmgpu_stepper_destroy(ibmgpu_stepper_t S) {
    delete S;
    return 0;
}

int ibmgpu_stepper_dims(ibmgpu_stepper_t S, int* d) {
    d[0] = S->g.nx;
    d[1] = S->g.ny;
    d[2] = S->n_q;
    d[3] = S->n_p;
    d[4] = S->n_b;
    d[5] = S->n_lambda;
    d[6] = S->hier ? (int)S->hier->levels.size() : 0;
    d[7] = S->lhs2 ? S->lhs2->nnz : 0;
    return 0;
}

int ibmgpu_stepper_scalars(ibmgpu_stepper_t S, double* s6) {
    s6[0] = S->dt;
    s6[1] = S->nu;
    s6[2] = S->g.h_min;
    s6[3] = S->cfg.u_inf;
    s6[4] = S->cfg.ref_length;
    s6[5] = S->t;
    return 0;
}

int ibmgpu_stepper_advance(ibmgpu_stepper_t S, ibm_step_report* rep) {
    return sguard(S, [&] { advance(S, rep); });
}

int ibmgpu_stepper_get(ibmgpu_stepper_t S, int which, double* out, int* n) {
    return sguard(S, [&] {
        const double* src = nullptr;
        int len = 0;
        double scal[3];
        switch (which) {
            case 0: src = S->q.p, len = S->n_q; break;
            case 1: src = S->lambda.p, len = S->n_lambda; break;
            case 2: src = S->conv_prev.p, len = S->n_q; break;
            case 3: src = S->bnd.p, len = S->bl.total; break;
            case 5: src = S->lambda.p + S->n_p, len = 2 * S->n_b; break;
            case 4:
                scal[0] = S->t, scal[1] = S->step, scal[2] = S->have_conv ? 1.0 : 0.0;
                len = 3;
                break;
            default: fail(IBMGPU_EINVAL, "stepper_get: unknown field");
        }
        if (n) *n = len;
        if (!out) return;
        if (which == 4) {
            std::memcpy(out, scal, sizeof scal);
            return;
        }
        d2h(S->c, out, src, (size_t)len);
        sync(S->c);
    });
}

int ibmgpu_stepper_set(ibmgpu_stepper_t S, int which, const double* in, int n) {
    return sguard(S, [&] {
        double* dst = nullptr;
        int len = 0;
        switch (which) {
            case 0: dst = S->q.p, len = S->n_q; break;
            case 1: dst = S->lambda.p, len = S->n_lambda; break;
            case 2: dst = S->conv_prev.p, len = S->n_q; break;
            case 3: dst = S->bnd.p, len = S->bl.total; break;
            case 4: {
                require(n == 3, "stepper_set: scalars expect t, step, have_conv");
                pipeline_free(S->pipe);  // its timeline starts from the old state
                S->pipe = nullptr;
                S->t = in[0];
                S->step = (int)in[1];
                S->have_conv = in[2] != 0.0;
                // Stepper::sync_bodies_to_time (stepper.hpp:214-221)
                for (auto& b : S->bodies) b.move_to(S->t);
                if (S->geom_static_after > 0.0) {
                    S->refresh_body_operators();
                    S->rebuild_hierarchy();
                }
                sync(S->c);
                return;
            }
            default: fail(IBMGPU_EINVAL, "stepper_set: unknown field");
        }
        require(n == len, "checkpoint: grid size mismatch");
        h2d(S->c, dst, in, (size_t)len);
        sync(S->c);
    });
}

int ibmgpu_stepper_forces(ibmgpu_stepper_t S, double* out4) {
    return sguard(S, [&] {
        Ctx* c = S->c;
        double f[2] = {0.0, 0.0};
        if (S->n_b) {
            launch_elem(c, S->n_b, 1, BodyForces{S->lambda.p + S->n_p, S->n_b, RedSlot{S->red_part.p, S->red_cnt.p},
                                                 S->forces.p},
                        c->stream);
            d2h(c, f, S->forces.p, 2);
            sync(c);
        }
        const double denom = 0.5 * S->cfg.u_inf * S->cfg.u_inf * S->cfg.ref_length;
        out4[0] = f[0];
        out4[1] = f[1];
        out4[2] = f[0] / denom;
        out4[3] = f[1] / denom;
    });
}

int ibmgpu_stepper_op(ibmgpu_stepper_t S, const char* name, ibmgpu_mat_t* out) {
    return sguard(S, [&] {
        const std::string n(name);
        Mat* m = n == "L" ? S->L : n == "G" ? S->G : n == "E" ? S->E : n == "H" ? S->ensure_H() : n == "A" ? S->A
               : n == "BN" ? S->BN : n == "Q" ? S->Q : n == "QT" ? S->QT : n == "lhs2" ? S->lhs2 : nullptr;
        require(m != nullptr, "stepper_op: unknown operator " + n);
        m->borrowed = true;
        *out = m;
    });
}

int ibmgpu_stepper_hier(ibmgpu_stepper_t S, ibmgpu_hier_t* out) {
    *out = S->hier;
    return 0;
}

int ibmgpu_stepper_grid(ibmgpu_stepper_t S, int which, double* out, int* n) {
    const std::vector<double>* v[] = {&S->g.x_faces, &S->g.y_faces, &S->g.dx, &S->g.dy,
                                      &S->g.x_c,     &S->g.y_c,     &S->g.del_x, &S->g.del_y};
    if (which < 0 || which > 7) return IBMGPU_EINVAL;
    if (n) *n = (int)v[which]->size();
    if (out) std::memcpy(out, v[which]->data(), sizeof(double) * v[which]->size());
    return 0;
}

int ibmgpu_stepper_bodies(ibmgpu_stepper_t S, double* x, double* y, double* ubx, double* uby, double* ds) {
    int k = 0;
    for (const auto& b : S->bodies)
        for (int p = 0; p < b.n(); ++p, ++k) {
            x[k] = b.x[p];
            y[k] = b.y[p];
            ubx[k] = b.ub_x[p];
            uby[k] = b.ub_y[p];
            ds[k] = b.ds;
        }
    return 0;
}

int ibmgpu_stepper_vorticity(ibmgpu_stepper_t S, double* out, int* n) {
    return sguard(S, [&] {
        Ctx* c = S->c;
        const int nx = S->g.nx, ny = S->g.ny;
        const long long m = (long long)(nx - 1) * (ny - 1);
        require(m < (1ll << 31), "stepper_vorticity: grid too large");
        if (n) *n = (int)m;
        if (!out || m == 0) return;
        DBuf<double> w(c, (size_t)m);
        k_vorticity<<<(unsigned)((m + 255) / 256), 256, 0, c->stream>>>(nx, ny, S->dx.p, S->dy.p, S->del_x.p,
                                                                        S->del_y.p, S->q.p, w.p);
        CK_LAUNCH(c);
        d2h(c, out, w.p, (size_t)m);
        sync(c);
    });
}

int ibmgpu_stepper_distribute(ibmgpu_stepper_t S, int virtual_ranks, int min_dist_rows) {
    return sguard(S, [&] {
        require(virtual_ranks >= 0, "stepper_distribute: virtual_ranks must be >= 0");
        require(!S->multi_rank() || virtual_ranks <= 1, "stepper_distribute: virtual ranks need a single-rank context");
        pipeline_free(S->pipe);  // distributed steps build their operators in line
        S->pipe = nullptr;
        S->dist_ranks = S->multi_rank() ? S->c->nranks : virtual_ranks;
        S->dist_min_rows = min_dist_rows;
        S->dist_stale = true;
        dist_destroy(S->dist);
        dist_destroy(S->dist1);
        S->dist = nullptr;
        S->dist1 = nullptr;
        if (S->dist_ranks > 0) {
            S->ensure_dist1();
            S->ensure_dist();
        }
    });
}

int ibmgpu_stepper_phase_ms(ibmgpu_stepper_t S, float* ms6) {
    std::memcpy(ms6, S->phase_ms, sizeof(S->phase_ms));
    return 0;
}

}  // extern "C"
