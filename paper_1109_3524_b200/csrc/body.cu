// body.cu — immersed-body operators on the device.
//
//   delta_roma               body.hpp:19-28       3-point Roma kernel, exact operation order
//   assemble_interpolation   operators.hpp:264-302  E (2n_b x n_q): one thread per (point, component);
//                                                  support by binary search on the monotone node
//                                                  coordinates with the reference's exact predicate
//                                                  (d > -1.5h && d < 1.5h, d = coord - xi); rows are
//                                                  emitted j-outer/i-inner, i.e. already column-sorted
//   assemble_regularization  operators.hpp:307-342  H (n_q x 2n_b) = transpose of the ds-weighted twin
//   assemble_coupled_system  operators.hpp:408-417  Q = [G E^T], QT, lhs2 = pin(sym(QT BN Q))
// Weights use explicit non-FMA arithmetic so the sparsity (w == 0 drops) is bit-exact with the
// reference built without -march (SURVEY §7 hard part 2).
#include <cmath>
#include <cstdio>
#include <string>

#include "internal.cuh"
#include "refresh.cuh"
#include "kern.cuh"

namespace ibmgpu {

__host__ __device__ inline double delta_roma_exact(double r, double h) {
#ifdef __CUDA_ARCH__
    const double a = __ddiv_rn(fabs(r), h);
    if (a <= 0.5) return __ddiv_rn(__dadd_rn(1.0, __dsqrt_rn(__dsub_rn(1.0, __dmul_rn(__dmul_rn(3.0, a), a)))),
                                   __dmul_rn(3.0, h));
    if (a <= 1.5) {
        const double t = __dsub_rn(1.0, a);
        return __ddiv_rn(__dsub_rn(__dsub_rn(5.0, __dmul_rn(3.0, a)),
                                   __dsqrt_rn(__dsub_rn(1.0, __dmul_rn(__dmul_rn(3.0, t), t)))),
                         __dmul_rn(6.0, h));
    }
    return 0.0;
#else
    const double a = std::fabs(r) / h;
    if (a <= 0.5) return (1.0 + std::sqrt(1.0 - 3.0 * a * a)) / (3.0 * h);
    if (a <= 1.5) {
        const double t = 1.0 - a;
        return (5.0 - 3.0 * a - std::sqrt(1.0 - 3.0 * t * t)) / (6.0 * h);
    }
    return 0.0;
#endif
}

namespace {

struct DevGrid {
    int nx, ny;
    const double *x_faces, *y_faces, *x_c, *y_c, *del_x, *del_y;
    double h;
};

// support_range (operators.hpp:238-249) by binary search; returns [first,last] (empty: first>last)
__device__ void support(const double* coords, int lo, int hi, double xi, double rad, int& first, int& last) {
    // first index with coords[i] - xi > -rad
    int a = lo, b = hi + 1;
    while (a < b) {
        const int m = (a + b) >> 1;
        if (__dsub_rn(coords[m], xi) > -rad)
            b = m;
        else
            a = m + 1;
    }
    // last index with coords[i] - xi < rad
    int c = lo - 1, d = hi;
    while (c < d) {
        const int m = (c + d + 1) >> 1;
        if (__dsub_rn(coords[m], xi) < rad)
            c = m;
        else
            d = m - 1;
    }
    first = a;
    last = c;
    if (first > last) {
        first = hi + 1;
        last = hi;
    }
}

// mode 0: count, mode 1: fill. comp 0: u rows (k), comp 1: v rows (n_b + k). wsel 0: E (del), 1: H^T (ds)
__global__ void k_eh(int n_b, DevGrid g, const double* __restrict__ px, const double* __restrict__ py,
                     const double* __restrict__ ds, int wsel, int* __restrict__ cnt, const int* __restrict__ rp,
                     int* __restrict__ ci, double* __restrict__ v) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * n_b) return;
    const int comp = t / n_b, k = t % n_b;
    const int row = comp == 0 ? k : n_b + k;
    const double x = px[k], y = py[k], h = g.h, rad = __dmul_rn(1.5, h);
    const int n_u = (g.nx - 1) * g.ny;
    int i0, i1, j0, j1;
    if (comp == 0) {  // u-nodes (x_f[i_f], y_c[j])
        support(g.x_faces, 1, g.nx - 1, x, rad, i0, i1);
        support(g.y_c, 0, g.ny - 1, y, rad, j0, j1);
    } else {  // v-nodes (x_c[i], y_f[j_f])
        support(g.x_c, 0, g.nx - 1, x, rad, i0, i1);
        support(g.y_faces, 1, g.ny - 1, y, rad, j0, j1);
    }
    int n = 0;
    const int o = rp ? rp[row] : 0;
    for (int j = j0; j <= j1; ++j)
        for (int i = i0; i <= i1; ++i) {
            double dxv, dyv, scale;
            int col;
            if (comp == 0) {
                dxv = delta_roma_exact(__dsub_rn(g.x_faces[i], x), h);
                dyv = delta_roma_exact(__dsub_rn(g.y_c[j], y), h);
                scale = wsel == 0 ? g.del_x[i - 1] : ds[k];
                col = (i - 1) + j * (g.nx - 1);
            } else {
                dxv = delta_roma_exact(__dsub_rn(g.x_c[i], x), h);
                dyv = delta_roma_exact(__dsub_rn(g.y_faces[j], y), h);
                scale = wsel == 0 ? g.del_y[j - 1] : ds[k];
                col = n_u + i + (j - 1) * g.nx;
            }
            const double w = __dmul_rn(__dmul_rn(scale, dxv), dyv);
            if (w != 0.0) {
                if (ci) {
                    ci[o + n] = col;
                    v[o + n] = w;
                }
                ++n;
            }
        }
    if (cnt) cnt[row] = n;
}

__global__ void k_delta(int n, const double* __restrict__ r, double h, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = delta_roma_exact(r[i], h);
}

Mat* build_eh(Ctx* c, const DevGrid& g, int n_b, const double* px, const double* py, const double* ds, int wsel,
              int n_q) {
    const int rows = 2 * n_b;
    Mat* m = mat_new(c, rows, n_q, 0);
    DBuf<int> cnt(c, (size_t)rows + 1);
    if (rows) {
        k_eh<<<(rows + 127) / 128, 128, 0, c->stream>>>(n_b, g, px, py, ds, wsel, cnt.p, nullptr, nullptr, nullptr);
        CK_LAUNCH(c);
    }
    exclusive_scan_total(c, cnt.p, m->rp.p, rows);
    m->nnz = d2h_scalar(c, m->rp.p + rows);
    m->ci.alloc(c, (size_t)m->nnz);
    m->v.alloc(c, (size_t)m->nnz);
    if (rows) {
        k_eh<<<(rows + 127) / 128, 128, 0, c->stream>>>(n_b, g, px, py, ds, wsel, nullptr, m->rp.p, m->ci.p, m->v.p);
        CK_LAUNCH(c);
    }
    return m;
}

}  // namespace

// Host-side support check (operators.hpp:251-257): throws ESUPPORT with a "uniform" message.
void check_support(const double uniform[4], double h_min, int n_b, const double* px, const double* py) {
    const double rad = 1.5 * h_min;
    const double margin = rad * (1.0 - 1e-9);
    for (int k = 0; k < n_b; ++k) {
        const double x = px[k], y = py[k];
        if (!(x >= uniform[0] + margin && x <= uniform[1] - margin && y >= uniform[2] + margin &&
              y <= uniform[3] - margin)) {
            char buf[256];
            std::snprintf(buf, sizeof buf,
                          "body point (%f, %f) too close to the edge of the uniform grid region; delta support "
                          "would extend onto stretched cells",
                          x, y);
            fail(IBMGPU_ESUPPORT, buf);
        }
    }
}

// Device grid arrays for repeated E/H assembly (moving bodies re-use them every step).
struct GridDev {
    int nx = 0, ny = 0;
    double h = 0.0;
    DBuf<double> xf, yf, xc, yc, dlx, dly;
    void upload(Ctx* c, const ibm_grid_desc& g) {
        nx = g.nx, ny = g.ny, h = g.h_min;
        xf.alloc(c, (size_t)nx + 1);
        yf.alloc(c, (size_t)ny + 1);
        xc.alloc(c, (size_t)nx);
        yc.alloc(c, (size_t)ny);
        dlx.alloc(c, (size_t)nx - 1);
        dly.alloc(c, (size_t)ny - 1);
        h2d(c, xf.p, g.x_faces, (size_t)nx + 1);
        h2d(c, yf.p, g.y_faces, (size_t)ny + 1);
        h2d(c, xc.p, g.x_c, (size_t)nx);
        h2d(c, yc.p, g.y_c, (size_t)ny);
        h2d(c, dlx.p, g.del_x, (size_t)nx - 1);
        h2d(c, dly.p, g.del_y, (size_t)ny - 1);
    }
};

GridDev* grid_dev_new(Ctx* c, const ibm_grid_desc& g) {
    auto* gd = new GridDev();
    gd->upload(c, g);
    return gd;
}
void grid_dev_free(GridDev* g) { delete g; }

// E and (optionally) H for n_b points whose coordinates are already on the device.
void assemble_eh_dev(Ctx* c, const GridDev& gd, int n_b, const double* px, const double* py, const double* ds,
                     Mat** E, Mat** H) {
    DevGrid g{gd.nx, gd.ny, gd.xf.p, gd.yf.p, gd.xc.p, gd.yc.p, gd.dlx.p, gd.dly.p, gd.h};
    const int n_q = (gd.nx - 1) * gd.ny + gd.nx * (gd.ny - 1);
    *E = build_eh(c, g, n_b, px, py, ds, 0, n_q);
    if (H) {
        Mat* Ht = build_eh(c, g, n_b, px, py, ds, 1, n_q);
        *H = transpose(c, Ht);
        delete Ht;
    }
}

void coupled_system(Ctx* c, const Mat* G, const Mat* E, const Mat* BN, int pin_idx, int slice_rows, Mat** Q,
                    Mat** QT, Mat** lhs2, long long* peak) {
    Mat* Et = transpose(c, E);
    *Q = concat_cols(c, G, Et);
    delete Et;
    *QT = transpose(c, *Q);
    const int slice = slice_rows > 0 ? slice_rows : (*QT)->rows;
    // Full-height product without slice statistics: every row of QT B^N Q has a few dozen products,
    // so the warp-per-row Gustavson kernel (refresh.cu; same order, same rounding) does it in one
    // pass instead of expand-sort-compress chunks (C5-8192: 2.4 s -> see DESIGN §(f)4).
    Mat* raw = (slice >= (*QT)->rows && !peak) ? triple_small(c, *QT, BN, *Q)
                                               : triple_product(c, *QT, BN, *Q, std::max(slice, 1), peak, nullptr);
    Mat* sym = symmetrized(c, raw);
    delete raw;
    *lhs2 = pin(c, sym, pin_idx);
    delete sym;
}

}  // namespace ibmgpu

using namespace ibmgpu;

namespace {
template <class F>
int guard2(ibmgpu_ctx* c, F&& f) {
    try {
        f();
        return IBMGPU_OK;
    } catch (const Error& e) {
        c->err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        c->err = e.what();
        return IBMGPU_ECUDA;
    }
}
}  // namespace

extern "C" {

int ibmgpu_assemble_EH(ibmgpu_ctx_t c, const ibm_grid_desc* grid, int n_b, const double* px, const double* py,
                       const double* ds, ibmgpu_mat_t* E, ibmgpu_mat_t* H) {
    return guard2(c, [&] {
        require(grid && E && n_b >= 0, "assemble_EH: bad argument");
        check_support(grid->uniform, grid->h_min, n_b, px, py);
        GridDev gd;
        gd.upload(c, *grid);
        DBuf<double> dx(c, (size_t)std::max(n_b, 1)), dy(c, (size_t)std::max(n_b, 1)), dd(c, (size_t)std::max(n_b, 1));
        h2d(c, dx.p, px, (size_t)n_b);
        h2d(c, dy.p, py, (size_t)n_b);
        h2d(c, dd.p, ds, (size_t)n_b);
        assemble_eh_dev(c, gd, n_b, dx.p, dy.p, dd.p, E, H);
        sync(c);
    });
}

int ibmgpu_coupled_system(ibmgpu_ctx_t c, ibmgpu_mat_t G, ibmgpu_mat_t E, ibmgpu_mat_t BN, int pin_idx,
                          int slice_rows, ibmgpu_mat_t* Q, ibmgpu_mat_t* QT, ibmgpu_mat_t* lhs2, long long* peak) {
    return guard2(c, [&] {
        require(G && E && BN && Q && QT && lhs2, "coupled_system: null argument");
        require(E->cols == G->rows && BN->rows == G->rows && BN->cols == G->rows, "coupled_system: dimension mismatch");
        coupled_system(c, G, E, BN, pin_idx, slice_rows, Q, QT, lhs2, peak);
        sync(c);
    });
}

int ibmgpu_delta_roma(ibmgpu_ctx_t c, int n, const double* r, double h, double* out) {
    return guard2(c, [&] {
        DBuf<double> dr(c, (size_t)std::max(n, 1)), dout(c, (size_t)std::max(n, 1));
        h2d(c, dr.p, r, (size_t)n);
        if (n) {
            k_delta<<<(n + 255) / 256, 256, 0, c->stream>>>(n, dr.p, h, dout.p);
            CK_LAUNCH(c);
        }
        d2h(c, out, dout.p, (size_t)n);
        sync(c);
    });
}

}  // extern "C"
