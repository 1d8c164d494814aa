/* TEST INFRASTRUCTURE ONLY — the CPU checker for the B200 hot path.
 *
 * Plain-C restatement of the reference's sparse linear-algebra hot path
 * (/root/reference/proj/include/ibm/{sparse,krylov,amg,dense,operators,body}.hpp).
 * Each function cites the reference file:line it follows. It is pinned against the
 * reference itself (oracle/_ref/libibmref.so, built from the reference headers) and
 * against tests/golden/ fixtures generated from it (tests/test_oracle_cpu.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this.
 */
#ifndef IBM_ORACLE_H
#define IBM_ORACLE_H
#include <stddef.h>

typedef struct {
    int rows, cols, nnz;
    int* rp;
    int* ci;
    double* v;
} orc_csr;

typedef struct {
    int n_levels;
    int stalled;
    orc_csr** A;   /* per level */
    orc_csr** P;
    orc_csr** Pt;
    double** inv_diag;
    double* omega;
    orc_csr* coarse_A;
    int n_c;
    double* chol; /* row-major n_c x n_c lower factor */
} orc_hier;

orc_csr* orc_csr_new(int rows, int cols, int nnz);
orc_csr* orc_csr_from(int rows, int cols, const int* rp, const int* ci, const double* v);
void orc_csr_free(orc_csr* m);
orc_csr* orc_from_triplets(int rows, int cols, int n, const int* r, const int* c, const double* v);
void orc_spmv(const orc_csr* A, const double* x, double* y);
orc_csr* orc_transpose(const orc_csr* A);
orc_csr* orc_spmm_rows(const orc_csr* A, int r0, int r1, const orc_csr* B);
orc_csr* orc_triple(const orc_csr* A, const orc_csr* B, const orc_csr* C, int slice, long long* peak, int* slices);
orc_csr* orc_add(double a, const orc_csr* A, double b, const orc_csr* B);
orc_csr* orc_symmetrized(const orc_csr* A);
orc_csr* orc_pin(const orc_csr* A, int pin);
orc_csr* orc_concat_cols(const orc_csr* G, const orc_csr* Et);

int orc_pcg(const orc_csr* A, const double* b, const double* x0, int kind, const orc_hier* h, double rel_tol,
            int max_iters, double* x_out, int* iters, double* rel_res, int* status, double* history, int hist_cap,
            int* hist_len);

orc_hier* orc_sa_build(const orc_csr* A, double theta, int max_coarse, int max_levels, int power_its, int tail);
void orc_hier_free(orc_hier* h);
void orc_sa_apply(const orc_hier* h, const double* r, double* z);
int orc_aggregate(const orc_csr* A, double theta, int n_core, int* agg);
double orc_rho(const orc_csr* A, int iters);

double orc_delta_roma(double r, double h);
/* E (2n_b x n_q) and H (n_q x 2n_b) on a staggered grid; returns 0, or 2 when a point's
 * support leaves the uniform region (operators.hpp:251). */
int orc_assemble_EH(int nx, int ny, const double* x_faces, const double* y_faces, const double* x_c,
                    const double* y_c, const double* del_x, const double* del_y, double h_min, const double* uniform,
                    int n_b, const double* px, const double* py, const double* ds, orc_csr** E, orc_csr** H);
#endif
