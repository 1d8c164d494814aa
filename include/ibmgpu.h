/* ibmgpu.h — C-ABI of the B200-native IBPM sparse linear-algebra hot path.
 *
 * Drop-in boundary for the reference's in-process operator API
 * (/root/reference/proj/include/ibm/<name>.hpp; the reference is header-only C++ with no FFI,
 * so each entry point below names the C++ function/method it replaces). Plain pointers
 * and sizes only; no torch or CUDA types in any signature. `*_dev` arguments are device
 * pointers obtained from ibmgpu_vec_alloc (or any cudaMalloc'd memory on the context's
 * device); everything else is host memory.
 *
 * Error convention: every function returns 0 on success or an IBMGPU_E* code;
 * the message is in ibmgpu_last_error(ctx). Codes map 1:1 onto the reference's exceptions:
 *   IBMGPU_EINVAL   -> std::invalid_argument (sparse.hpp:39,114,227,286; krylov.hpp:22-23,55,74-82; amg.hpp:128,147)
 *   IBMGPU_ESUPPORT -> std::runtime_error whose message contains "uniform" (operators.hpp:251-256)
 *   IBMGPU_ECUDA / IBMGPU_ENCCL / IBMGPU_ENOMEM -> std::runtime_error
 * Non-convergence and breakdown are NOT errors: they travel in ibm_solve_result.status, exactly
 * as SolveStatus does (krylov.hpp:27).
 *
 * Threading: one host thread drives one context; calls are ordered on the context's stream and
 * are not reentrant (as Stepper, stepper.hpp:167-168).
 */
#ifndef IBMGPU_H
#define IBMGPU_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IBMGPU_OK 0
#define IBMGPU_EINVAL 1
#define IBMGPU_ESUPPORT 2
#define IBMGPU_ECUDA 3
#define IBMGPU_ENCCL 4
#define IBMGPU_ENOMEM 5

typedef struct ibmgpu_ctx* ibmgpu_ctx_t;
typedef struct ibmgpu_mat* ibmgpu_mat_t;
typedef struct ibmgpu_hier* ibmgpu_hier_t;
typedef struct ibmgpu_stepper* ibmgpu_stepper_t;

/* krylov.hpp:15-25 SolverParams */
typedef struct {
    double rel_tol;     /* default 1e-5 */
    int max_iters;      /* default 2000 */
    int record_history; /* history is copied to ibmgpu_pcg's history_host when non-zero */
    int check_symmetry; /* max|A-A^T| <= 1e-12 max|A| checked on the device */
} ibm_solver_params;

/* krylov.hpp:27-37 SolveResult (x stays on the device) */
typedef struct {
    int iterations;
    double rel_residual;
    int status; /* 0 converged, 1 max_iterations, 2 breakdown (SolveStatus order) */
    int history_len;
} ibm_solve_result;

/* amg.hpp:21-31 SaOptions */
typedef struct {
    double theta;
    int max_coarse;
    int max_levels;
    int power_iterations;
    int keep_fine_tail;
} ibm_sa_options;

/* Preconditioner kinds for ibmgpu_pcg (krylov.hpp:46-66, amg.hpp:237-246) */
#define IBMGPU_PC_IDENTITY 0
#define IBMGPU_PC_DIAGONAL 1
#define IBMGPU_PC_SA 2

/* ---------------------------------------------------------------- context / memory */
/* One context per GPU: owns the stream, the memory pool, cached graphs and (rank>0 runs) the
 * NCCL communicator. nranks=1, rank=0, nccl_id=NULL for single-GPU use. */
int ibmgpu_init(int device, int nranks, int rank, const void* nccl_id, ibmgpu_ctx_t* ctx);
int ibmgpu_destroy(ibmgpu_ctx_t ctx);
const char* ibmgpu_last_error(ibmgpu_ctx_t ctx);
const char* ibmgpu_version(void);
int ibmgpu_synchronize(ibmgpu_ctx_t ctx);
int ibmgpu_vec_alloc(ibmgpu_ctx_t ctx, size_t n_doubles, double** dev);
int ibmgpu_vec_free(ibmgpu_ctx_t ctx, double* dev);
int ibmgpu_h2d(ibmgpu_ctx_t ctx, double* dev, const double* host, size_t n);
int ibmgpu_d2h(ibmgpu_ctx_t ctx, double* host, const double* dev, size_t n);
/* device-side timing on the context stream: start, stop -> milliseconds */
int ibmgpu_timer_start(ibmgpu_ctx_t ctx);
int ibmgpu_timer_stop(ibmgpu_ctx_t ctx, float* ms);
/* number of this library's kernels launched on the context since init (graph nodes included) */
int ibmgpu_launch_count(ibmgpu_ctx_t ctx, long long* n);

/* ---------------------------------------------------------------- CSR (sparse.hpp:27-222) */
/* SparseMatrix(rows, cols, row_ptr, col_idx, values) (sparse.hpp:31-34): the CSR is taken as is
 * (strictly increasing columns per row assumed, as the reference's invariant). */
int ibmgpu_csr_upload(ibmgpu_ctx_t ctx, int rows, int cols, int nnz, const int* rptr, const int* cidx,
                      const double* val, ibmgpu_mat_t* out);
/* SparseMatrix::from_triplets (sparse.hpp:36-67): sort, sum duplicates, drop exact zeros */
int ibmgpu_csr_from_triplets(ibmgpu_ctx_t ctx, int rows, int cols, int n, const int* r, const int* c,
                             const double* v, ibmgpu_mat_t* out);
int ibmgpu_csr_info(ibmgpu_mat_t m, int* rows, int* cols, int* nnz);
int ibmgpu_csr_download(ibmgpu_ctx_t ctx, ibmgpu_mat_t m, int* rptr, int* cidx, double* val);
int ibmgpu_csr_destroy(ibmgpu_ctx_t ctx, ibmgpu_mat_t m);
/* bytes one SpMV moves in the matrix's device format (plan arrays as stored, x read once, y
 * written once) — the format-actual counterpart of the reference-CSR algorithmic bytes;
 * kind: 0 SELL-32, 2 SELL-32-sigma, 3 stencil/DIA hybrid, else CSR-adaptive; +16 when the slices
 * carry 16-bit column codes */
int ibmgpu_csr_format_bytes(ibmgpu_ctx_t ctx, ibmgpu_mat_t m, long long* bytes, int* kind);
/* SparseMatrix::spmv_into (sparse.hpp:101-110): y = A x, device pointers */
int ibmgpu_spmv(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, const double* x_dev, double* y_dev);
/* SparseMatrix::spmv (sparse.hpp:112-118) with host vectors (H2D, SpMV, D2H) */
int ibmgpu_spmv_host(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, const double* x_host, double* y_host);
/* benchmark helper (no reference counterpart): `reps` back-to-back y = A x launches captured in one
 * CUDA graph (programmatic dependent launch between them), timed warm with events; *us_per_launch */
int ibmgpu_spmv_timed(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, const double* x_dev, double* y_dev, int reps,
                      double* us_per_launch);
/* SparseMatrix::transpose (sparse.hpp:120-138) */
int ibmgpu_transpose(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, ibmgpu_mat_t* out);
/* spmm (sparse.hpp:270) — Gustavson order, cancelled entries kept */
int ibmgpu_spmm(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, ibmgpu_mat_t B, ibmgpu_mat_t* out);
/* sliced_triple_product (sparse.hpp:282-314) */
int ibmgpu_triple_product(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, ibmgpu_mat_t B, ibmgpu_mat_t C, int max_slice_rows,
                          ibmgpu_mat_t* out, long long* peak_slice_nnz, int* slices);
/* add_sparse (sparse.hpp:317-329) */
int ibmgpu_add(ibmgpu_ctx_t ctx, double a, ibmgpu_mat_t A, double b, ibmgpu_mat_t B, ibmgpu_mat_t* out);
/* symmetrized (sparse.hpp:351-353) */
int ibmgpu_symmetrized(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, ibmgpu_mat_t* out);
/* pin_row_col (operators.hpp:381-392) */
int ibmgpu_pin(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, int pin, ibmgpu_mat_t* out);
/* is_symmetric (sparse.hpp:331-348) */
int ibmgpu_is_symmetric(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, double tol, int* result);
/* scaled / scaled_rows / scaled_cols (sparse.hpp:141-161); d_host may be NULL for `scaled` */
int ibmgpu_scale(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, int mode /*0 scalar,1 rows,2 cols*/, double a,
                 const double* d_host, ibmgpu_mat_t* out);

/* ---------------------------------------------------------------- solvers */
/* pcg (krylov.hpp:70-136) / cg (:138). x_dev holds x0 on entry (NULL-equivalent: zeros) and x on
 * exit. precond: IBMGPU_PC_*; hier required for IBMGPU_PC_SA. history_host (optional) receives
 * params.max_iters+1 relative residuals at most. */
int ibmgpu_pcg(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, int precond, ibmgpu_hier_t hier, const double* b_dev,
               double* x_dev, const ibm_solver_params* params, ibm_solve_result* result, double* history_host);
/* build_sa_hierarchy (amg.hpp:127-194), entirely on the device */
int ibmgpu_sa_build(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, const ibm_sa_options* opts, ibmgpu_hier_t* out);
int ibmgpu_sa_destroy(ibmgpu_ctx_t ctx, ibmgpu_hier_t h);
/* sa_apply (amg.hpp:231): one V(1,1) cycle z = M^{-1} r */
int ibmgpu_sa_apply(ibmgpu_ctx_t ctx, ibmgpu_hier_t h, const double* r_dev, double* z_dev);
/* amg_solve (amg.hpp:250-280) */
int ibmgpu_amg_solve(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, ibmgpu_hier_t h, const double* b_dev, double* x_dev,
                     const ibm_solver_params* params, ibm_solve_result* result);
/* SaHierarchy inspection (amg.hpp:33-52): levels, coarsening_stalled, coarse size */
int ibmgpu_hier_info(ibmgpu_hier_t h, int* n_levels, int* stalled, int* coarse_rows);
/* device-only (no reference counterpart): how many of the last levels the V-cycle applies as one
 * folded dense operator, and its dimension (0 and coarse_rows when nothing is folded; fold.cu) */
int ibmgpu_hier_folded(ibmgpu_hier_t h, int* n_fold, int* dense_rows);
/* device-only: the level-0 grid transfers applied through the pressure stencil (xfer.cuh) instead
 * of streaming the explicit P and P^T — the same operator as amg.hpp:163-183, rounded differently.
 * mode 0 turns them off, 1 on (if level 0 qualifies), -1 only queries; *active gets the state.
 * PCG plans capture the state when they are made. */
int ibmgpu_hier_transfers(ibmgpu_ctx_t ctx, ibmgpu_hier_t h, int mode, int* active);
/* level l: borrowed handles (valid while h lives) and omega; l == n_levels gives coarse_A in *A */
int ibmgpu_hier_level(ibmgpu_hier_t h, int l, ibmgpu_mat_t* A, ibmgpu_mat_t* P, ibmgpu_mat_t* Pt, double* omega);
/* aggregate ids of level l's core rows (sa_detail::aggregate, amg.hpp:79-107); returns count */
int ibmgpu_hier_aggregates(ibmgpu_ctx_t ctx, ibmgpu_hier_t h, int l, int* agg_host, int* n_agg);
/* standalone strength graph + greedy aggregation (amg.hpp:110-123, :79-107) */
int ibmgpu_aggregate(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, double theta, int n_core, int* agg_host, int* n_agg);

/* ---------------------------------------------------------------- body operators */
/* Staggered-grid description (grid.hpp:29-49). Arrays are host pointers; lengths nx+1, ny+1,
 * nx, ny, nx, ny, nx-1, ny-1. uniform = {x0, x1, y0, y1} of the snapped uniform region. */
typedef struct {
    int nx, ny;
    const double *x_faces, *y_faces, *dx, *dy, *x_c, *y_c, *del_x, *del_y;
    double h_min;
    double uniform[4];
} ibm_grid_desc;

/* assemble_interpolation / assemble_regularization (operators.hpp:264-342) on the device.
 * ds: per-point arc quadrature (LagrangianBody::ds of the owning body). H may be NULL. */
int ibmgpu_assemble_EH(ibmgpu_ctx_t ctx, const ibm_grid_desc* grid, int n_b, const double* px, const double* py,
                       const double* ds, ibmgpu_mat_t* E, ibmgpu_mat_t* H);
/* assemble_coupled_system (operators.hpp:408-417): Q = [G E^T], QT = Q^T, lhs2 = pin(sym(QT BN Q)) */
int ibmgpu_coupled_system(ibmgpu_ctx_t ctx, ibmgpu_mat_t G, ibmgpu_mat_t E, ibmgpu_mat_t BN, int pin,
                          int slice_rows, ibmgpu_mat_t* Q, ibmgpu_mat_t* QT, ibmgpu_mat_t* lhs2,
                          long long* peak_slice_nnz);
/* delta_roma (body.hpp:19-28), evaluated on the device for n arguments */
int ibmgpu_delta_roma(ibmgpu_ctx_t ctx, int n, const double* r_host, double h, double* out_host);

/* ---------------------------------------------------------------- case + stepper */
/* The stepper reproduces Stepper (stepper.hpp:169-370) with every vector and operator resident in
 * HBM. The case is read from a config file in the reference's format (config.hpp:236-355); the
 * grid, bodies, M/L/G are assembled on the host (grid.hpp, body.hpp, operators.hpp:75-228),
 * everything else on the device. Overrides <= 0 are ignored. */
typedef struct {
    double h_min;      /* grid.h_min override */
    double dt;         /* time.dt override */
    int n_pc;          /* stepping.n_pc override */
    int force_rebuild; /* SteppingParams::force_rebuild */
    int slice_rows;    /* stepping.slice_rows override */
} ibm_case_overrides;

/* StepReport (stepper.hpp:128-145) */
typedef struct {
    int ok;
    int solve1_iters, solve2_iters;
    double solve1_res, solve2_res;
    double div_residual, noslip_residual;
    int rebuilt_hierarchy, rebuilt_operators;
    double bc_cfl;
    double t_assembly, t_precond, t_explicit, t_solve1, t_solve2, t_projection; /* seconds */
    char message[256];
} ibm_step_report;

int ibmgpu_stepper_create(ibmgpu_ctx_t ctx, const char* cfg_path, const ibm_case_overrides* ov,
                          ibmgpu_stepper_t* out);
int ibmgpu_stepper_destroy(ibmgpu_stepper_t st);
/* dims: nx, ny, n_q, n_p, n_b, n_lambda, n_levels, nnz(lhs2) */
int ibmgpu_stepper_dims(ibmgpu_stepper_t st, int* dims8);
/* scalars: dt, nu, h_min, u_inf, ref_length, t */
int ibmgpu_stepper_scalars(ibmgpu_stepper_t st, double* s6);
/* Stepper::advance (stepper.hpp:231-356) */
int ibmgpu_stepper_advance(ibmgpu_stepper_t st, ibm_step_report* rep);
/* state download: which 0 q, 1 lambda, 2 conv_prev, 3 boundary arrays (BoundaryState order),
 * 4 scalars {t, step_index, have_conv_prev}, 5 f~ (the 2 n_b force entries of lambda);
 * returns the length in *n (pass out=NULL to query). */
int ibmgpu_stepper_get(ibmgpu_stepper_t st, int which, double* out, int* n);
/* state upload (checkpoint restore, io.hpp:112-145): same `which` codes */
int ibmgpu_stepper_set(ibmgpu_stepper_t st, int which, const double* in, int n);
/* compute_force_coefficients (diagnostics.hpp:26-38) on the device: out {fx, fy, cd, cl} */
int ibmgpu_stepper_forces(ibmgpu_stepper_t st, double* out4);
/* borrowed operator handle by name: "L","G","E","H","A","BN","Q","QT","lhs2" */
int ibmgpu_stepper_op(ibmgpu_stepper_t st, const char* name, ibmgpu_mat_t* out);
int ibmgpu_stepper_hier(ibmgpu_stepper_t st, ibmgpu_hier_t* out);
/* host grid arrays (which: 0 x_faces,1 y_faces,2 dx,3 dy,4 x_c,5 y_c,6 del_x,7 del_y) */
int ibmgpu_stepper_grid(ibmgpu_stepper_t st, int which, double* out, int* n);
/* body points at the current time: x, y, ub_x, ub_y, ds (each n_b) */
int ibmgpu_stepper_bodies(ibmgpu_stepper_t st, double* x, double* y, double* ubx, double* uby, double* ds);
/* compute_vorticity (diagnostics.hpp:42-56) on the device: (nx-1)(ny-1) values at the interior
 * vertices, row-major in j; *n receives the length (out may be NULL to query) */
int ibmgpu_stepper_vorticity(ibmgpu_stepper_t st, double* out, int* n);
/* time the last advance() spent in each device phase, from CUDA events (ms) */
int ibmgpu_stepper_phase_ms(ibmgpu_stepper_t st, float* ms6);

/* ---------------------------------------------------------------- reference-shaped construction
 * Stepper(grid, bodies, bc, nu, params, u0, v0) (stepper.hpp:171-195) and assemble_operators
 * (operators.hpp:420-442) from in-memory objects instead of a case file; the C++ shim
 * (ibm_b200.hpp) builds these descriptors from its StaggeredGrid / LagrangianBody / BcSpec /
 * SteppingParams, the reference's own types. */
typedef struct {
    int kind; /* BcKind: 0 dirichlet, 1 convective (boundary.hpp:15-21) */
    double u, v;
} ibm_edge_bc;
typedef struct {
    ibm_edge_bc left, right, bottom, top;
    double u_inf;
} ibm_bc_spec; /* BcSpec (boundary.hpp:23-32) */
typedef struct {
    int n_points;
    const double *ref_x, *ref_y; /* shape about the centroid (LagrangianBody::ref_x/ref_y) */
    double center_x, center_y, ds;
    int motion; /* MotionKind: 0 stationary, 1 rotating, 2 heaving, 3 flapping (body.hpp:30-63) */
    double omega, k, kh, heave_omega, heave_amp, A0, f, alpha0, beta, phase;
    int shape_rotation_invariant;
    double preamble_offset, preamble_duration;
} ibm_body_desc; /* LagrangianBody (body.hpp:85-148) */
typedef struct {
    double dt;
    int n_order, n_pc, force_rebuild, slice_rows;
    ibm_solver_params solve1, solve2;
    ibm_sa_options sa;
} ibm_stepping_params; /* SteppingParams (stepper.hpp:110-125) */

/* Stepper::Stepper (stepper.hpp:171-195). The grid's domain is its first/last faces. */
int ibmgpu_stepper_create_from(ibmgpu_ctx_t ctx, const ibm_grid_desc* grid, int n_bodies,
                               const ibm_body_desc* bodies, const ibm_bc_spec* bc, double nu,
                               const ibm_stepping_params* params, double u0, double v0, ibmgpu_stepper_t* out);
/* assemble_operators (operators.hpp:420-442): the returned stepper handle holds only the operator
 * set (read with ibmgpu_stepper_op; advance is refused) */
int ibmgpu_operators_create(ibmgpu_ctx_t ctx, const ibm_grid_desc* grid, int n_bodies, const ibm_body_desc* bodies,
                            double dt, double nu, int n_order, int pin, int slice_rows, ibmgpu_stepper_t* out);

/* pcg (krylov.hpp:70-136) with a caller-supplied preconditioner — the reference's polymorphic
 * Preconditioner::apply (krylov.hpp:39-43). apply(user, n, r_dev, z_dev) must write z = M^{-1} r
 * (device pointers, context stream order; it may launch its own kernels or copy through the
 * host) and return 0, or nonzero to abort the solve with IBMGPU_EINVAL. */
typedef int (*ibmgpu_apply_fn)(void* user, int n, const double* r_dev, double* z_dev);
int ibmgpu_pcg_callback(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, ibmgpu_apply_fn apply, void* user, const double* b_dev,
                        double* x_inout_dev, const ibm_solver_params* params, ibm_solve_result* result,
                        double* history_host);

/* host-only builders (no CUDA; the reference's grid.hpp / body.hpp / config.hpp functions).
 * Two-phase: call with NULL outputs to get the sizes. err: message on failure. */
/* build_stretched_grid (grid.hpp:148-192): packed = x_faces, y_faces, dx, dy, x_c, y_c, del_x,
 * del_y (lengths nx+1, ny+1, nx, ny, nx, ny, nx-1, ny-1); uniform4 = snapped uniform region */
int ibmgpu_host_grid(const double domain[4], const double uniform[4], double h_min, const double ratio[4], int* nx,
                     int* ny, double* packed, double* uniform4, char* err, int err_cap);
/* discretize_circle / discretize_ellipse (body.hpp:151-261) */
int ibmgpu_host_circle(double cx, double cy, double diameter, double h, int* n, double* ref_x, double* ref_y,
                       double* ds, char* err, int err_cap);
int ibmgpu_host_ellipse(double cx, double cy, double chord, double thickness_ratio, double h, int n_override, int* n,
                        double* ref_x, double* ref_y, double* ds, char* err, int err_cap);
/* the scalar part of CaseConfig (config.hpp:54-95) as parse_config reads it */
typedef struct {
    int kind; /* SolverKind: 0 cg, 1 pcg-diag, 2 pcg-sa, 3 amg */
    double rel_tol;
    int max_iters;
    double sa_theta;
    int sa_max_coarse;
} ibm_solver_config;
typedef struct {
    double domain[4], uniform[4], h_min, ratio[4];
    double nu, re, u_inf, ref_length, u0, v0, dt;
    int n_steps, n_out, checkpoint_every, n_pc, n_order, slice_rows, n_bodies;
    ibm_bc_spec bc;
    ibm_solver_config solve1, solve2;
    char out_dir[512];
} ibm_case_config;
int ibmgpu_host_case_config(const char* cfg_path, ibm_case_config* out, char* err, int err_cap);
/* build_bodies (config.hpp:358-385): descs[k].ref_x/ref_y point into xy (2 * n_points_total) */
int ibmgpu_host_case_bodies(const char* cfg_path, int* n_bodies, int* n_points_total, ibm_body_desc* descs,
                            double* xy, char* err, int err_cap);

/* ---------------------------------------------------------------- host-only case setup
 * The host half of case loading (config.hpp parse_config, grid.hpp build_stretched_grid,
 * body.hpp discretisation + move_to(0), operators.hpp metric / diffusion / gradient). No CUDA
 * calls: usable without a GPU (CPU parity tests). Arrays by name: "x_faces","y_faces","dx","dy",
 * "x_c","y_c","del_x","del_y","uniform","M","body_x","body_y","body_ub_x","body_ub_y","body_ds",
 * "visc_bc" (row, slot, idx, coeff quadruples), "boundary"; matrices: "L","G". dims8 as
 * ibmgpu_stepper_dims (levels/nnz zero). */
typedef struct ibmgpu_hostcase* ibmgpu_hostcase_t;
int ibmgpu_hostcase_open(const char* cfg_path, const ibm_case_overrides* ov, ibmgpu_hostcase_t* out, int* dims8,
                         char* err, int err_cap);
int ibmgpu_hostcase_array(ibmgpu_hostcase_t h, const char* name, double* out, int* n);
int ibmgpu_hostcase_csr(ibmgpu_hostcase_t h, const char* name, int* rows, int* cols, int* nnz, int* rptr, int* cidx,
                        double* val);
/* move every body to time t (LagrangianBody::move_to, body.hpp:125-148) */
int ibmgpu_hostcase_move(ibmgpu_hostcase_t h, double t);
int ibmgpu_hostcase_free(ibmgpu_hostcase_t h);

/* ---------------------------------------------------------------- row-slab multi-GPU
 * The reference is single-address-space; these entries are the distributed form of
 * pcg (krylov.hpp:70-136) with the SaPreconditioner (amg.hpp:237-246). Every rank passes the FULL
 * matrix and hierarchy (built identically everywhere) and the row owner of every row; each rank
 * keeps its owned rows with halo-extended columns, fine levels distributed, levels below
 * min_dist_rows replicated. Context with nranks > 1: NCCL between processes (ibmgpu_init with the
 * id from ibmgpu_nccl_unique_id on rank 0). Single-rank context: virtual_ranks > 1 emulates the
 * whole partition on this GPU (loopback halos), for parity tests of the decomposition; if that
 * single-rank context also has an NCCL communicator (nccl id given), the loopback halos travel as
 * ncclSend/ncclRecv pairs to self, so the NCCL p2p path runs on one GPU. */
typedef struct ibmgpu_dist* ibmgpu_dist_t;
int ibmgpu_nccl_unique_id(void* id128);
int ibmgpu_dist_create(ibmgpu_ctx_t ctx, ibmgpu_mat_t A, int precond, ibmgpu_hier_t hier, const int* owner_host,
                       int virtual_ranks, int min_dist_rows, ibmgpu_dist_t* out);
/* info: nranks, distributed levels, loopback (0 NCCL, 1 device copies, 2 NCCL p2p to self),
 * own rows (first local rank), its A halo, local ranks,
 * hierarchy levels, SpMV kind of the local A */
int ibmgpu_dist_info(ibmgpu_dist_t d, int* info8);
/* b_dev, x_dev: full-length device vectors on every rank; x holds x0 on entry (owned rows used) and
 * the full solution on exit on every rank */
int ibmgpu_dist_pcg(ibmgpu_dist_t d, const double* b_dev, double* x_dev, const ibm_solver_params* params,
                    ibm_solve_result* result, double* history_host);
int ibmgpu_dist_destroy(ibmgpu_dist_t d);
/* Run the stepper's modified-Poisson solve (stepper.hpp:294-313) row-slab distributed: lambda rows
 * by ibmgpu_partition_lambda, re-planned whenever the body operators or the hierarchy are rebuilt.
 * Multi-rank context: all ctx ranks (virtual_ranks ignored). Single-rank context: virtual_ranks
 * emulated ranks (0 switches back to the single-GPU graph solve). */
int ibmgpu_stepper_distribute(ibmgpu_stepper_t st, int virtual_ranks, int min_dist_rows);

/* host-only halo planning (no CUDA): rank `rank`'s part of an rows x cols CSR under row/column
 * owners. sizes6: own rows, own input entries, halo entries, local nnz, send entries, nranks. */
typedef struct ibmgpu_distplan* ibmgpu_distplan_t;
int ibmgpu_distplan_build(int rows, int cols, const int* rptr, const int* cidx, const double* val,
                          const int* row_owner, const int* col_owner, int rank, int nranks, ibmgpu_distplan_t* out);
int ibmgpu_distplan_sizes(ibmgpu_distplan_t p, int* sizes6);
/* any output may be NULL: rows[own rows], own[own inputs], rptr[own rows+1], cidx/val[local nnz]
 * (extended numbering), recv_off[nranks+1], halo[halo] (global ids), send_off[nranks+1],
 * send_idx[send entries] (owned-local indices) */
int ibmgpu_distplan_get(ibmgpu_distplan_t p, int* rows, int* own, int* rptr, int* cidx, double* val, int* recv_off,
                        int* halo, int* send_off, int* send_idx);
int ibmgpu_distplan_free(ibmgpu_distplan_t p);
/* row owners of the coupled system: pressure rows by balanced j-slabs, the two force rows of body
 * point k by the slab of body_cell_j[k] */
int ibmgpu_partition_lambda(int nx, int ny, int n_b, const int* body_cell_j, int nranks, int* owner);
/* owners of level l+1 (n_agg aggregates, then the identity tail) from level l's: an aggregate
 * goes to the owner of its lowest-index member (amg.hpp:79-107 numbering, :166-178 tail) */
int ibmgpu_partition_coarse(int n_core, const int* agg, int n_agg, int tail, const int* owner_fine, int* owner_coarse);

#ifdef __cplusplus
}
#endif
#endif /* IBMGPU_H */
