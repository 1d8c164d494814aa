// pcg.cuh — PCG plan (device state, work vectors, captured graph) shared with the stepper.
#pragma once
#include "amg.cuh"
#include "internal.cuh"

namespace ibmgpu {

// Device-resident scalars of one solve (krylov.hpp:91-135 locals + SolveResult fields).
struct PcgState {
    double bnorm, rel, rel_tol, rz, pAp, alpha, beta;
    int it, max_iters, status, done, iterations, zero_x, hist_len, use_cond;
    double* hist;
    cudaGraphConditionalHandle cond;
};

struct PcgPlan {
    Mat* A;
    int kind;
    Hier* h;
    long long hier_id = 0;
    DBuf<double> b, x, r, z, p, Ap, invd;
    DBuf<PcgState> st;
    DBuf<double> partials;
    DBuf<unsigned> counter;
    PcgState* host_st = nullptr;  // pinned (recycled slot, pcg.cu pin_acquire)
    cudaStream_t last_stream = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphConditionalHandle cond = 0;
    int kernels_init = 0, kernels_iter = 0;
    bool last_eager = false;

    PcgPlan(Ctx* c, Mat* A, int kind, Hier* h);
    ~PcgPlan();
    void enqueue_init(Ctx* c, cudaStream_t s);
    void enqueue_body(Ctx* c, cudaStream_t s);
    void build_graph(Ctx* c);
    // launch the solve on b -> x (the plan's own buffers); asynchronous
    void run(Ctx* c, const ibm_solver_params& prm, double* hist_dev);
    // wait and report
    void finish(Ctx* c, ibm_solve_result* res);
};

PcgPlan* pcg_plan(Ctx* c, Mat* A, int kind, Hier* h);
void pcg_forget(Ctx* c, const Mat* A, const Hier* h);
void pcg_cache_free(Ctx* c);
void validate_params(const ibm_solver_params& p);
void pcg_callback(Ctx* c, Mat* A, ibmgpu_apply_fn apply, void* user, const double* b, double* x,
                  const ibm_solver_params& prm, ibm_solve_result* res, double* hist_host);
void pcg_solve(Ctx* c, Mat* A, int kind, Hier* h, const double* b, double* x, const ibm_solver_params& prm,
               ibm_solve_result* res, double* hist_host);

}  // namespace ibmgpu
