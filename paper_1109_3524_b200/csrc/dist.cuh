// dist.cuh — row-slab multi-GPU PCG (dist.cu).
#pragma once
#include "amg.cuh"
#include "internal.cuh"

struct ibmgpu_dist;

namespace ibmgpu {
using Dist = ibmgpu_dist;
void nccl_comm_init(Ctx* c, const void* id);
void nccl_comm_free(Ctx* c);
void nccl_unique_id(void* out);
Dist* dist_create(Ctx* c, Mat* A, int kind, Hier* h, const int* owner0, int virtual_ranks, int min_rows);
void dist_destroy(Dist* d);
void dist_solve(Dist* d, const double* b_full, double* x_full, const ibm_solver_params& prm, ibm_solve_result* res,
                double* hist_host);
void dist_info(const Dist* d, int* info8);
Ctx* dist_ctx(const Dist* d);
}  // namespace ibmgpu
