// stepper.cu — placeholder until the device Stepper lands (returns EINVAL).
#include "internal.cuh"
namespace ibmgpu { void ctx_free_extras(Ctx*) {} }
extern "C" {
#define NI { return IBMGPU_EINVAL; }
int ibmgpu_stepper_create(ibmgpu_ctx_t, const char*, const ibm_case_overrides*, ibmgpu_stepper_t*) NI
int ibmgpu_stepper_destroy(ibmgpu_stepper_t) { return 0; }
int ibmgpu_stepper_dims(ibmgpu_stepper_t, int*) NI
int ibmgpu_stepper_scalars(ibmgpu_stepper_t, double*) NI
int ibmgpu_stepper_advance(ibmgpu_stepper_t, ibm_step_report*) NI
int ibmgpu_stepper_get(ibmgpu_stepper_t, int, double*, int*) NI
int ibmgpu_stepper_set(ibmgpu_stepper_t, int, const double*, int) NI
int ibmgpu_stepper_forces(ibmgpu_stepper_t, double*) NI
int ibmgpu_stepper_op(ibmgpu_stepper_t, const char*, ibmgpu_mat_t*) NI
int ibmgpu_stepper_hier(ibmgpu_stepper_t, ibmgpu_hier_t*) NI
int ibmgpu_stepper_grid(ibmgpu_stepper_t, int, double*, int*) NI
int ibmgpu_stepper_bodies(ibmgpu_stepper_t, double*, double*, double*, double*, double*) NI
int ibmgpu_stepper_phase_ms(ibmgpu_stepper_t, float*) NI
}
