// assemble.cuh — device assembly of the grid operators M, L, G (assemble.cu).
#pragma once
#include "internal.cuh"

namespace ibmgpu {

struct GridOps {
    DBuf<double> M;                 // metric diagonal (n_q)
    Mat* L = nullptr;               // diffusion (n_q x n_q)
    Mat* G = nullptr;               // gradient (n_q x n_p)
    // viscous wall couplings grouped by row (the stepper's k_visc_bc operands): rows with
    // couplings, their start offsets (n_wall_rows + 1), boundary-array position and coefficient
    int n_wall = 0, n_wall_rows = 0;
    DBuf<int> wall_rows, wall_off, wall_pos;
    DBuf<double> wall_coeff;
};

// operators.hpp:75-228 on the device. slot_off: offset of each BoundaryState array (LU, RU, LV,
// RV, BV, TV, BU, TU) in the packed boundary vector.
GridOps assemble_grid_ops(Ctx* c, int nx, int ny, const double* dx, const double* dy, const double* del_x,
                          const double* del_y, const int slot_off[8]);

}  // namespace ibmgpu
