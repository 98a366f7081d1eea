// Coefficient-space subtomogram averaging (kernel K9), see average.cu.
#pragma once

#include <cuda_runtime.h>

namespace bmb {

// sum (device complex128, reference layout, coeff_count entries) +=
//   sum_p rotate_expansion(coef_p, g_p^-1); quats: device (count x 4)
void launch_average(const float* coef, int ldc, const double* quats, int count, int L, const int* block_off,
                    const int* radial_count, double* sum, cudaStream_t s);

}  // namespace bmb
