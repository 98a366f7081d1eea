// Fine-grained FP64 operators on the reference layouts (ops.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace bmb {

// xi_coefficients (xcorr.cpp:21-50) of n coefficient sets f (row stride ldf
// complex) against t (stride ldt, 0 = one shared set) -> n XiBlocks of degree L
int launch_xi_coefficients(const double* f, long long ldf, const double* t, long long ldt, int n,
                           const int* coef_off, const int* radial_count, int L, double* out, cudaStream_t s);
// xi_compose_right (xcorr.cpp:149-155): out = xi D(a)^T per degree <= l_limit (D: XiBlocks of D^l(a))
int launch_xi_compose_right(const double* xi, const double* D, int L, int l_limit, double* out, cudaStream_t s);
// rotate_expansion (steer.cpp:208-223): out = D f per (l, k) row
int launch_rotate_expansion(const double* f, const double* D, const int* coef_off, const int* radial_count, int L,
                            int coeffs, double* out, cudaStream_t s);
// exhaustive_baseline (optimize.cpp:523-539) of one XiBlocks kernel at band l_cut on the
// na x nb x ng Euler grid (dgrid: [nb][N_xi(l_cut)] d-blocks at beta_j); best score and
// flat index (j na + i) ng + k to host memory (stream-ordered)
int launch_exhaustive(const double* xi, const double* dgrid, int L, int l_cut, int na, int nb, int ng,
                      double* scratch, double* best_score, long long* best_flat, cudaStream_t s);
size_t exhaustive_scratch_bytes(int l_cut, int nb, int ng);

}  // namespace bmb
