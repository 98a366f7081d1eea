// Seed-grid kernel interface (kernel K6).
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace bmb {

struct SeedArgs {
    const float* coef = nullptr;   // [n_win][ldc] real-packed window coefficients
    int ldc = 0;
    const float* t_hat = nullptr;  // real-packed template coefficients
    const int* block_off = nullptr;
    const int* radial_count = nullptr;
    int rows_low = 0;              // real-packed rows of degrees <= L_low
    int L_low = 0;
    int nxi = 0;                   // N_xi(L_low)
    int na = 0, nb = 0, ng = 0;    // Euler grid (optimize.cpp:27-44)
    const double* dgrid = nullptr;   // [nb][nxi] d^l_{m,m'}(beta_j), packed blocks
    const double2* ua = nullptr;     // [na][2L+1] exp(-i m alpha_i), m = -L..L
    const double2* ug = nullptr;     // [ng][2L+1]
    const double* wedge_sqrt = nullptr;  // [grid] sqrt(clamp(1 - rho, 0.02, 2)) or null
    int max_cand = 0;
    CandState* cand = nullptr;     // [n_win][max_cand]
    int* cand_count = nullptr;     // [n_win]
    double* seed_score = nullptr;  // [n_win][max_cand] or null
    double2* xi_scratch = nullptr; // [scratch_windows][nxi] when xi does not fit in shared memory
    int scratch_windows = 0;
};

int launch_seed(const SeedArgs& a, int n_win, cudaStream_t s);
bool seed_needs_scratch(const SeedArgs& a);

}  // namespace bmb
