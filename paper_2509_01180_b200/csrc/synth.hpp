// Voxel synthesis (kernel K11), see synth.cu.
#pragma once

#include <cuda_runtime.h>

namespace bmb {

struct SynthArgs {
    const double2* coef = nullptr;  // complex coefficients, reference layout (block l, row k, column m+l)
    bool real_volume = true;        // f(k,l,-m) = (-1)^m conj f(k,l,m)
    int n = 0, L = 0;
    const int* block_off = nullptr;    // [L+1]
    const int* radial_count = nullptr; // [L+1]
    const int* pair_off = nullptr;     // [L+1]
    const double* table = nullptr;     // [pairs][row_len] c_lk j_l(lambda_lk (j-1)/n_fine), row[0] = (-1)^l row[2]
    int n_fine = 2048, row_len = 2051;
    double* out = nullptr;             // n^3, x fastest
};

int launch_synthesize(const SynthArgs& a, cudaStream_t s);

}  // namespace bmb
