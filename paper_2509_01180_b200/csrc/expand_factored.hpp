// Factored expansion (kernel K2f), see expand_factored.cu.
#pragma once

#include <cuda_runtime.h>

namespace bmb {

struct FactoredTables {
    int n = 0, L = 0, nr = 0, nt = 0, np = 0;
    int coeffs = 0, ntri = 0;
    const double* r = nullptr;     // [nr] GL radii on [0, 1]
    const double* st = nullptr;    // [nt] sin theta_t
    const double* u = nullptr;     // [nt] cos theta_t (GL nodes)
    const double* cphi = nullptr;  // [np] cos phi_p
    const double* sphi = nullptr;  // [np] sin phi_p
    const float2* tw = nullptr;    // [np/2 + 1][L + 1] (cos, -sin)(2 pi m p / np)
    const float* ptab = nullptr;   // [ntri][nt] Pbar_l^m(u_t) w_t
    const int2* tri_lm = nullptr;  // [ntri] (l, m)
    const float* radial = nullptr; // [pairs][nr]
    const int4* rowmap = nullptr;  // [coeffs] (tri(l,m), part, pair(l,k), 0) per real-packed row
};

size_t factored_smem_bytes(const FactoredTables& T);
// coefficients of windows (volume win_vol[w] shifted by win_shift[3w..3w+2]) into
// out[w * ldo + row], real-packed FP32 rows
// vols: raster (x fastest) or, bricked = true, the 4x4x4-brick layout of launch_to_bricks
int launch_expand_factored(const FactoredTables& T, const float* vols, long long vol_stride, bool bricked,
                           const int* win_vol, const int* win_shift, int n_win, float* out, int ldo, cudaStream_t s);
// raster volumes (in_stride apart) -> 4x4x4 bricks (n % 4 == 0), n^3 apart
void launch_to_bricks(const float* in, long long in_stride, int count, float* out, int n, cudaStream_t s);

}  // namespace bmb
