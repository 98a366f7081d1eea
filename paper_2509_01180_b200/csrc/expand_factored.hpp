// Factored expansion (kernel K2f), see expand_factored.cu.
#pragma once

#include <cuda_runtime.h>

namespace bmb {

struct FactoredTables {
    int n = 0, L = 0, nr = 0, nt = 0, np = 0;
    int coeffs = 0, ntri = 0, pairs = 0;
    const double* r = nullptr;        // [nr] GL radii on [0, 1]
    const int4* samp = nullptr;       // [nt * np][nr] trilinear footprint: x0 | y0 << 10 | z0 << 20, fx, fy, fz (FP32 bits)
    const float2* tw = nullptr;       // [np/2 + 1][L + 1] (cos, -sin)(2 pi m p / np)
    const float* ptab = nullptr;      // [ntri][nt] Pbar_l^m(u_t) w_t
    const int2* tri_lm = nullptr;     // [ntri] (l, m)
    const float* radial_t = nullptr;  // [nr][pairs] c_lk j_l(lambda r_i) r_i^2 w_i 2pi/np
    const int* rowpack = nullptr;     // [coeffs] pair(l,k) << 16 | (l^2 + packed index j) per real-packed row
};

size_t factored_smem_bytes(const FactoredTables& T);
// coefficients of windows (volume win_vol[w] shifted by win_shift[3w..3w+2]) into
// out[w * ldo + row], real-packed FP32 rows; vols: raster (x fastest), vol_stride apart
// pairs (optional, else nullptr): the volumes in x-paired layout (launch_pair_volumes)
// same_volume_pairs: consecutive windows mostly come from one volume (the shift
// search), so the two-window kernel shares their footprints; false for one window
// per volume, where it would only cost occupancy
int launch_expand_factored(const FactoredTables& T, const float* vols, long long vol_stride, const int* win_vol,
                           const int* win_shift, int n_win, float* out, int ldo, cudaStream_t s,
                           const float2* pairs = nullptr, bool same_volume_pairs = true);
// x-paired copy of n_vol volumes for the trilinear gathers of the expansion:
// pairs[v][z][y][x + 1] = (v[x], v[x + 1]) for x = -1 .. n-1, zero outside the row
// (n * n * (n + 1) float2 per volume), so one 8-byte load serves both x taps
constexpr long long pair_volume_elems(int n) { return (long long)n * n * (n + 1); }
void launch_pair_volumes(const float* vols, long long vol_stride, int n_vol, int n, float2* pairs, cudaStream_t s);

// zero-padded quad copy for the shift search (kernel K2q):
// quads[v][z + M][y + M][x + M] = (v[x], v[x+1], v[x+2], v[x+3]), zero outside the
// grid, M = kQuadPad, (n + 2M)^3 float4 per volume.  Valid for |shift| <= kQuadPad.
constexpr int kQuadPad = 6;
constexpr long long quad_volume_elems(int n) { return (long long)(n + 2 * kQuadPad) * (n + 2 * kQuadPad) * (n + 2 * kQuadPad); }
void launch_quad_volumes(const float* vols, long long vol_stride, int n_vol, int n, float4* quads, cudaStream_t s);
// one CTA per pair_list entry (window a, window b, mode, 0): mode 1 / 2 = windows of
// one volume whose shifts differ by that much in x only (one 16-byte load per
// footprint row serves both), mode 0 = any two windows; b == a for a single window.
// The footprint table must flag entries that leave the window grid in bit 30.
// Returns 1 when the basis has no specialised kernel (the caller falls back;
// expand_quads_supported tells beforehand).
bool expand_quads_supported(const FactoredTables& T);
int launch_expand_quads(const FactoredTables& T, const float4* quads, const int* win_vol, const int* win_shift,
                        const int4* pair_list, int n_pairs, float* out, int ldo, cudaStream_t s);

}  // namespace bmb
