// Device data structures and kernel launchers of the alignment hot path.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace bmb {

constexpr int kMaxL = 48;  // largest band limit the device tables support
constexpr int kMaxBands = 16;  // bands of one marching schedule (bm_align_config.bands)

// Per-band evaluation tables (host-built, device-resident).  The half-plane
// items (m,m') of degree <= L (m > 0, or m = 0 and m' >= 0) are sorted by
// their first degree l0 = max(|m|,|m'|) and packed in groups of 32 lanes;
// entry (group g, step s, lane j) refers to item 32g+j at degree l0 + s and
// lives at row (row_off[g] + s), column j of every [rows x 32] table.
struct BandTables {
    int L = 0;
    int n_items = 0;
    int n_groups = 0;
    int rows = 0;                    // sum of group lengths
    const int* row_off = nullptr;    // [n_groups + 1]
    const char2* item_mm = nullptr;  // [n_groups*32] (m, m'), m >= |m'|; padded lanes (0, 0) with len 0
    const char2* item_pm = nullptr;  // [n_groups*32] half-plane partner (m', m) or (-m', -m)
    const float2* item_w = nullptr;  // [n_groups*32] (weight of A, sign * weight of B; 0 if self-paired)
    const int* item_len = nullptr;   // [n_groups*32] steps of the item (0 for padding)
    const float* bfac = nullptr;     // [n_groups*32] sign * sqrt_binom of the border closed form
    const int* bexp = nullptr;       // [n_groups*32] packed exponents: a | p << 8 (cos^a sin^p)
    const float4* PQR = nullptr;     // [rows*32] (P, Q, R, 0): t1 = P cos b + Q,
                                     // t1' = -P sin b, t1'' = -P cos b, t2 = R
    const int* item_of = nullptr;    // [(2L+1)^2] 2 item + slot of each half-plane entry (m, m'), else -1
    const int2* at_desc = nullptr;   // [rows*32] layout position descriptors (tables.hpp)
    const int* out_pos = nullptr;    // [(2L+1)^2] 2 ((row_off[g] - m_item) 32 + lane) + slot: + 64 l = 2 at + slot
    const float4* wedge = nullptr;   // [rows*32] wedge-power kernel entries (A, B) (or null)
    const float4* wedge_side = nullptr;  // [rows*32] the same composed with D(K^-1)^T (side kernels)
};

// Per-context constants used by the kernels.
struct Geometry {
    int n = 0;
    int l_max = 0;
    int coeffs = 0;       // C (real-packed rows)
    int support = 0;      // V
    int m_pad = 0, k_pad = 0;
    const int* block_off = nullptr;   // [l_max+1] real-packed offset of degree l
    const int* radial_count = nullptr;  // [l_max+1]
    const float* row_weight = nullptr;  // [coeffs] 1 for m = 0 rows, 2 for m > 0 (Parseval)
    const int4* row_lkm = nullptr;      // [coeffs] (l, k, m, part) of each real-packed row
};

// Candidate state of the device Newton state machine (one per candidate).
struct CandState {
    double g[4];        // global iterate (quaternion w,x,y,z)
    double anchor[4];   // chart anchor
    double best_g[4];
    double best_score;
    double score;       // final unanchored score at the top band
    int anchored;
    int anchor_limit;
    int diverged;
    int band_converged;
    int evals;
    int active;         // 0 for empty candidate slots
};

struct WindowOutcome {
    int particle;
    int shift[3];
    int valid;
    int n_cand;
    int best_cand;
    int converged;
    double raw_score;
    double norm_score;
    double sub_norm;
    double quat[4];
    long long evals;
    long long band_evals[kMaxBands];  // by band index; the seed grid counts at band 0
};

struct RefineParams {
    int band;
    int newton_max_iter;
    double grad_tol;
    double accept_tol;    // relative acceptance slack (reference: 1e-12)
    double step_damping;
    double koffset[4];    // ZYZ(0, pi/2, 0)
    int max_cand;
    int has_wedge;
    int first_band;
    int band_index;       // position of band in the schedule (per-band counters)
};

// ---- launchers (stream-ordered, no host sync)
void launch_gather_windows(const float* vols, long long vol_stride, const int* win_vol,
                           const int* win_shift, int n_win, const float* vol_scale,
                           const int* voxels, int support, int k_pad, int n, __half* b_hi,
                           __half* b_lo, float* col_scale, cudaStream_t s);
void launch_absmax_scale(const float* vols, int count, long long stride, float* scale,
                         cudaStream_t s);
void launch_window_norms(const float* coef, int n_win, int ldc, const Geometry& geo,
                         double* norm, cudaStream_t s);  // sqrt(sum |f_klm|^2) over all m
void launch_from_complex(const double* in, int count, const Geometry& geo, float* out, int ldo,
                         cudaStream_t s);
void launch_to_complex(const float* coef, int n_win, int ldc, const Geometry& geo, double* out,
                       cudaStream_t s);

}  // namespace bmb
