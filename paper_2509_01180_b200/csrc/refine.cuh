// Refinement kernel interface (kernels K4/K5/K7).
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace bmb {

struct RefineArgs {
    BandTables T;                   // tables of this band
    const int* row_group = nullptr;  // [T.rows] group of each table row
    const float* coef = nullptr;    // [n_win][ldc] real-packed window coefficients
    int ldc = 0;
    const float* t_hat = nullptr;
    const int* block_off = nullptr;
    const int* radial_count = nullptr;
    int rows_band = 0;              // real-packed rows of degrees <= band
    const int* cand_count = nullptr;
    CandState* cand = nullptr;
    int max_cand = 0;
    int n_win = 0;
    int batch = 1;                  // windows per CTA batch (refine_batch)
    int* win_counter = nullptr;     // zeroed before launch
    float* scratch = nullptr;       // per resident warp: anchored-chart kernels
    long long scratch_per_warp = 0; // floats
    RefineParams prm;
    int last_band = 0;
    // outcome (last band only)
    const double* sub_norm = nullptr;
    double t_norm = 0.0;
    const int* win_particle = nullptr;
    const int* win_shift = nullptr;
    long long grid_evals = 0;       // seed-grid evaluations per window
    WindowOutcome* out = nullptr;
    // wedge-power factors (packed (l, m >= 0)) for the anchored-chart composition
    const double2* chi_hat = nullptr;
    const double2* q_hat = nullptr;
    double wp_total = 1.0;
};

int refine_batch(const BandTables& T, int rows_band);
size_t refine_smem_bytes(const BandTables& T, int rows_band, int batch);
long long refine_scratch_floats(const BandTables& T);
int refine_warps();
int refine_resident_blocks(const BandTables& T, int rows_band, int batch, int device);
int launch_refine(const RefineArgs& a, int blocks, cudaStream_t s);

// standalone batched evaluation (rotate-score-gradient sweep, config 4):
// value + gradient of C(g) = Re sum xi D(g) for n_xi kernels x n_rot angle
// triples; out[(p*n_rot + g)*4 + {0..3}] = value, dC/dalpha, dC/dbeta, dC/dgamma.
struct EvalArgs {
    BandTables T;
    const float2* xi = nullptr;     // [n_xi][T.rows*32] kernels in band layout
    const double* euler = nullptr;  // [n_rot][3]
    int n_xi = 0, n_rot = 0;
    int order = 1;
    double* out = nullptr;
};
int launch_eval_sweep(const EvalArgs& a, cudaStream_t s);

// build band-layout kernels xi_l[m,m'] = sum_k conj(f_klm) t_klm' for many
// coefficient pairs (f from real-packed rows)
struct XiArgs {
    BandTables T;
    const int* row_group = nullptr;
    const float* f = nullptr;   // [n][ldf] real-packed
    int ldf = 0;
    const float* t = nullptr;   // [n][ldt] real-packed (ldt = 0: one shared template)
    int ldt = 0;
    const int* block_off = nullptr;
    const int* radial_count = nullptr;
    int n = 0;
    float2* out = nullptr;      // [n][T.rows*32]
};
int launch_build_xi(const XiArgs& a, cudaStream_t s);

}  // namespace bmb
