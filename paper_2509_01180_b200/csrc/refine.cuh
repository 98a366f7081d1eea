// Refinement interface (kernels K4/K5/K7): bulk-synchronous damped Newton.
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace bmb {

// Per-candidate working state of the bulk-synchronous Newton iteration.
enum CandStatus : int { ST_DONE = 0, ST_START = 1, ST_EVAL2 = 2, ST_EVAL0 = 3, ST_FINAL = 4 };

struct CandWork {
    double e[3];    // chart Euler angles of the current iterate
    double et[3];   // chart Euler angles of the trial iterate
    double gt[4];   // trial chart rotation h_try
    double c[10];   // raw correlation derivatives (value, grad, hess aa ab ag bb bg gg)
    double r[10];   // raw wedge-power derivatives
    double f[13];   // objective at e: value, grad[3], hess[9]
    double ev[3];   // anchored: Euler angles of the order-2 evaluation (g, or g K on the side kernels)
    double lambda;  // Levenberg parameter of the iteration
    double lam;     // damping of the current retry
    int status;
    int retry;
    int iter;
    int side;       // order-2 evaluation: 0 chart angles e on the window kernel (unanchored),
                    // 1 angles of g on the window kernel, 2 angles of g K on the side kernels
    double evt[3];  // frame of the trial's order-2 evaluation (same convention, sidet)
    int sidet;
    int fresh;      // c / r hold the order-2 results of the accepted trial at g (frame ev, side)
    // (cos a, sin a, cos b, sin b) of the chart angles e, of the evaluation frame ev and of
    // the trial frame evt, taken from the rotation matrices (chart_transform needs no sincos)
    double te[4], tv[4], tvt[4];
    double val;     // objective value at g of the last evaluation there ...
    int val_band;   // ... and its band index (-1: none); serves the final score
    unsigned short band_evals[kMaxBands];  // evaluations by band index (evaluations_per_band, optimize.hpp:83)
};

struct StageArgs {
    BandTables T;
    const int* row_group = nullptr;
    const float4* xi_win = nullptr;   // [n_win][T.rows*32] window kernels (A, B entries)
    const float4* xi_side = nullptr;  // [n_win][T.rows*32] side kernels xi D(K^-1)^T (anchored candidates)
    CandState* cand = nullptr;
    CandWork* work = nullptr;
    const int* cand_count = nullptr;
    int max_cand = 0;
    int n_win = 0;
    RefineParams prm;
    int* counts = nullptr;           // [CNT_*] list lengths
    int* list2 = nullptr;            // candidates awaiting the order-2 evaluation (or final)
    unsigned long long* eval_stats = nullptr;  // [kMaxL+1][2][2] evaluations by (L, order, wedge)
};
enum { CNT_L2 = 0, CNT_STEP = 1, CNT_T0 = 2, CNT_T1 = 3 };

// one window outcome per window (last band)
struct ReduceArgs {
    const CandState* cand = nullptr;
    const CandWork* work = nullptr;  // per-band evaluation counters
    const int* cand_count = nullptr;
    int max_cand = 0;
    int n_win = 0;
    const double* sub_norm = nullptr;
    double t_norm = 0.0;
    const int* win_particle = nullptr;
    const int* win_shift = nullptr;
    long long grid_evals = 0;
    int extra_candidates = 0;   // prune_after_band: the winner's second refine() run
    WindowOutcome* out = nullptr;
};

// band start of every candidate; the started ones are appended to start
void launch_band_begin(const StageArgs& a, int* start, int* start_count, cudaStream_t s);
// iteration start of the candidates on a start list (max_n bounds its length)
void launch_iter_begin(const StageArgs& a, const int* start, const int* start_count, int max_n, cudaStream_t s);
// order 2 at the iteration point (trial = false) or at the trial point (trial = true,
// the refinement's trials: their derivatives serve the next iteration when accepted);
// order 0 at the global angles et (final scores)
void launch_eval(const StageArgs& a, int order, const int* list, const int* count, int max_n, cudaStream_t s,
                 bool trial = false);
// Newton step of the candidates on list_in (order-2 results in c / r); trials to list_out
void launch_step(const StageArgs& a, const int* list_in, const int* count_in, int* list_out, int* count_out,
                 int max_n, cudaStream_t s);
// one round over pending trials (order-2 evaluated): accept / retry, and for accepted
// trials the next iteration's start and step (advance_kernel)
void launch_advance(const StageArgs& a, const int* list_in, const int* count_in, int* trial_out, int* trial_count,
                    int* fresh_out, int* fresh_count, int max_n, cudaStream_t s);
void launch_final_prep(const StageArgs& a, cudaStream_t s);
void launch_final_score(const StageArgs& a, int max_n, cudaStream_t s);
void launch_window_reduce(const ReduceArgs& a, cudaStream_t s);
void launch_prune(const StageArgs& a, cudaStream_t s);

// Objective::eval of the refinement at n chart points (angles euler[3n], anchors
// [4n] quaternions or null) on the window kernels of a.xi_win / a.xi_side (one
// window): out[13n] = value, gradient, Hessian (order 2) in the chart angles.
// a.cand / a.work / a.list2 / a.counts need n slots (a.max_cand = n, a.n_win = 1).
int launch_objective_eval(const StageArgs& a, const double* euler, const double* anchors, int n, int order,
                          double* out, cudaStream_t s);

// standalone batched evaluation (rotate-score-gradient sweep, config 4):
// value + gradient of C(g) = Re sum xi D(g) for n_xi kernels x n_rot angle
// triples; out[(p*n_rot + g)*4 + {0..3}] = value, dC/dalpha, dC/dbeta, dC/dgamma.
struct EvalArgs {
    BandTables T;
    const float4* xi = nullptr;     // [n_xi][T.rows*32] kernels in band layout
    const double* euler = nullptr;  // [n_rot][3]
    int n_xi = 0, n_rot = 0;
    int order = 1;
    double* out = nullptr;
};
int launch_eval_sweep(const EvalArgs& a, cudaStream_t s);

// algorithmic FLOPs of one evaluation (SURVEY.md §8(d) accounting, full (m,m') plane):
// recursion 6 N_xi per derivative order, contraction 4 N_xi and phases 6 (2L+1)^2 per
// reduced value and kernel (correlation, + wedge-power kernel)
double eval_flops(int L, int order, bool wedge);

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
    float4* out = nullptr;      // [n][T.rows*32]
    const float* t2 = nullptr;  // optional second (shared) template: kernels of (f, t2) into out2
    float4* out2 = nullptr;
    int nf = 0;                 // real-packed floats of degrees <= T.L (> 0: one CTA per set, rows staged in smem)
    int npairs = 0;             // complex (order >= 0) entries of degrees <= T.L: sum_l n_k(l) (l + 1) (staged pair kernel)
};
int launch_build_xi(const XiArgs& a, cudaStream_t s);

}  // namespace bmb
