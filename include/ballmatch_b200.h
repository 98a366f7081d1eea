/* ballmatch_b200 — C ABI of the B200-native ball-harmonics alignment hot path.
 *
 * Plain C: opaque handles, plain pointers and sizes, integer status codes.
 * No exceptions cross this boundary; the host shim maps status codes back to
 * the reference's exception types (std::invalid_argument -> BM_ERR_ARG,
 * std::domain_error -> BM_ERR_DOMAIN).  Each entry point names the reference
 * interface it replaces (paths relative to the reference's proj/).
 */
#ifndef BALLMATCH_B200_H
#define BALLMATCH_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define BM_ABI_VERSION 3

enum bm_status {
    BM_OK = 0,
    BM_ERR_ARG = 1,
    BM_ERR_CUDA = 2,
    BM_ERR_DOMAIN = 3,
    BM_ERR_STATE = 4,
    BM_ERR_NOMEM = 5
};

/* Last error message of the calling thread ("" if none). */
const char* bm_last_error(void);
int bm_abi_version(void);

/* Split-precision tensor-core GEMM used by the expansion (kernel K2):
 *   out[n*ldo + m] = row_scale[m] col_scale[n] sum_k (Ahi Bhi + Ahi Blo + Alo Bhi)[m,n,k]
 * A: m_pad x k_pad, B: n_pad x k_pad, both K-major, device pointers.
 * fmt 2: float parts consumed as TF32; fmt 0: __half parts.  row/col scales may be NULL.
 * block_n: 64 or 128.  kchunk: K-blocks (128 bytes of K each) accumulated in TMEM
 * before the partial sum is drained to FP32 registers (0 = whole K).
 * Replaces the stage-2..4 contractions of expand() (src/basis.cpp:271-328). */
int bm_split3_gemm(int fmt, int block_n, int kchunk, const void* a_hi, const void* a_lo, const void* b_hi,
                   const void* b_lo, float* out, long long ldo, long long m_pad, long long n_pad,
                   long long k_pad, int m_valid, int n_valid, const float* row_scale,
                   const float* col_scale, void* stream);

/* ------------------------------------------------------------------ context
 * One context per device: the basis (BasisSpec, include/ballmatch/basis.hpp:31-58,
 * built by build_spec, src/basis.cpp:88-115) and the pulled-back expansion
 * operator for an n^3 grid, resident in HBM.  lambda_cut <= 0 selects
 * default_lambda_cut(n, l_max) (src/basis.cpp:117-138). */
typedef struct bm_context bm_context;
int bm_context_create(int device, int n, int l_max, double lambda_cut, bm_context** out);
int bm_context_destroy(bm_context* ctx);
/* info[0..9]: n, l_max, coeff_count, support_voxels, m_pad, k_pad, n_r, n_theta, n_phi, pair_count */
int bm_context_info(const bm_context* ctx, long long* info);
/* Expansion algorithm of the context: 0 = factored (trilinear samples, phi-DFT,
 * theta and radial contractions per window; default), 1 = dense pulled-back
 * operator on the tensor cores (gather + bm_split3_gemm; the operator is built
 * on first use).  Both follow expand() (src/basis.cpp:254-328). */
int bm_context_set_expand_mode(bm_context* ctx, int mode);
/* Concurrent lanes of bm_align_batch: a batch of at least lanes * min_per_lane
 * particles is split into `lanes` slices aligned concurrently, each on its own
 * stream with its own buffers and host thread (default 4 lanes, 64 particles per
 * lane).  Results do not depend on the lane count. */
int bm_context_set_lanes(bm_context* ctx, int lanes, int min_per_lane);
/* Expansion gathers of the factored mode: 0 = direct loads, 1 = from a copy of
 * each volume when it has >= 4 windows (default; the shift search: the
 * zero-padded quad copy when every |shift| <= 6, else the x-paired copy),
 * 2 = always from the x-paired copy, 3 = always from the quad copy when the
 * shifts allow it.  The coefficients are bit-identical. */
int bm_context_set_expand_pairs(bm_context* ctx, int mode);
/* Host-buffer staging: with reuse on, a bm_average_accumulate directly after a
 * completed bm_align_batch of the same host buffer and count uses the device
 * copy that bm_align_batch staged (once), instead of copying the buffer again.
 * The caller promises not to modify the buffer in between.  Default off: every
 * call stages its host particles. */
int bm_context_set_stage_reuse(bm_context* ctx, int on);
/* lambda_cut actually used by the context */
double bm_context_lambda_cut(const bm_context* ctx);
/* radial roots / norms of degree l (BasisSpec::root/norm, basis.hpp:40-41); returns count k_l */
int bm_context_roots(const bm_context* ctx, int l, double* roots, double* norms);
double bm_default_lambda_cut(int n, int l_max);
/* Host-only basis setup (build_spec, src/basis.cpp:88-115, no device needed):
 * the radial roots lambda_lk <= lambda_cut of degree l <= l_max and their norms
 * c_lk = sqrt(2) / |j_{l+1}(lambda_lk)| (BasisSpec::root/norm, basis.hpp:40-41);
 * roots / norms need room for the count (<= lambda_cut / pi + 1 entries). */
int bm_basis_roots(int l_max, double lambda_cut, int l, double* roots, double* norms, int* count);

/* Batched expansion (expand(shift_volume(v, s)), src/basis.cpp:247-330 with
 * src/volume.cpp:50-67): `count` float32 volumes (device, n^3 each, x fastest)
 * with optional integer shifts (host int[3*count], NULL = 0) -> complex128
 * coefficients (device, count x coeff_count, interleaved re/im) in the
 * reference's layout (block l, row k, column m+l).
 * Streams: every call is ordered after prior work on `stream` (NULL = the
 * legacy default stream) and later work on `stream` is ordered after it. */
int bm_expand(bm_context* ctx, const float* vols, int count, const int* shifts, double* out,
              void* stream);
/* The same for shift windows that share volumes (the shift search of
 * search_one_shift, src/optimize.cpp:361-419: expand(shift_volume(f, s)) for
 * many s of one subtomogram): window w reads volume win_vol[w] (host int[n_win],
 * 0 <= win_vol[w] < n_vol) shifted by win_shift[3w..3w+2] (host); out is
 * n_win x coeff_count complex128 on the device. */
int bm_expand_windows(bm_context* ctx, const float* vols, int n_vol, const int* win_vol, const int* win_shift,
                      int n_win, double* out, void* stream);

/* ------------------------------------------------------------------ alignment
 * Mirrors OptimizerConfig (include/ballmatch/optimize.hpp:15-32); l_max and
 * lambda_cut are the context's.  accept_tol is the relative slack of the Newton
 * acceptance test (reference: 1e-12 with FP64 scores, src/optimize.cpp:332);
 * the FP32 evaluation uses a wider default.  auto_bands != 0 selects
 * each particle's bands from its zero-shift kernel (select_bands with the
 * thresholds, optimize.cpp:179-195, 455-460; n_thresholds 0: 0.5, 0.25, 0.05);
 * prune_after_band != 0 keeps only each window's best candidate after the
 * first band (optimize.cpp:391-403). */
typedef struct bm_align_config {
    int n_bands;
    int bands[16];
    double seed_grid_step;
    int max_candidates;
    int newton_max_iter;
    double grad_tol;
    double step_damping;
    int shift_radius;
    int shift_step;
    double accept_tol;
    int auto_bands;
    int prune_after_band;
    int n_thresholds;
    double thresholds[8];
} bm_align_config;

/* AlignmentResult (optimize.hpp:71-88): shift, rotation (template -> particle,
 * quaternion w,x,y,z), score normalized by the expansion norms. */
typedef struct bm_align_result {
    int shift[3];
    double quat[4];
    double score;
    int converged;
    long long candidates;
    long long evaluations;
    double subtomo_norm;
    int windows;
    int n_bands;   /* the band schedule used (auto_bands: per particle) */
    int bands[16];
    long long evaluations_per_band[16];  /* aligned with bands; the seed grid counts at bands[0] */
    double expand_template_s;  /* phase timings (optimize.hpp:83-86), of the batch call: */
    double coarse_search_s;    /* the particles are aligned together, so these are shared */
    double fine_search_s;
} bm_align_result;

/* One window outcome (search_one_shift, src/optimize.cpp:361-419). */
typedef struct bm_window_result {
    int volume;
    int shift[3];
    int valid;
    int n_candidates;
    int converged;
    double raw_score;
    double norm_score;
    double subtomo_norm;
    double quat[4];
    long long evaluations;
} bm_window_result;

/* Template state of align() (src/optimize.cpp:438-454): expand the template
 * (device float32 n^3), and for a wedge (theta in (0,90), tilt axis y) build
 * the tapered filter and the wedge-power kernel.  theta <= 0: no wedge. */
int bm_set_template(bm_context* ctx, const float* tmpl, double wedge_theta_deg, void* stream);
/* template norm ||t_hat|| */
double bm_template_norm(const bm_context* ctx);

/* align() for `count` particles (float32, count x n^3, device OR host memory):
 * wedge filter, coarse + fine shift windows, seeding, device Newton with
 * frequency marching.  Host particles (pinned for overlap) are staged by each
 * concurrent lane on its own stream right before it aligns its slice; the
 * staged copy also serves a following bm_average_accumulate of the same host
 * buffer.  Results to host memory; synchronizes the context stream. */
int bm_align_batch(bm_context* ctx, const float* particles, int count, const bm_align_config* cfg,
                   bm_align_result* out, void* stream);

/* search_one_shift for explicit windows (volume index, shift) of device
 * volumes (already wedge-filtered by the caller if needed); results to host. */
int bm_search_windows(bm_context* ctx, const float* vols, int n_vol, const int* win_vol,
                      const int* win_shift, int n_win, const bm_align_config* cfg,
                      bm_window_result* out, void* stream);

/* Batched rotate-score-gradient (correlation_derivatives order 0/1,
 * src/xcorr.cpp:52-105) of xi_p = xi_coefficients(f_p, t) at band L = l_max:
 * f: device complex128 (n_f x coeff_count, reference layout, real-volume
 * symmetric), t: one device complex128 coefficient set, euler: device
 * double (n_rot x 3).  out: device double (n_f x n_rot x 4):
 * value, dC/dalpha, dC/dbeta, dC/dgamma. */
int bm_eval_sweep(bm_context* ctx, const double* f, int n_f, const double* t, const double* euler,
                  int n_rot, int order, double* out, void* stream);

/* Objective::eval (src/optimize.cpp:102-131) exactly as the refinement evaluates
 * it: kernels xi = xi_coefficients(f, t) (xcorr.cpp:21-50) of one coefficient set
 * f (device complex128, reference layout, real-volume symmetric) against t
 * (device, same layout; NULL = the context's template), with the wedge-power
 * quotient C / sqrt(clamp(1 - rho, 0.02, 2)) when the template state has a wedge,
 * at band L for n points.  euler (device double, n x 3) are chart angles e and
 * anchors (device double, n x 4 quaternions, or NULL) chart anchors a: the
 * function is C~(e) = C(R(e) a), as on the composed kernel xi D(a)^T of
 * xi_compose_right (xcorr.cpp:149-155) that refine() uses near the poles
 * (optimize.cpp:268-299).  order 2: value, gradient, Hessian
 * (correlation_derivatives order 2, xcorr.cpp:52-105); order 0: value only.
 * out (device double, n x 13): value, d/d(alpha, beta, gamma), Hessian row-major. */
int bm_objective_eval(bm_context* ctx, const double* f, const double* t, const double* euler,
                      const double* anchors, int n, int L, int order, double* out, void* stream);

/* seed_candidates (src/optimize.cpp:197-253, grid_scores 48-97) for n_f
 * coefficient sets f (device complex128, reference layout) against the context's
 * template at band L_low on the Euler grid of `step`, with the template's wedge
 * quotient: quats (host, n_f x max_candidates x 4) in rank order, counts (host,
 * n_f), scores (host, n_f x max_candidates, may be NULL) the seed grid scores. */
int bm_seed_candidates(bm_context* ctx, const double* f, int n_f, int L_low, double step,
                       int max_candidates, double* quats, int* counts, double* scores, void* stream);

/* Template coefficients t_hat (expand of the template, complex128 device,
 * reference layout) of the current template state. */
int bm_template_coeffs(bm_context* ctx, double* out, void* stream);

/* Wedge-power kernel of the current template state (wedge_power_kernel,
 * src/xcorr.cpp:234-357): XiBlocks layout, degree blocks l = 0..l_max of
 * (2l+1)^2 complex128 entries [m][m'] (host memory, N_xi(l_max) entries).
 * BM_ERR_STATE without a wedge. */
int bm_wedge_power_kernel(bm_context* ctx, double* out);

/* ------------------------------------------------------------------ reference operators
 * FP64 device operators on the reference's layouts: coefficient sets complex128
 * (degree blocks, row k, column m + l: BallExpansion, basis.hpp:67-91), kernels
 * as XiBlocks (degree blocks l = 0..l_max of (2l+1)^2 entries [m][m'],
 * xcorr.hpp:22-43).  All pointers are device memory unless noted. */
/* xi_coefficients (src/xcorr.cpp:21-50): out[p] = xi(f[p], t), f: n sets, t: one set */
int bm_xi_coefficients(bm_context* ctx, const double* f, int n, const double* t, double* out, void* stream);
/* xi_compose_right (src/xcorr.cpp:149-155): out = xi D(a)^T for degrees <= l_limit
 * (l_limit < 0: all), a = quat (host, w x y z) */
int bm_xi_compose_right(bm_context* ctx, const double* xi, const double* quat, int l_limit, double* out,
                        void* stream);
/* rotate_expansion (src/steer.cpp:208-223): out = D(g) f per (k, l) row, g = quat (host) */
int bm_rotate_expansion(bm_context* ctx, const double* f, const double* quat, double* out, void* stream);
/* wigner_D (src/steer.cpp:158-178) for degrees <= L (host memory, XiBlocks layout) */
int bm_wigner_D(int L, const double* quat, double* out);
/* exhaustive_baseline (src/optimize.cpp:523-539): the first maximum of grid_scores
 * at band l_cut on the full ZYZ grid of `angular_step` (EulerGrid::with_step) of
 * one XiBlocks kernel (device); rotation (host quat), score and evaluation count. */
int bm_exhaustive_baseline(bm_context* ctx, const double* xi, int l_cut, double angular_step, double* quat,
                           double* score, long long* evaluations, void* stream);
/* baseline_evaluation_count (src/optimize.cpp:541-544): na * nb * ng of the grid */
long long bm_baseline_evaluation_count(double angular_step);

/* The same sweep (order 1: value and Euler gradient) as two tensor-core GEMMs:
 * per-particle rows of xi (value, -i m, -i m' weighted, half plane folded by the
 * real-volume symmetry) against per-rotation rows of D^l(g) and D'^l(g), FP16
 * three-pass split on tcgen05 (FP32-accurate).  Same inputs and output layout as
 * bm_eval_sweep.  timing (host, may be NULL, 4 doubles): tables ms, GEMM ms,
 * gather ms, tensor-pipe FLOPs of the GEMMs (synchronizes when given). */
int bm_eval_sweep_tc(bm_context* ctx, const double* f, int n_f, const double* t, const double* euler, int n_rot,
                     double* out, double* timing, void* stream);

/* Tapered missing-wedge filter of the current template's context on device
 * volumes (apply_wedge_taper, src/xcorr.cpp:210-232). */
int bm_apply_wedge_taper(bm_context* ctx, const float* in, float* out, int count, void* stream);

/* Subtomogram averaging (new; building blocks rotate_expansion,
 * src/steer.cpp:208-223): sum (device complex128, coeff_count entries,
 * reference layout) += sum_p rotate_expansion(expand(shift_volume(f_w,p, s_p)),
 * g_p^-1) for the particles and their align results (host).  f_w is the
 * wedge-filtered particle when the template state has a wedge.  Dividing by
 * the particle count (after the cross-device allreduce) gives the average. */
int bm_average_accumulate(bm_context* ctx, const float* particles, int count,
                          const bm_align_result* results, double* sum, void* stream);
/* (particles: device or host memory, as for bm_align_batch) */

/* Voxel synthesis of a coefficient set (synthesize, src/basis.cpp:332-419,
 * with its Catmull-Rom radial table, basis.cpp:221-245): coeffs device
 * complex128 (coeff_count, reference layout), real_volume != 0 when the set has
 * the real-volume symmetry (e.g. an average of expansions); out device double
 * n^3 (x fastest), zero outside the unit ball.  FP64. */
int bm_synthesize(bm_context* ctx, const double* coeffs, int real_volume, int n, double* out, void* stream);

/* Kernel timing evidence: with timing on, CUDA events on the context stream
 * bracket every launch of this library.  out_ms[0..14]: gather, expansion,
 * seed, refine, wedge filter, misc, refine by band position 0, 1, 2, 3+, and
 * inside refine: order-2 evaluations, order-0 evaluations, chart-kernel
 * composition, Newton bookkeeping (iteration start, step, acceptance), window
 * kernel build (milliseconds, accumulated since reset);
 * out_counts[0..3]: kernels launched, windows expanded, GEMM launches,
 * refine launches.  reset != 0 clears after reading. */
int bm_context_set_timing(bm_context* ctx, int on);
/* Per-band split of the refinement timers (timing on): ms[b * 15 + k] for band
 * index b = 0, 1, 2, 3+ and the timer classes k of bm_context_timings. */
int bm_context_band_timings(bm_context* ctx, double* ms);
/* Evaluations at band L since the last eval-stats reset: out[0] order 2, out[1] order 0. */
int bm_context_eval_counts(bm_context* ctx, int L, long long* out);
int bm_context_timings(bm_context* ctx, double* out_ms, long long* out_counts, int reset);
/* Rotate-score-gradient evaluations run by the refinement since the last reset:
 * evals[0] order 2 (value, gradient, Hessian), evals[1] order 0 (value), and
 * their algorithmic FLOPs (DESIGN.md §3 K5 accounting).  Always counted. */
int bm_context_eval_stats(bm_context* ctx, long long* evals, double* flops, int reset);

/* ------------------------------------------------------------------ synthetic inputs
 * Seeded generator on the device (BASELINE.json configs; particle pipeline of
 * make_phantom, src/volio.cpp:285-314).  Template: isotropic Gaussian blobs
 * (Philox stream 0 of `seed`).  Particle p uses seed base_seed + p: Haar
 * rotation (stream 1), shift in [-shift_max, shift_max]^3 (stream 2), rotate ->
 * shift by -s -> binary wedge (wedge_deg in (0,90), else none) -> noise at
 * `snr` inside the unit ball (stream 3; snr <= 0: none) -> float32.
 * out: device float32; quats (4 per particle) / shifts (3): host, may be NULL. */
int bm_make_template(int device, int n, int blobs, unsigned long long seed, float* out, void* stream);
int bm_make_particles(int device, const float* tmpl, int n, int count, unsigned long long base_seed,
                      int shift_max, double snr, double wedge_deg, float* out, double* quats,
                      int* shifts, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BALLMATCH_B200_H */
