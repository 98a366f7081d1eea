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

#define BM_ABI_VERSION 1

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
/* lambda_cut actually used by the context */
double bm_context_lambda_cut(const bm_context* ctx);
/* radial roots / norms of degree l (BasisSpec::root/norm, basis.hpp:40-41); returns count k_l */
int bm_context_roots(const bm_context* ctx, int l, double* roots, double* norms);
double bm_default_lambda_cut(int n, int l_max);

/* Batched expansion (expand(shift_volume(v, s)), src/basis.cpp:247-330 with
 * src/volume.cpp:50-67): `count` float32 volumes (device, n^3 each, x fastest)
 * with optional integer shifts (host int[3*count], NULL = 0) -> complex128
 * coefficients (device, count x coeff_count, interleaved re/im) in the
 * reference's layout (block l, row k, column m+l).
 * Streams: every call is ordered after prior work on `stream` (NULL = the
 * legacy default stream) and later work on `stream` is ordered after it. */
int bm_expand(bm_context* ctx, const float* vols, int count, const int* shifts, double* out,
              void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BALLMATCH_B200_H */
