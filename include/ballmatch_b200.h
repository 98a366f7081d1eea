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

#ifdef __cplusplus
}
#endif

#endif /* BALLMATCH_B200_H */
