// Internal declarations shared by the CUDA translation units of libballmatch_b200.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

namespace bmb {

enum Status : int {
    BMB_OK = 0,
    BMB_ERR_ARG = 1,     // std::invalid_argument in the reference
    BMB_ERR_CUDA = 2,    // CUDA / driver failure (or no device)
    BMB_ERR_DOMAIN = 3,  // std::domain_error (e.g. zero energy)
    BMB_ERR_STATE = 4,   // bad handle / wrong call order
    BMB_ERR_NOMEM = 5,
};

void set_last_error(const std::string& msg);

struct SplitGemmArgs {
    int fmt = 2;         // 2 = TF32 parts, 0 = FP16 parts
    int block_n = 128;   // 64 or 128
    const void* a_hi = nullptr;
    const void* a_lo = nullptr;
    const void* b_hi = nullptr;
    const void* b_lo = nullptr;
    float* out = nullptr;
    long long ldo = 0;   // out[n * ldo + m]
    long long m_pad = 0, n_pad = 0, k_pad = 0;
    int m_valid = 0, n_valid = 0;
    const float* row_scale = nullptr;
    const float* col_scale = nullptr;
    int num_sms = 0;
    int kchunk = 4;      // K-blocks per TMEM accumulation chunk (0 = whole K)
};

int make_operand_tmap(CUtensorMap* map, const void* base, int fmt, long long rows,
                      long long k_pad, int box_rows);
int launch_split3_gemm(const SplitGemmArgs& a, cudaStream_t stream);

}  // namespace bmb
