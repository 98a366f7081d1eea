// extern "C" boundary of libballmatch_b200 (declared in include/ballmatch_b200.h).
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "../../include/ballmatch_b200.h"
#include "bmb_internal.hpp"

namespace bmb {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace bmb

extern "C" {

const char* bm_last_error(void) { return bmb::g_last_error.c_str(); }

int bm_abi_version(void) { return BM_ABI_VERSION; }

int bm_split3_gemm(int fmt, int block_n, int kchunk, const void* a_hi, const void* a_lo, const void* b_hi,
                   const void* b_lo, float* out, long long ldo, long long m_pad, long long n_pad,
                   long long k_pad, int m_valid, int n_valid, const float* row_scale,
                   const float* col_scale, void* stream) {
    bmb::SplitGemmArgs a;
    a.fmt = fmt;
    a.block_n = block_n;
    a.kchunk = kchunk;
    a.a_hi = a_hi;
    a.a_lo = a_lo;
    a.b_hi = b_hi;
    a.b_lo = b_lo;
    a.out = out;
    a.ldo = ldo;
    a.m_pad = m_pad;
    a.n_pad = n_pad;
    a.k_pad = k_pad;
    a.m_valid = m_valid;
    a.n_valid = n_valid;
    a.row_scale = row_scale;
    a.col_scale = col_scale;
    const int rc = bmb::launch_split3_gemm(a, static_cast<cudaStream_t>(stream));
    if (rc != BM_OK) bmb::set_last_error("bm_split3_gemm: bad shape or launch failure");
    return rc;
}

}  // extern "C"
