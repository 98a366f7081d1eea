// Host side of the split-precision tcgen05 GEMM: tensor maps + launch.
#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>

#include "bmb_internal.hpp"
#include "split_gemm.cuh"

namespace bmb {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

}  // namespace

// 2-D K-major operand: rows x k_pad elements, row pitch k_pad elements,
// box = (128 bytes of K) x box_rows, 128-byte swizzle.
int make_operand_tmap(CUtensorMap* map, const void* base, int fmt, long long rows,
                      long long k_pad, int box_rows) {
    auto encode = get_encode_fn();
    if (!encode) return BMB_ERR_CUDA;
    const int elem = fmt == 2 ? 4 : 2;
    const CUtensorMapDataType dt =
        fmt == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    cuuint64_t dims[2] = {(cuuint64_t)k_pad, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(k_pad * elem)};
    cuuint32_t box[2] = {(cuuint32_t)(128 / elem), (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? BMB_OK : BMB_ERR_CUDA;
}

template <int FMT, int BN>
static int launch_impl(const SplitGemmArgs& a, cudaStream_t stream) {
    using Cfg = SplitGemmCfg<FMT, BN>;
    CUtensorMap ta_hi, ta_lo, tb_hi, tb_lo;
    int rc = BMB_OK;
    rc |= make_operand_tmap(&ta_hi, a.a_hi, FMT, a.m_pad, a.k_pad, kGemmBlockM);
    rc |= make_operand_tmap(&ta_lo, a.a_lo, FMT, a.m_pad, a.k_pad, kGemmBlockM);
    rc |= make_operand_tmap(&tb_hi, a.b_hi, FMT, a.n_pad, a.k_pad, BN);
    rc |= make_operand_tmap(&tb_lo, a.b_lo, FMT, a.n_pad, a.k_pad, BN);
    if (rc != BMB_OK) return BMB_ERR_CUDA;
    auto kern = split3_gemm_kernel<FMT, BN>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg::kSmemBytes) != cudaSuccess)
        return BMB_ERR_CUDA;
    const int mt = (int)(a.m_pad / kGemmBlockM), nt = (int)(a.n_pad / BN);
    const int tiles = mt * nt;
    int grid = a.num_sms > 0 ? a.num_sms : 148;
    if (grid > tiles) grid = tiles;
    kern<<<grid, kGemmThreads, Cfg::kSmemBytes, stream>>>(
        ta_hi, ta_lo, tb_hi, tb_lo, a.out, a.ldo, a.m_valid, a.n_valid, mt, nt,
        (int)(a.k_pad / Cfg::kBlockK), a.kchunk > 0 ? a.kchunk : (int)(a.k_pad / Cfg::kBlockK),
        a.row_scale, a.col_scale);
    return cudaGetLastError() == cudaSuccess ? BMB_OK : BMB_ERR_CUDA;
}

int launch_split3_gemm(const SplitGemmArgs& a, cudaStream_t stream) {
    const int bk = a.fmt == 2 ? 32 : 64;
    if (a.m_pad % kGemmBlockM || a.k_pad % bk) return BMB_ERR_ARG;
    if (a.fmt == 2) {
        if (a.block_n == 64 && a.n_pad % 64 == 0) return launch_impl<2, 64>(a, stream);
        if (a.n_pad % 128 == 0) return launch_impl<2, 128>(a, stream);
    } else if (a.fmt == 0) {
        if (a.block_n == 64 && a.n_pad % 64 == 0) return launch_impl<0, 64>(a, stream);
        if (a.n_pad % 128 == 0) return launch_impl<0, 128>(a, stream);
    }
    return BMB_ERR_ARG;
}

}  // namespace bmb
