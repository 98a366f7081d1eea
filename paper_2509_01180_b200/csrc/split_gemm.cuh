// Split-precision tcgen05 GEMM for the ball-harmonic expansion (kernel K2).
//
//   out[n][m] = row_scale[m] * col_scale[n] *
//               sum_k (Ahi[m][k] Bhi[n][k] + Ahi[m][k] Blo[n][k] + Alo[m][k] Bhi[n][k])
//
// A = the pulled-back expansion operator E (coefficient rows x support voxels),
// B = the gathered shift windows (window rows x support voxels); both are
// K-major and split into hi + lo parts so that three tensor-core passes give an
// FP32-accurate product ("3xTF32", or the same split with FP16 parts and
// power-of-two row/column scaling).  The lo.lo term is dropped (relative size
// 2^-22).
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer      : 4 tiles per stage (Ahi, Alo, Bhi, Blo), SW128
//   warp 1      MMA issuer        : 3 passes x (128 B / 32 B) tcgen05.mma per stage
//   warp 2      TMEM allocator
//   warps 4..7  epilogue          : tcgen05.ld 32x32b -> scale -> coalesced st.global
// Accuracy: the tensor-core accumulator rounds toward zero on every MMA
// accumulate step (measured on B200: error grows linearly with K, 2e-4 relative
// at K = 89,600).  The K loop is therefore cut into chunks of `kchunk` K-blocks;
// each chunk accumulates in one of two ping-pong TMEM buffers and the epilogue
// warps drain it into FP32 registers with round-to-nearest adds while the MMA
// warp fills the other buffer.  The same ping-pong overlaps the epilogue of
// tile i with the main loop of tile i+1.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "sm100_ptx.cuh"

namespace bmb {

constexpr int kGemmBlockM = 128;
constexpr int kGemmThreads = 256;

template <int FMT, int BLOCK_N>
struct SplitGemmCfg {
    static constexpr int kElem = (FMT == 2) ? 4 : 2;      // bytes per element
    static constexpr int kBlockK = 128 / kElem;           // one 128-byte swizzle row
    static constexpr int kUmmaK = 32 / kElem;             // K per tcgen05.mma
    static constexpr int kTileA = kGemmBlockM * 128;      // bytes
    static constexpr int kTileB = BLOCK_N * 128;
    static constexpr int kStageBytes = 2 * kTileA + 2 * kTileB;
    static constexpr int kStages = (BLOCK_N >= 128) ? 3 : 4;
    static constexpr int kTmemCols = (2 * BLOCK_N <= 256) ? 256 : 512;
    static_assert(BLOCK_N <= 128, "register accumulators hold BLOCK_N columns per thread");
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

template <int FMT, int BLOCK_N>
__global__ void __launch_bounds__(kGemmThreads, 1)
    split3_gemm_kernel(const __grid_constant__ CUtensorMap tm_a_hi,
                       const __grid_constant__ CUtensorMap tm_a_lo,
                       const __grid_constant__ CUtensorMap tm_b_hi,
                       const __grid_constant__ CUtensorMap tm_b_lo, float* __restrict__ out,
                       long long ldo, int m_valid, int n_valid, int num_m_tiles, int num_n_tiles,
                       int num_k_blocks, int kchunk, const float* __restrict__ row_scale,
                       const float* __restrict__ col_scale) {
    using Cfg = SplitGemmCfg<FMT, BLOCK_N>;
    constexpr int S = Cfg::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
    uint64_t* empty_bar = full_bar + S;
    uint64_t* tfull_bar = empty_bar + S;   // [2]
    uint64_t* tempty_bar = tfull_bar + 2;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

    const uint32_t warp = ptx::warp_id();
    const int num_tiles = num_m_tiles * num_n_tiles;

    if (warp == 0 && ptx::lane_id() == 0) {
        ptx::tma_prefetch_desc(&tm_a_hi);
        ptx::tma_prefetch_desc(&tm_a_lo);
        ptx::tma_prefetch_desc(&tm_b_hi);
        ptx::tma_prefetch_desc(&tm_b_lo);
        for (int i = 0; i < S; ++i) {
            ptx::mbar_init(&full_bar[i], 1);
            ptx::mbar_init(&empty_bar[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull_bar[i], 1);
            ptx::mbar_init(&tempty_bar[i], 4);  // one arrival per epilogue warp
        }
        ptx::fence_mbar_init();
    }
    if (warp == 2) {
        ptx::tmem_alloc(tmem_slot, Cfg::kTmemCols);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (ptx::elect_one()) {
            const uint64_t pol_a = ptx::policy_evict_last();   // operator: reused by all windows
            const uint64_t pol_b = ptx::policy_evict_first();  // windows: reused by M tiles only
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int m0 = (tile % num_m_tiles) * kGemmBlockM;
                const int n0 = (tile / num_m_tiles) * BLOCK_N;
                for (int kb = 0; kb < num_k_blocks; ++kb) {
                    ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
                    uint8_t* st = smem + stage * Cfg::kStageBytes;
                    ptx::mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
                    const int k0 = kb * Cfg::kBlockK;
                    ptx::tma_load_2d_hint(st, &tm_a_hi, &full_bar[stage], k0, m0, pol_a);
                    ptx::tma_load_2d_hint(st + Cfg::kTileA, &tm_a_lo, &full_bar[stage], k0, m0,
                                          pol_a);
                    ptx::tma_load_2d_hint(st + 2 * Cfg::kTileA, &tm_b_hi, &full_bar[stage], k0, n0,
                                          pol_b);
                    ptx::tma_load_2d_hint(st + 2 * Cfg::kTileA + Cfg::kTileB, &tm_b_lo,
                                          &full_bar[stage], k0, n0, pol_b);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        constexpr uint32_t idesc = ptx::make_idesc(FMT, kGemmBlockM, BLOCK_N);
        int stage = 0;
        uint32_t phase = 0;
        int buf = 0;
        uint32_t buf_phase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            for (int kb0 = 0; kb0 < num_k_blocks; kb0 += kchunk) {
                const int kb1 = min(kb0 + kchunk, num_k_blocks);
                ptx::mbar_wait(&tempty_bar[buf], buf_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + buf * BLOCK_N;
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&full_bar[stage], phase);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        uint8_t* st = smem + stage * Cfg::kStageBytes;
                        const uint64_t a_hi = ptx::smem_desc_k_sw128(st);
                        const uint64_t a_lo = ptx::smem_desc_k_sw128(st + Cfg::kTileA);
                        const uint64_t b_hi = ptx::smem_desc_k_sw128(st + 2 * Cfg::kTileA);
                        const uint64_t b_lo =
                            ptx::smem_desc_k_sw128(st + 2 * Cfg::kTileA + Cfg::kTileB);
#pragma unroll
                        for (int kk = 0; kk < 128 / 32; ++kk) {
                            const uint64_t off = (uint64_t)(kk * 32) >> 4;  // 32 B per UMMA_K
                            const uint32_t first = (kb > kb0 || kk > 0) ? 1u : 0u;
                            if constexpr (FMT == 2) {
                                ptx::mma_tf32(d_tmem, a_hi + off, b_hi + off, idesc, first);
                                ptx::mma_tf32(d_tmem, a_hi + off, b_lo + off, idesc, 1u);
                                ptx::mma_tf32(d_tmem, a_lo + off, b_hi + off, idesc, 1u);
                            } else {
                                ptx::mma_f16(d_tmem, a_hi + off, b_hi + off, idesc, first);
                                ptx::mma_f16(d_tmem, a_hi + off, b_lo + off, idesc, 1u);
                                ptx::mma_f16(d_tmem, a_lo + off, b_hi + off, idesc, 1u);
                            }
                        }
                        ptx::tc_commit(&empty_bar[stage]);
                        if (kb == kb1 - 1) ptx::tc_commit(&tfull_bar[buf]);
                    }
                    __syncwarp();
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (++buf == 2) {
                    buf = 0;
                    buf_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue
        const uint32_t sub = warp & 3;  // TMEM lane quarter this warp may access
        const int lane = ptx::lane_id();
        int buf = 0;
        uint32_t buf_phase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const int m0 = (tile % num_m_tiles) * kGemmBlockM;
            const int n0 = (tile / num_m_tiles) * BLOCK_N;
            float acc[BLOCK_N];
#pragma unroll
            for (int j = 0; j < BLOCK_N; ++j) acc[j] = 0.0f;
            for (int kb0 = 0; kb0 < num_k_blocks; kb0 += kchunk) {
                ptx::mbar_wait(&tfull_bar[buf], buf_phase);
                ptx::tc_fence_after();
#pragma unroll
                for (int c = 0; c < BLOCK_N / 32; ++c) {
                    uint32_t r[32];
                    ptx::tmem_ld_32x32b_x32(
                        tmem_base + ((sub * 32u) << 16) + buf * BLOCK_N + c * 32, r);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) acc[c * 32 + j] += __uint_as_float(r[j]);
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&tempty_bar[buf]);
                if (++buf == 2) {
                    buf = 0;
                    buf_phase ^= 1;
                }
            }
            const int m = m0 + sub * 32 + lane;
            if (m < m_valid) {
                const float rs = (row_scale != nullptr) ? row_scale[m] : 1.0f;
#pragma unroll
                for (int j = 0; j < BLOCK_N; ++j) {
                    const int n = n0 + j;
                    if (n < n_valid) {
                        const float cs = (col_scale != nullptr) ? col_scale[n] : 1.0f;
                        out[(long long)n * ldo + m] = acc[j] * rs * cs;
                    }
                }
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, Cfg::kTmemCols);
    }
}

}  // namespace bmb
