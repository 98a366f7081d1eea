// Per-device context of the B200 alignment path: basis + operator resident in
// HBM, template state, per-band evaluation tables and grown-on-demand work
// buffers.  One context per device; calls on a context are stream-ordered on
// its stream and not thread-safe (one host thread per device).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cufft.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "basis_host.hpp"
#include "bmb_internal.hpp"
#include "kernels.cuh"

namespace bmb {

// RAII device buffer
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    // grow (never shrink); contents are not preserved
    void reserve(size_t b) {
        if (b <= bytes) return;
        release();
        if (cudaMalloc(&p, b) != cudaSuccess) {
            p = nullptr;
            throw std::bad_alloc();
        }
        bytes = b;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

template <class T>
void upload(DevBuf& d, const std::vector<T>& h, cudaStream_t s) {
    d.reserve(sizeof(T) * (h.size() ? h.size() : 1));
    if (!h.empty())
        cudaMemcpyAsync(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, s);
}

struct BandTablesHost;  // owned device storage of one band's tables

struct AlignConfig {
    std::vector<int> bands;
    double seed_grid_step;
    int max_candidates;
    int newton_max_iter;
    double grad_tol;
    double step_damping;
    int shift_radius;
    int shift_step;
};

struct ParticleResult {
    int shift[3];
    double quat[4];
    double score;
    int converged;
    long long candidates;
    long long evaluations;
    double subtomo_norm;
    int windows;
};

class Context {
public:
    Context(int device, int n, int l_max, double lambda_cut);
    ~Context();

    int device = 0;
    cudaStream_t stream = nullptr;
    int n = 0;
    host::Basis basis;
    Geometry geo;
    std::vector<int> voxels_host;

    // resident operator + geometry tables
    DevBuf E_hi, E_lo, row_scale, voxels, block_off, radial_count, row_weight, row_lkm;

    // work buffers
    DevBuf B_hi, B_lo, col_scale, coef, win_vol, win_shift, vol_scale, norms;

    // expansion of `count` windows (volume index + integer shift) of volumes
    // already on the device; real-packed FP32 coefficients into ctx.coef
    // (row stride geo.m_pad), returns the number of windows.
    void expand_windows(const float* vols, long long vol_stride, int n_vol,
                        const std::vector<int>& wvol, const std::vector<int>& wshift);

    int gemm_block_n = 128;
    int gemm_kchunk = 4;
};

}  // namespace bmb
