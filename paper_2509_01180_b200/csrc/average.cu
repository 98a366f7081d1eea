// Subtomogram averaging in coefficient space (kernel K9; the reference has the
// building blocks only: rotate_expansion, src/steer.cpp:208-223).
//
//   sum_hat += sum_p rotate_expansion(f_hat_{p, s_p}, g_p^-1)
//
// f_hat_{p,s_p} = expand(shift_volume(f_w,p, s_p)) is the winning window of
// particle p (re-expanded through the tensor-core path), g_p its template ->
// particle rotation.  One CTA per particle: the full little-d stack d^l(beta)
// of g_p^-1 in shared memory (FP64 three-term recursion, steer.cpp:43-144),
// f'_{klm} = sum_m' e^{-i m a} d^l_{m m'}(b) e^{-i m' g} f_{klm'}, FP64 atomics
// into the per-device sum.  The cross-device sum is one NCCL allreduce of the
// coefficient vector (host side).
#include <cuda_runtime.h>

#include <cmath>
#include <stdexcept>
#include <vector>

#include "smem_attr.hpp"
#include "average.hpp"
#include "rotation.cuh"

namespace bmb {

namespace {

__device__ double sqrt_binom_a(int n, int k) {
    double r = 1.0;
    for (int i = 1; i <= k; ++i) r *= (double)(n - k + i) / i;
    return sqrt(r);
}

__device__ __forceinline__ int dxi_off(int l) { return l * (2 * l - 1) * (2 * l + 1) / 3; }

__global__ void average_kernel(const float* __restrict__ coef, int ldc, const double* __restrict__ quats,
                               int L, const int* __restrict__ block_off, const int* __restrict__ radial_count,
                               double2* __restrict__ sum, int count, double* __restrict__ dglob) {
    extern __shared__ double dsm[];
    // large L: the d stack in a per-CTA global scratch slice, CTAs loop over particles
    for (int p = blockIdx.x; p < count; p += gridDim.x) {
    // rotation g^-1 and its ZYZ angles
    const Quat g{quats[4 * p], quats[4 * p + 1], quats[4 * p + 2], quats[4 * p + 3]};
    const Euler3 e = q_euler(q_inv(g));
    const double cb = cos(e.b), ch = cos(0.5 * e.b), sh = sin(0.5 * e.b);
    const int W = 2 * L + 1;
    double* d = dglob ? dglob + (size_t)blockIdx.x * dxi_off(L + 1) : dsm;  // N_xi(L) full-plane little-d
    for (int idx = threadIdx.x; idx < W * W; idx += blockDim.x) {
        const int m = idx / W - L, n = idx % W - L;
        const int l0 = max(abs(m), abs(n));
        double fac;
        int pa, pp;
        if (l0 == 0) {
            fac = 1.0, pa = pp = 0;
        } else if (m == l0) {
            fac = (((l0 - n) & 1) ? -1.0 : 1.0) * sqrt_binom_a(2 * l0, l0 + n), pa = l0 + n, pp = l0 - n;
        } else if (m == -l0) {
            fac = sqrt_binom_a(2 * l0, l0 + n), pa = l0 - n, pp = l0 + n;
        } else if (n == l0) {
            fac = sqrt_binom_a(2 * l0, l0 + m), pa = l0 + m, pp = l0 - m;
        } else {
            fac = (((l0 + m) & 1) ? -1.0 : 1.0) * sqrt_binom_a(2 * l0, l0 + m), pa = l0 - m, pp = l0 + m;
        }
        double c = 1.0, s = 1.0;
        for (int q = 0; q < pa; ++q) c *= ch;
        for (int q = 0; q < pp; ++q) s *= sh;
        double cur = fac * (c * s), prev = 0.0;
        d[dxi_off(l0) + (m + l0) * (2 * l0 + 1) + (n + l0)] = cur;
        for (int l = l0 + 1; l <= L; ++l) {
            double nx;
            if (l == 1) {
                nx = cb;
            } else {
                const double a2 = sqrt(((double)l * l - (double)m * m) * ((double)l * l - (double)n * n));
                const double den = (l - 1.0) * a2;
                const double t1 = (2.0 * l - 1.0) * (l * (l - 1.0) * cb - (double)m * n) / den;
                const bool has2 = abs(m) <= l - 2 && abs(n) <= l - 2;
                const double b2 = has2 ? sqrt(((double)(l - 1) * (l - 1) - (double)m * m) *
                                              ((double)(l - 1) * (l - 1) - (double)n * n))
                                       : 0.0;
                nx = t1 * cur - (has2 ? l * b2 / den * prev : 0.0);
            }
            prev = cur;
            cur = nx;
            d[dxi_off(l) + (m + l) * (2 * l + 1) + (n + l)] = cur;
        }
    }
    __syncthreads();
    const float* c = coef + (long long)p * ldc;
    // outputs: every (l, k, m), m = -l..l  (complex reference layout offset)
    int total = 0;
    for (int l = 0; l <= L; ++l) total += radial_count[l] * (2 * l + 1);
    for (int o = threadIdx.x; o < total; o += blockDim.x) {
        int l = 0;
        while (o >= block_off[l] + radial_count[l] * (2 * l + 1)) ++l;
        const int r = o - block_off[l];
        const int k = r / (2 * l + 1), m = r % (2 * l + 1) - l;
        const int base = block_off[l] + k * (2 * l + 1);
        const double* drow = d + dxi_off(l) + (m + l) * (2 * l + 1) + l;
        double re = 0.0, im = 0.0;
        for (int mp = -l; mp <= l; ++mp) {
            const int amp = abs(mp);
            double fre = c[base + (amp == 0 ? 0 : 2 * amp - 1)];
            double fim = amp == 0 ? 0.0 : (double)c[base + 2 * amp];
            if (mp < 0) {
                const double sg = (amp & 1) ? -1.0 : 1.0;
                fre *= sg;
                fim *= -sg;
            }
            // e^{-i m' g} f
            double sg_, cg_;
            sincos(mp * e.g, &sg_, &cg_);
            const double xr = cg_ * fre + sg_ * fim, xi = cg_ * fim - sg_ * fre;
            re += drow[mp] * xr;
            im += drow[mp] * xi;
        }
        double sa, ca;
        sincos(m * e.a, &sa, &ca);
        atomicAdd(&sum[o].x, ca * re + sa * im);
        atomicAdd(&sum[o].y, ca * im - sa * re);
    }
    __syncthreads();  // d is rebuilt for the next particle
    }
}

}  // namespace

void launch_average(const float* coef, int ldc, const double* quats, int count, int L, const int* block_off,
                    const int* radial_count, double* sum, cudaStream_t s) {
    if (count <= 0) return;
    const size_t smem = sizeof(double) * (size_t)(L + 1) * (2 * L + 1) * (2 * L + 3) / 3;
    if (smem <= 200 * 1024) {
        if (ensure_dynamic_smem(average_kernel, (int)smem) != cudaSuccess)
            throw std::runtime_error("average: shared-memory opt-in failed");
        average_kernel<<<count, 256, smem, s>>>(coef, ldc, quats, L, block_off, radial_count,
                                                reinterpret_cast<double2*>(sum), count, nullptr);
    } else {  // large bases: d stacks in global scratch, 1024 CTAs
        const int grid = count < 1024 ? count : 1024;
        double* scratch = nullptr;
        if (cudaMallocAsync(&scratch, smem * grid, s) != cudaSuccess) throw std::bad_alloc();
        average_kernel<<<grid, 256, 0, s>>>(coef, ldc, quats, L, block_off, radial_count,
                                            reinterpret_cast<double2*>(sum), count, scratch);
        cudaFreeAsync(scratch, s);
    }
    if (cudaGetLastError() != cudaSuccess) throw std::runtime_error("average kernel launch failed");
}

}  // namespace bmb
