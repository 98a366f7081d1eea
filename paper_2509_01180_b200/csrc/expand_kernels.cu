// Expansion (kernel K2) side kernels: window gather + FP16 split (the GEMM's B
// operand), per-volume power-of-two scales, window norms, layout conversion.
#include <cuda_fp16.h>

#include "kernels.cuh"

namespace bmb {

// B[w][k] = vol_p[voxel_k + s_w] / scale_p (zero where the shifted source leaves
// the grid: shift_volume, src/volume.cpp:50-67), split into FP16 hi + lo.
__global__ void gather_windows_kernel(const float* __restrict__ vols, long long vol_stride,
                                      const int* __restrict__ win_vol,
                                      const int* __restrict__ win_shift, int n_win,
                                      const float* __restrict__ vol_scale,
                                      const int* __restrict__ voxels, int support, int k_pad,
                                      int n, __half* __restrict__ b_hi, __half* __restrict__ b_lo,
                                      float* __restrict__ col_scale) {
    const int w = blockIdx.y;
    if (w >= n_win) return;
    const int p = win_vol[w];
    const int sx = win_shift[3 * w], sy = win_shift[3 * w + 1], sz = win_shift[3 * w + 2];
    const float inv = 1.0f / vol_scale[p];
    const float* v = vols + (long long)p * vol_stride;
    __half* hi = b_hi + (long long)w * k_pad;
    __half* lo = b_lo + (long long)w * k_pad;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < k_pad; k += gridDim.x * blockDim.x) {
        float x = 0.0f;
        if (k < support) {
            const int vox = voxels[k];
            const int xx = vox % n + sx, yy = (vox / n) % n + sy, zz = vox / (n * n) + sz;
            if ((unsigned)xx < (unsigned)n && (unsigned)yy < (unsigned)n && (unsigned)zz < (unsigned)n)
                x = v[((long long)zz * n + yy) * n + xx] * inv;
        }
        const __half h = __float2half_rn(x);
        hi[k] = h;
        lo[k] = __float2half_rn(x - __half2float(h));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) col_scale[w] = vol_scale[p];
}

void launch_gather_windows(const float* vols, long long vol_stride, const int* win_vol,
                           const int* win_shift, int n_win, const float* vol_scale,
                           const int* voxels, int support, int k_pad, int n, __half* b_hi,
                           __half* b_lo, float* col_scale, cudaStream_t s) {
    if (n_win <= 0) return;
    dim3 grid((k_pad + 1023) / 1024, n_win);
    gather_windows_kernel<<<grid, 256, 0, s>>>(vols, vol_stride, win_vol, win_shift, n_win,
                                               vol_scale, voxels, support, k_pad, n, b_hi, b_lo,
                                               col_scale);
}

// scale_p = smallest power of two >= max |vol_p| (1 for an all-zero volume)
__global__ void absmax_scale_kernel(const float* __restrict__ vols, long long stride,
                                    float* __restrict__ scale) {
    const float* v = vols + (long long)blockIdx.x * stride;
    float m = 0.0f;
    for (long long i = threadIdx.x; i < stride; i += blockDim.x) m = fmaxf(m, fabsf(v[i]));
    __shared__ float red[32];
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0f;
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0) {
            float s = 1.0f;
            if (m > 0.0f) {
                int e;
                const float f = frexpf(m, &e);
                s = ldexpf(1.0f, f == 0.5f ? e - 1 : e);
            }
            scale[blockIdx.x] = s;
        }
    }
}

void launch_absmax_scale(const float* vols, int count, long long stride, float* scale,
                         cudaStream_t s) {
    if (count > 0) absmax_scale_kernel<<<count, 512, 0, s>>>(vols, stride, scale);
}

// ||f_hat|| = sqrt(sum_all_m |f_klm|^2) = sqrt(sum_rows w_r c_r^2)  (basis.cpp:166-172)
__global__ void window_norms_kernel(const float* __restrict__ coef, int ldc, int rows,
                                    const float* __restrict__ weight, double* __restrict__ norm) {
    const float* c = coef + (long long)blockIdx.x * ldc;
    double acc = 0.0;
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
        const double x = c[r];
        acc += weight[r] * x * x;
    }
    __shared__ double red[32];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (threadIdx.x == 0) norm[blockIdx.x] = sqrt(acc);
    }
}

void launch_window_norms(const float* coef, int n_win, int ldc, const Geometry& geo,
                         double* norm, cudaStream_t s) {
    if (n_win > 0) window_norms_kernel<<<n_win, 256, 0, s>>>(coef, ldc, geo.coeffs, geo.row_weight, norm);
}

// real-packed rows -> the reference's complex layout (block l, row k, column m+l),
// filling m < 0 by (-1)^m conj (src/basis.cpp:325)
__global__ void to_complex_kernel(const float* __restrict__ coef, int ldc, int rows,
                                  const int4* __restrict__ lkm, const int* __restrict__ block_off,
                                  double2* __restrict__ out) {
    const float* c = coef + (long long)blockIdx.y * ldc;
    double2* o = out + (long long)blockIdx.y * rows;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        const int4 q = lkm[r];  // (l, k, m, part)
        if (q.w != 0) continue;
        const int l = q.x, k = q.y, m = q.z;
        const int base = block_off[l] + (k - 1) * (2 * l + 1) + l;
        const double re = c[r];
        const double im = m > 0 ? (double)c[r + 1] : 0.0;
        o[base + m] = make_double2(re, im);
        if (m > 0) {
            const double sg = (m & 1) ? -1.0 : 1.0;
            o[base - m] = make_double2(sg * re, -sg * im);
        }
    }
}

void launch_to_complex(const float* coef, int n_win, int ldc, const Geometry& geo, double* out,
                       cudaStream_t s) {
    if (n_win <= 0) return;
    dim3 grid((geo.coeffs + 255) / 256, n_win);
    to_complex_kernel<<<grid, 256, 0, s>>>(coef, ldc, geo.coeffs, geo.row_lkm, geo.block_off,
                                           reinterpret_cast<double2*>(out));
}

// reference complex layout -> real-packed rows (Re of m >= 0, Im of m > 0)
__global__ void from_complex_kernel(const double2* __restrict__ in, int rows,
                                    const int4* __restrict__ lkm, const int* __restrict__ block_off,
                                    float* __restrict__ out, int ldo) {
    const double2* c = in + (long long)blockIdx.y * rows;
    float* o = out + (long long)blockIdx.y * ldo;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        const int4 q = lkm[r];
        const int l = q.x, k = q.y, m = q.z;
        const double2 v = c[block_off[l] + (k - 1) * (2 * l + 1) + l + m];
        o[r] = (float)(q.w == 0 ? v.x : v.y);
    }
}

void launch_from_complex(const double* in, int count, const Geometry& geo, float* out, int ldo,
                         cudaStream_t s) {
    if (count <= 0) return;
    dim3 grid((geo.coeffs + 255) / 256, count);
    from_complex_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const double2*>(in), geo.coeffs,
                                             geo.row_lkm, geo.block_off, out, ldo);
}

}  // namespace bmb
