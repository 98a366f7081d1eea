// Factored ball-harmonic expansion (kernel K2f): the four
// stages of expand() (src/basis.cpp:254-328) run per shift window on the
// device, radius by radius, instead of the dense pulled-back operator:
//   1. trilinear samples f(r_i, theta_t, phi_p) of the shifted window
//      (sample_trilinear + shift_volume, src/volume.cpp:19-67): FP64 sample
//      coordinates, FP32 tap weights, volumes read from a 4x4x4-brick copy;
//   2. unnormalized phi-DFT of every theta ring (dft_r2c_rows,
//      src/detail/fftw_util.cpp:16-28), folded over p <-> n_phi - p;
//   3. theta contraction with Pbar_l^m(u_t) w_t, folded over the GL symmetry
//      u_{n-1-t} = -u_t (Pbar_l^m(-u) = (-1)^(l+m) Pbar_l^m(u));
//   4. radial contraction c_lk j_l(lambda r_i) r_i^2 w_i 2pi/n_phi accumulated
//      into the real-packed coefficient rows.
// One CTA per window; stages 2-4 use FP32 tables with FP32 accumulation.
// Algorithmic work per window (DESIGN.md §3 K2f): 8 n_r n_theta n_phi taps +
// ~2 n_r n_theta (L+1) n_phi + 2 n_r tri(L) n_theta + n_r C FLOP — about
// 100x fewer than the dense 2 C V of the pulled-back operator.
#include "expand_factored.hpp"

namespace bmb {

namespace {

constexpr int kThreads = 256;

struct Smem {
    size_t cphi, sphi, st, u, tw, samp, F, G, acc, total;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) / 16 * 16; }

__host__ __device__ inline Smem smem_plan(const FactoredTables& T) {
    Smem s;
    const int L = T.L, half = T.np / 2;
    size_t o = 0;
    s.cphi = o;
    o = al16(o + sizeof(double) * T.np);
    s.sphi = o;
    o = al16(o + sizeof(double) * T.np);
    s.st = o;
    o = al16(o + sizeof(double) * T.nt);
    s.u = o;
    o = al16(o + sizeof(double) * T.nt);
    s.tw = o;
    o = al16(o + sizeof(float2) * (size_t)(half + 1) * (L + 1));
    s.samp = o;
    o = al16(o + sizeof(float) * (size_t)T.nt * T.np);
    s.F = o;
    o = al16(o + sizeof(float2) * (size_t)T.nt * (L + 1));
    s.G = o;
    o = al16(o + sizeof(float2) * (size_t)T.ntri);
    s.acc = o;
    o = al16(o + sizeof(float) * (size_t)T.coeffs);
    s.total = o;
    return s;
}

// 4x4x4 bricks (256 B): the 2x2x2 trilinear footprint of a sample then touches
// ~1.5 cache lines instead of 4 rows of the raster layout
__host__ __device__ inline long long brick_offset(int x, int y, int z, int nb) {
    return ((((long long)(z >> 2) * nb + (y >> 2)) * nb + (x >> 2)) << 6) + ((z & 3) << 4) + ((y & 3) << 2) + (x & 3);
}

__global__ void to_bricks_kernel(const float* __restrict__ in, long long in_stride, float* __restrict__ out, int n) {
    const float* v = in + (long long)blockIdx.y * in_stride;
    float* o = out + (long long)blockIdx.y * n * n * n;
    const int nb = n >> 2;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * n * n; i += gridDim.x * blockDim.x) {
        const int x = i % n, y = (i / n) % n, z = i / (n * n);
        o[brick_offset(x, y, z, nb)] = v[i];
    }
}

template <bool BRICK>
__global__ void __launch_bounds__(kThreads) expand_factored_kernel(FactoredTables T, const float* __restrict__ vols,
                                                                    long long vol_stride, const int* __restrict__ win_vol,
                                                                    const int* __restrict__ win_shift, float* __restrict__ out,
                                                                    int ldo) {
    extern __shared__ __align__(16) unsigned char sm[];
    const Smem P = smem_plan(T);
    double* cphi = reinterpret_cast<double*>(sm + P.cphi);
    double* sphi = reinterpret_cast<double*>(sm + P.sphi);
    double* st = reinterpret_cast<double*>(sm + P.st);
    double* uu = reinterpret_cast<double*>(sm + P.u);
    float2* tw = reinterpret_cast<float2*>(sm + P.tw);
    float* samp = reinterpret_cast<float*>(sm + P.samp);
    float2* F = reinterpret_cast<float2*>(sm + P.F);
    float2* G = reinterpret_cast<float2*>(sm + P.G);
    float* acc = reinterpret_cast<float*>(sm + P.acc);

    const int w = blockIdx.x, tid = threadIdx.x;
    const int n = T.n, L = T.L, nt = T.nt, np = T.np, half = np / 2, nl = L + 1;
    const float* __restrict__ v = vols + (long long)win_vol[w] * vol_stride;
    const int sx = win_shift[3 * w], sy = win_shift[3 * w + 1], sz = win_shift[3 * w + 2];
    for (int i = tid; i < np; i += kThreads) {
        cphi[i] = T.cphi[i];
        sphi[i] = T.sphi[i];
    }
    for (int i = tid; i < nt; i += kThreads) {
        st[i] = T.st[i];
        uu[i] = T.u[i];
    }
    for (int i = tid; i < (half + 1) * nl; i += kThreads) tw[i] = T.tw[i];
    for (int i = tid; i < T.coeffs; i += kThreads) acc[i] = 0.0f;
    const double h = 0.5 * n;
    __syncthreads();

    for (int ir = 0; ir < T.nr; ++ir) {
        const double r = T.r[ir];
        // 1. trilinear samples of the shifted window (zero outside the grid and
        //    where the shifted source leaves it)
        for (int s = tid; s < nt * np; s += kThreads) {
            const int t = s / np, p = s - t * np;
            const double rs = r * st[t];
            const double gx = rs * cphi[p] * h + h, gy = rs * sphi[p] * h + h, gz = r * uu[t] * h + h;
            const double fx0 = floor(gx), fy0 = floor(gy), fz0 = floor(gz);
            const int x0 = (int)fx0, y0 = (int)fy0, z0 = (int)fz0;
            const float fx = (float)(gx - fx0), fy = (float)(gy - fy0), fz = (float)(gz - fz0);
            // source voxel of the base tap and the +1 steps along each axis
            const int xs0 = x0 + sx, ys0 = y0 + sy, zs0 = z0 + sz;
            long long o0;
            int dx, dy, dz;
            if (BRICK) {
                o0 = brick_offset(xs0, ys0, zs0, n >> 2);
                dx = (xs0 & 3) != 3 ? 1 : 61;
                dy = (ys0 & 3) != 3 ? 4 : (n >> 2) * 64 - 12;
                dz = (zs0 & 3) != 3 ? 16 : (n >> 2) * (n >> 2) * 64 - 48;
            } else {
                o0 = ((long long)zs0 * n + ys0) * n + xs0;
                dx = 1;
                dy = n;
                dz = n * n;
            }
            // a tap contributes when it lies in the window grid and its source in the volume
            const bool vx0 = (unsigned)x0 < (unsigned)n && (unsigned)xs0 < (unsigned)n;
            const bool vx1 = (unsigned)(x0 + 1) < (unsigned)n && (unsigned)(xs0 + 1) < (unsigned)n;
            const bool vy0 = (unsigned)y0 < (unsigned)n && (unsigned)ys0 < (unsigned)n;
            const bool vy1 = (unsigned)(y0 + 1) < (unsigned)n && (unsigned)(ys0 + 1) < (unsigned)n;
            const bool vz0 = (unsigned)z0 < (unsigned)n && (unsigned)zs0 < (unsigned)n;
            const bool vz1 = (unsigned)(z0 + 1) < (unsigned)n && (unsigned)(zs0 + 1) < (unsigned)n;
            float val = 0.0f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {  // (y, z) rows of the footprint
                const int b = c & 1, a = c >> 1;
                if (!(b ? vy1 : vy0) || !(a ? vz1 : vz0)) continue;
                const long long orow = o0 + (b ? dy : 0) + (a ? dz : 0);
                const float v0 = vx0 ? __ldg(v + orow) : 0.0f;
                const float v1 = vx1 ? __ldg(v + orow + dx) : 0.0f;
                const float wyz = (b ? fy : 1.0f - fy) * (a ? fz : 1.0f - fz);
                val = fmaf(wyz, fmaf(fx, v1 - v0, v0), val);
            }
            samp[s] = val;
        }
        __syncthreads();
        // 2. phi-DFT: F[t][m] = sum_p f[t][p] e^{-2 pi i m p / n_phi}, folded
        for (int o = tid; o < nt * nl; o += kThreads) {
            const int t = o / nl, m = o - t * nl;
            const float* f = samp + t * np;
            float re = f[0] + ((m & 1) ? -f[half] : f[half]);
            float im = 0.0f;
            for (int p = 1; p < half; ++p) {
                const float2 c = tw[p * nl + m];  // (cos, -sin)
                re = fmaf(f[p] + f[np - p], c.x, re);
                im = fmaf(f[p] - f[np - p], c.y, im);
            }
            F[o] = make_float2(re, im);
        }
        __syncthreads();
        // 3. theta: G[l,m] = sum_t Pbar_l^m(u_t) w_t F[t][m], folded over t <-> nt-1-t
        for (int q = tid; q < T.ntri; q += kThreads) {
            const int2 lm = T.tri_lm[q];
            const float sgn = ((lm.x + lm.y) & 1) ? -1.0f : 1.0f;
            const float* pt = T.ptab + (size_t)q * nt;
            float re = 0.0f, im = 0.0f;
            for (int t = 0; t < nt / 2; ++t) {
                const float2 a = F[t * nl + lm.y], b = F[(nt - 1 - t) * nl + lm.y];
                const float wgt = __ldg(pt + t);
                re = fmaf(wgt, fmaf(sgn, b.x, a.x), re);
                im = fmaf(wgt, fmaf(sgn, b.y, a.y), im);
            }
            G[q] = make_float2(re, im);
        }
        __syncthreads();
        // 4. radial: row (l,k,m,part) += radial[(l,k)][i] * G[l,m].part
        for (int row = tid; row < T.coeffs; row += kThreads) {
            const int4 rm = T.rowmap[row];
            const float g = rm.y ? G[rm.x].y : G[rm.x].x;
            acc[row] = fmaf(__ldg(T.radial + (size_t)rm.z * T.nr + ir), g, acc[row]);
        }
        // (the next radius only rewrites samp / F / G after further barriers)
    }
    __syncthreads();
    float* o = out + (long long)w * ldo;
    for (int row = tid; row < T.coeffs; row += kThreads) o[row] = acc[row];
}

}  // namespace

size_t factored_smem_bytes(const FactoredTables& T) { return smem_plan(T).total; }

void launch_to_bricks(const float* in, long long in_stride, int count, float* out, int n, cudaStream_t s) {
    if (count <= 0) return;
    dim3 grid((n * n * n + 1023) / 1024, count);
    to_bricks_kernel<<<grid, 256, 0, s>>>(in, in_stride, out, n);
}

int launch_expand_factored(const FactoredTables& T, const float* vols, long long vol_stride, bool bricked,
                           const int* win_vol, const int* win_shift, int n_win, float* out, int ldo, cudaStream_t s) {
    if (n_win <= 0) return 0;
    const size_t smem = factored_smem_bytes(T);
    if (smem > 220 * 1024) return 1;
    if (bricked) {
        cudaFuncSetAttribute(expand_factored_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        expand_factored_kernel<true><<<n_win, kThreads, smem, s>>>(T, vols, vol_stride, win_vol, win_shift, out, ldo);
    } else {
        cudaFuncSetAttribute(expand_factored_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        expand_factored_kernel<false><<<n_win, kThreads, smem, s>>>(T, vols, vol_stride, win_vol, win_shift, out, ldo);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace bmb
