// Factored ball-harmonic expansion (kernel K2f): the four
// stages of expand() (src/basis.cpp:254-328) run per shift window on the
// device, radius by radius, instead of the dense pulled-back operator:
//   1. trilinear samples f(r_i, theta_t, phi_p) of the shifted window
//      (sample_trilinear + shift_volume, src/volume.cpp:19-67): base voxel and
//      FP32 weights from a per-sample table (FP64 coordinates r * (h d_tp) + h,
//      computed once on the host), FP32 taps;
//   2. unnormalized phi-DFT of every theta ring (dft_r2c_rows,
//      src/detail/fftw_util.cpp:16-28), folded over p <-> n_phi - p, with each
//      thread's order m fixed so its twiddle row lives in registers;
//   3. theta contraction with Pbar_l^m(u_t) w_t, folded over the GL symmetry
//      u_{n-1-t} = -u_t (Pbar_l^m(-u) = (-1)^(l+m) Pbar_l^m(u)), written in the
//      packed real row layout [Re m0, Re m1, Im m1, ...] of each degree;
//   4. radial contraction c_lk j_l(lambda r_i) r_i^2 w_i 2pi/n_phi into
//      register accumulators (a fixed set of real-packed rows per thread).
// One CTA per window; stages 2-4 in FP32.  Algorithmic work per window
// (DESIGN.md §3 K2f): 16 S + 4 n_phi n_r n_theta (L+1) + 4 n_r tri(L) n_theta +
// 2 n_r C FLOP, S = n_r n_theta n_phi — 4.47 MFLOP at config 2, about 120x fewer
// than the dense 2 C V of the pulled-back operator.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <set>
#include <type_traits>
#include <vector>

#include "smem_attr.hpp"
#include "expand_factored.hpp"
#include "sm100_ptx.cuh"

namespace bmb {

namespace {

constexpr int kThreads = 256;
#ifndef BMB_EXPAND_RC
#define BMB_EXPAND_RC 4
#endif
constexpr int kRC = BMB_EXPAND_RC;  // radii sampled per pass (lanes run along the ray: adjacent radii share cache lines)

struct Smem {
    size_t samp, F, G, rad, rowpack, total;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) / 16 * 16; }

__host__ __device__ inline Smem smem_plan(const FactoredTables& T) {
    Smem s;
    size_t o = 0;
    s.samp = o;
    o = al16(o + sizeof(float) * (size_t)kRC * T.nt * T.np);
    s.F = o;
    o = al16(o + sizeof(float2) * (size_t)T.nt * (T.L + 1));
    s.G = o;
    o = al16(o + sizeof(float) * (size_t)(T.L + 1) * (T.L + 1));
    s.rad = o;
    o = al16(o + sizeof(float) * (size_t)T.pairs);
    s.rowpack = o;
    o = al16(o + sizeof(int) * (size_t)T.coeffs);
    s.total = o;
    return s;
}

// phi-DFT twiddles of the common n_phi (= 2L + 2 for L = 8 / 16 / 20 / 24) as
// compile-time constants: the FFMAs take them as immediates, no table loads
// compile-time twiddles (Taylor series in double, |x| <= pi): FFMA immediates
constexpr double ct_sin(double x) {
    double term = x, sum = x;
    for (int n = 1; n < 40; ++n) {
        term *= -x * x / ((2.0 * n) * (2.0 * n + 1.0));
        sum += term;
    }
    return sum;
}
constexpr double ct_cos(double x) {
    double term = 1.0, sum = 1.0;
    for (int n = 1; n < 40; ++n) {
        term *= -x * x / ((2.0 * n - 1.0) * (2.0 * n));
        sum += term;
    }
    return sum;
}
template <int NP>
struct DftTab {
    float c[NP / 2][NP / 2] = {};
    float s[NP / 2][NP / 2] = {};
    constexpr DftTab() {
        for (int m = 0; m < NP / 2; ++m)
            for (int p = 0; p < NP / 2; ++p) {
                const long long a = ((long long)m * p) % NP;
                double x = 2.0 * 3.14159265358979323846 * (double)a / NP;
                if (x > 3.14159265358979323846) x -= 2.0 * 3.14159265358979323846;
                c[m][p] = (float)ct_cos(x);
                s[m][p] = (float)-ct_sin(x);
            }
    }
};
template <int NP, int M0, int MH>
__device__ __forceinline__ void dft_ring(const float* f, float2* Frow) {
    constexpr int H = NP / 2;
    constexpr DftTab<NP> tab{};
    float a[H], b[H];
#pragma unroll
    for (int p = 1; p < H; ++p) {
        const float x = f[p], y = f[NP - p];
        a[p] = x + y;
        b[p] = x - y;
    }
    const float f0 = f[0], fh = f[H];
#pragma unroll
    for (int m = M0; m < MH; ++m) {
        float re = f0 + ((m & 1) ? -fh : fh);
        float im = 0.0f;
#pragma unroll
        for (int p = 1; p < H; ++p) {
            re = fmaf(a[p], tab.c[m][p], re);
            im = fmaf(b[p], tab.s[m][p], im);
        }
        Frow[m] = make_float2(re, im);
    }
}

// compile-time knobs (measured defaults): the radial stage's row map in registers,
// phi-DFT order groups per ring (2 groups of 64 threads)
#ifndef BMB_RP_REG
#define BMB_RP_REG 1
#endif
#ifndef BMB_DFT_GROUPS
#define BMB_DFT_GROUPS 2
#endif
// HALF: compile-time bound on n_phi / 2 (twiddles in registers); RPT: bound on
// the real-packed rows per thread (accumulators in registers)
#ifndef BMB_EXPAND_MINB
#define BMB_EXPAND_MINB 3
#endif
template <int HALF, int RPT, int NPC>
__global__ void __launch_bounds__(kThreads, BMB_EXPAND_MINB) expand_factored_kernel(FactoredTables T, const float* __restrict__ vols,
                                                                    long long vol_stride, const int* __restrict__ win_vol,
                                                                    const int* __restrict__ win_shift, float* __restrict__ out,
                                                                    int ldo, const float2* __restrict__ pairs) {
    extern __shared__ __align__(16) unsigned char sm[];
    const Smem P = smem_plan(T);
    float* samp = reinterpret_cast<float*>(sm + P.samp);
    float2* F = reinterpret_cast<float2*>(sm + P.F);
    float* Gp = reinterpret_cast<float*>(sm + P.G);       // packed real rows of degree l at l^2
    float* rad = reinterpret_cast<float*>(sm + P.rad);    // radial table slice of the current radius
    int* rowpack = reinterpret_cast<int*>(sm + P.rowpack);

    const int w = blockIdx.x, tid = threadIdx.x;
    const int n = T.n, L = T.L, nt = T.nt, np = T.np, half = np / 2, nl = L + 1;
    const int nsamp = nt * np;
    const float* __restrict__ v = vols + (long long)win_vol[w] * vol_stride;
    const float2* __restrict__ vp = pairs ? pairs + win_vol[w] * pair_volume_elems(T.n) : nullptr;
    const int sx = win_shift[3 * w], sy = win_shift[3 * w + 1], sz = win_shift[3 * w + 2];
    for (int i = tid; i < T.coeffs; i += kThreads) rowpack[i] = T.rowpack[i];
    // DFT role: fixed order m, rings t = tg, tg + TG, ...
    const int TG = kThreads / nl;
    const int dm = tid % nl, dtg = tid / nl;
    float2 tw[HALF];
#pragma unroll
    for (int p = 1; p < HALF; ++p) tw[p] = p < half ? T.tw[p * nl + dm] : make_float2(0.f, 0.f);
    float acc[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) acc[q] = 0.0f;
#if BMB_RP_REG
    int rpr[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) rpr[q] = tid + q * kThreads < T.coeffs ? T.rowpack[tid + q * kThreads] : 0;
#endif
    // theta role of the specialised kernel (n_theta = NPC, tri(L) <= threads): one
    // (l, m) per thread, its weights P_l^m(u_t) w_t in registers for all radii
    float th_w[NPC > 0 ? NPC / 2 : 1];
    int th_m = 0, th_base = 0;
    float th_sgn = 1.0f;
    if constexpr (NPC > 0 && (NPC / 2) * (NPC / 2 + 1) / 2 <= kThreads) {
        if (tid < T.ntri) {
            const int2 lm = T.tri_lm[tid];
            th_m = lm.y;
            th_base = lm.x * lm.x;
            th_sgn = ((lm.x + lm.y) & 1) ? -1.0f : 1.0f;
#pragma unroll
            for (int t = 0; t < NPC / 2; ++t) th_w[t] = __ldg(T.ptab + (size_t)tid * NPC + t);
        }
    }
    __syncthreads();

    for (int ir = 0; ir < T.nr; ++ir) {
        const int rc = ir % kRC;
        if (rc == 0) {
            // 1. trilinear samples of the shifted window for radii ir .. ir+kRC-1
            //    (zero outside the grid and where the shifted source leaves it);
            //    0 < g < n, so truncation = floor.  Item = (ray, radius), radius fastest.
            const int nrc = min(kRC, T.nr - ir);
            const int items = nsamp * kRC;
            // the footprint of the next item is loaded one iteration ahead
            auto entry = [&](int it) {
                const int s = it / kRC, j = it - s * kRC;
                return (it < items && j < nrc) ? __ldg(T.samp + (size_t)s * T.nr + ir + j) : make_int4(0, 0, 0, 0);
            };
            int4 e_next = entry(tid);
            for (int it = tid; it < items; it += kThreads) {
                const int s = it / kRC, j = it - s * kRC;
                const int4 e = e_next;
                e_next = entry(it + kThreads);
                if (j >= nrc) continue;
                const int x0 = e.x & 1023, y0 = (e.x >> 10) & 1023, z0 = (e.x >> 20) & 1023;
                const float fx = __int_as_float(e.y), fy = __int_as_float(e.z), fz = __int_as_float(e.w);
                const int xs0 = x0 + sx, ys0 = y0 + sy, zs0 = z0 + sz;
                const bool vx0 = (unsigned)x0 < (unsigned)n && (unsigned)xs0 < (unsigned)n;
                const bool vx1 = (unsigned)(x0 + 1) < (unsigned)n && (unsigned)(xs0 + 1) < (unsigned)n;
                const bool vy0 = (unsigned)y0 < (unsigned)n && (unsigned)ys0 < (unsigned)n;
                const bool vy1 = (unsigned)(y0 + 1) < (unsigned)n && (unsigned)(ys0 + 1) < (unsigned)n;
                const bool vz0 = (unsigned)z0 < (unsigned)n && (unsigned)zs0 < (unsigned)n;
                const bool vz1 = (unsigned)(z0 + 1) < (unsigned)n && (unsigned)(zs0 + 1) < (unsigned)n;
                float val = 0.0f;
                if (vp) {  // x-paired layout: one 8-byte load per (y, z) row; vx0 || vx1 => -1 <= xs0 < n
                    const int o0 = (zs0 * n + ys0) * (n + 1) + xs0 + 1;  // within one volume: 32-bit
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int bb = c & 1, aa = c >> 1;
                        const bool vr = (bb ? vy1 : vy0) && (aa ? vz1 : vz0);
                        const float2 pr = (vr && (vx0 || vx1))
                                              ? __ldg(vp + o0 + (bb ? n + 1 : 0) + (aa ? n * (n + 1) : 0))
                                              : make_float2(0.0f, 0.0f);
                        const float v0 = vx0 ? pr.x : 0.0f;
                        const float v1 = vx1 ? pr.y : 0.0f;
                        const float wyz = (bb ? fy : 1.0f - fy) * (aa ? fz : 1.0f - fz);
                        val = fmaf(wyz, fmaf(fx, v1 - v0, v0), val);
                    }
                } else {
                    const int o0 = (zs0 * n + ys0) * n + xs0;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {  // (y, z) rows of the footprint
                        const int bb = c & 1, aa = c >> 1;
                        const bool vr = (bb ? vy1 : vy0) && (aa ? vz1 : vz0);
                        const float* row = v + o0 + (bb ? n : 0) + (aa ? n * n : 0);
                        const float v0 = (vr && vx0) ? __ldg(row) : 0.0f;
                        const float v1 = (vr && vx1) ? __ldg(row + 1) : 0.0f;
                        const float wyz = (bb ? fy : 1.0f - fy) * (aa ? fz : 1.0f - fz);
                        val = fmaf(wyz, fmaf(fx, v1 - v0, v0), val);
                    }
                }
                samp[j * nsamp + s] = val;
            }
        }
        // radial slice of this radius (read after the barriers below)
        for (int i = tid; i < T.pairs; i += kThreads) rad[i] = T.radial_t[(size_t)ir * T.pairs + i];
        __syncthreads();
        // 2. phi-DFT: F[t][m] = sum_p f[t][p] e^{-2 pi i m p / n_phi}, folded
        if constexpr (NPC > 0) {  // one ring per thread, all orders
            // orders split over two groups of 64 threads (whole warps: no divergence)
            constexpr int MH = NPC / 2;
            static_assert(NPC <= 64, "one ring per thread of a 64-thread group");
#if BMB_DFT_GROUPS == 4
            constexpr int Q = (MH + 3) / 4;
            {
                const int it = tid, t = it & 63, g = it >> 6;
                if (t < nt) {
                    const float* f = samp + rc * nsamp + t * np;
                    if (g == 0) dft_ring<NPC, 0, Q>(f, F + t * nl);
                    else if (g == 1) dft_ring<NPC, Q, 2 * Q>(f, F + t * nl);
                    else if (g == 2) dft_ring<NPC, 2 * Q, 3 * Q>(f, F + t * nl);
                    else dft_ring<NPC, 3 * Q, MH>(f, F + t * nl);
                }
            }
#else
            constexpr int MS = (MH + 1) / 2;
            for (int it = tid; it < 128; it += kThreads) {
                const int t = it & 63;
                if (t >= nt) continue;
                if (it < 64) dft_ring<NPC, 0, MS>(samp + rc * nsamp + t * np, F + t * nl);
                else dft_ring<NPC, MS, MH>(samp + rc * nsamp + t * np, F + t * nl);
            }
#endif
        } else if (dtg < TG) {
            for (int t = dtg; t < nt; t += TG) {
                const float* f = samp + rc * nsamp + t * np;
                float re = f[0] + ((dm & 1) ? -f[half] : f[half]);
                float im = 0.0f;
#pragma unroll
                for (int p = 1; p < HALF; ++p) {
                    if (p < half) {
                        const float a = f[p], b = f[np - p];
                        re = fmaf(a + b, tw[p].x, re);
                        im = fmaf(a - b, tw[p].y, im);
                    }
                }
                F[t * nl + dm] = make_float2(re, im);
            }
        }
        __syncthreads();
        // 3. theta: G[l,m] = sum_t Pbar_l^m(u_t) w_t F[t][m], folded over t <-> nt-1-t
        if constexpr (NPC > 0 && (NPC / 2) * (NPC / 2 + 1) / 2 <= kThreads) {  // n_theta = n_phi = NPC: the thread's P.w row in registers
            if (tid < T.ntri) {
                float re = 0.0f, im = 0.0f;
#pragma unroll
                for (int t = 0; t < NPC / 2; ++t) {
                    const float2 a = F[t * nl + th_m], b = F[(NPC - 1 - t) * nl + th_m];
                    re = fmaf(th_w[t], fmaf(th_sgn, b.x, a.x), re);
                    im = fmaf(th_w[t], fmaf(th_sgn, b.y, a.y), im);
                }
                if (th_m == 0) {
                    Gp[th_base] = re;
                } else {
                    Gp[th_base + 2 * th_m - 1] = re;
                    Gp[th_base + 2 * th_m] = im;
                }
            }
        } else
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
            const int base = lm.x * lm.x;
            if (lm.y == 0) {
                Gp[base] = re;
            } else {
                Gp[base + 2 * lm.y - 1] = re;
                Gp[base + 2 * lm.y] = im;
            }
        }
        __syncthreads();
        // 4. radial: row (l, k, j) += radial[(l,k)][i] * Gp[l^2 + j]
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int row = tid + q * kThreads;
            if (row < T.coeffs) {
#if BMB_RP_REG
                const int rp = rpr[q];
#else
                const int rp = rowpack[row];
#endif
                acc[q] = fmaf(rad[rp >> 16], Gp[rp & 0xffff], acc[q]);
            }
        }
        // rad (and samp at the next chunk) are rewritten: all threads must be done here
        __syncthreads();
    }
    float* o = out + (long long)w * ldo;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int row = tid + q * kThreads;
        if (row < T.coeffs) o[row] = acc[q];
    }
}

// ---------------------------------------------------------------- large bases
// Bases beyond the register-resident specialisations (the paper's L = 42,
// C = 34,949 at 64^3): stages 1-3 per radius write the packed theta output
// G[w][i][(L+1)^2] to global memory (kernel A), then the radial contraction
// out[w][row] = sum_i radial[i][pair(row)] G[w][i][lm(row)] runs as its own
// kernel (B) with one thread per (window, row) -- no per-thread accumulator bound.
__global__ void __launch_bounds__(kThreads) expand_theta_kernel(FactoredTables T, const float* __restrict__ vols,
                                                                long long vol_stride, const int* __restrict__ win_vol,
                                                                const int* __restrict__ win_shift, int w0,
                                                                float* __restrict__ G, const float2* __restrict__ pairs) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int n = T.n, L = T.L, nt = T.nt, np = T.np, half = np / 2, nl = L + 1, nsamp = nt * np;
    float* samp = reinterpret_cast<float*>(sm);
    float2* F = reinterpret_cast<float2*>(sm + al16(sizeof(float) * (size_t)nsamp));
    const int w = w0 + blockIdx.x, tid = threadIdx.x;
    const float* __restrict__ v = vols + (long long)win_vol[w] * vol_stride;
    const float2* __restrict__ vp = pairs ? pairs + win_vol[w] * pair_volume_elems(n) : nullptr;
    const int sx = win_shift[3 * w], sy = win_shift[3 * w + 1], sz = win_shift[3 * w + 2];
    float* Gw = G + (size_t)blockIdx.x * T.nr * nl * nl;
    for (int ir = 0; ir < T.nr; ++ir) {
        for (int s = tid; s < nsamp; s += kThreads) {  // 1. trilinear samples of radius ir
            const int4 e = __ldg(T.samp + (size_t)s * T.nr + ir);
            const int x0 = e.x & 1023, y0 = (e.x >> 10) & 1023, z0 = (e.x >> 20) & 1023;
            const float fx = __int_as_float(e.y), fy = __int_as_float(e.z), fz = __int_as_float(e.w);
            const int xs0 = x0 + sx, ys0 = y0 + sy, zs0 = z0 + sz;
            const bool vx0 = (unsigned)x0 < (unsigned)n && (unsigned)xs0 < (unsigned)n;
            const bool vx1 = (unsigned)(x0 + 1) < (unsigned)n && (unsigned)(xs0 + 1) < (unsigned)n;
            const bool vy0 = (unsigned)y0 < (unsigned)n && (unsigned)ys0 < (unsigned)n;
            const bool vy1 = (unsigned)(y0 + 1) < (unsigned)n && (unsigned)(ys0 + 1) < (unsigned)n;
            const bool vz0 = (unsigned)z0 < (unsigned)n && (unsigned)zs0 < (unsigned)n;
            const bool vz1 = (unsigned)(z0 + 1) < (unsigned)n && (unsigned)(zs0 + 1) < (unsigned)n;
            float val = 0.0f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int bb = c & 1, aa = c >> 1;
                const bool vr = (bb ? vy1 : vy0) && (aa ? vz1 : vz0);
                float v0 = 0.0f, v1 = 0.0f;
                if (vp) {
                    const long long o = ((long long)(zs0 + aa) * n + ys0 + bb) * (n + 1) + xs0 + 1;
                    const float2 pr = (vr && (vx0 || vx1)) ? __ldg(vp + o) : make_float2(0.0f, 0.0f);
                    v0 = vx0 ? pr.x : 0.0f;
                    v1 = vx1 ? pr.y : 0.0f;
                } else {
                    const float* row = v + ((long long)(zs0 + aa) * n + ys0 + bb) * n + xs0;
                    v0 = (vr && vx0) ? __ldg(row) : 0.0f;
                    v1 = (vr && vx1) ? __ldg(row + 1) : 0.0f;
                }
                const float wyz = (bb ? fy : 1.0f - fy) * (aa ? fz : 1.0f - fz);
                val = fmaf(wyz, fmaf(fx, v1 - v0, v0), val);
            }
            samp[s] = val;
        }
        __syncthreads();
        for (int q = tid; q < nt * nl; q += kThreads) {  // 2. folded phi-DFT per (ring, order)
            const int t = q / nl, m = q - t * nl;
            const float* f = samp + t * np;
            float re = f[0] + ((m & 1) ? -f[half] : f[half]);
            float im = 0.0f;
            for (int p = 1; p < half; ++p) {
                const float2 tw = __ldg(T.tw + p * nl + m);
                const float a = f[p], b = f[np - p];
                re = fmaf(a + b, tw.x, re);
                im = fmaf(a - b, tw.y, im);
            }
            F[q] = make_float2(re, im);
        }
        __syncthreads();
        float* Gr = Gw + (size_t)ir * nl * nl;
        for (int q = tid; q < T.ntri; q += kThreads) {  // 3. folded theta contraction
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
            const int base = lm.x * lm.x;
            if (lm.y == 0) {
                Gr[base] = re;
            } else {
                Gr[base + 2 * lm.y - 1] = re;
                Gr[base + 2 * lm.y] = im;
            }
        }
        __syncthreads();
    }
}

__global__ void expand_radial_kernel(FactoredTables T, const float* __restrict__ G, int w0, float* __restrict__ out,
                                     int ldo) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= T.coeffs) return;
    const int nl2 = (T.L + 1) * (T.L + 1);
    const int rp = __ldg(T.rowpack + row), pr = rp >> 16;
    const float* g = G + (size_t)blockIdx.y * T.nr * nl2 + (rp & 0xffff);
    float acc = 0.0f;
    for (int i = 0; i < T.nr; ++i) acc = fmaf(__ldg(T.radial_t + (size_t)i * T.pairs + pr), g[(size_t)i * nl2], acc);
    out[(long long)(w0 + blockIdx.y) * ldo + row] = acc;
}

int launch_split(const FactoredTables& T, const float* vols, long long vol_stride, const int* win_vol,
                 const int* win_shift, int n_win, float* out, int ldo, cudaStream_t s, const float2* pairs) {
    const size_t smem = al16(sizeof(float) * (size_t)T.nt * T.np) + sizeof(float2) * (size_t)T.nt * (T.L + 1);
    if (smem > 220 * 1024) return 1;
    if (ensure_dynamic_smem(expand_theta_kernel, (int)smem) != cudaSuccess) return 2;
    const size_t per = sizeof(float) * (size_t)T.nr * (T.L + 1) * (T.L + 1);
    const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)n_win, (size_t(2) << 30) / per));
    float* G = nullptr;
    if (cudaMallocAsync(&G, per * chunk, s) != cudaSuccess) return 2;
    for (int w0 = 0; w0 < n_win; w0 += chunk) {
        const int cnt = std::min(chunk, n_win - w0);
        expand_theta_kernel<<<cnt, kThreads, smem, s>>>(T, vols, vol_stride, win_vol, win_shift, w0, G, pairs);
        expand_radial_kernel<<<dim3((T.coeffs + 255) / 256, cnt), 256, 0, s>>>(T, G, w0, out, ldo);
    }
    cudaFreeAsync(G, s);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

// ---------------------------------------------------------------- window pairs
// Two windows per CTA (consecutive windows of the alignment's shift lists: the
// same particle, shifts a voxel or two apart).  Each sample's footprint is
// loaded and decoded once for both windows and the second window's gathers
// mostly hit the L1 lines the first one pulled in; the phi-DFT of the pair keeps
// all 256 threads busy (2 windows x 2 order groups x 64 rings) and the theta
// threads reuse their register weights for both.  Same FP32 values and FMA order
// per window as expand_factored_kernel (bit-identical coefficients).
#ifndef BMB_EXPAND_PAIR_MINB
#define BMB_EXPAND_PAIR_MINB 2
#endif
struct SmemPair {
    size_t samp, F, G, rad, total;
};
__host__ __device__ inline SmemPair smem_plan_pair(const FactoredTables& T) {
    SmemPair s;
    size_t o = 0;
    s.samp = o;
    o = al16(o + 2 * sizeof(float) * (size_t)kRC * T.nt * T.np);
    s.F = o;
    o = al16(o + 2 * sizeof(float2) * (size_t)T.nt * (T.L + 1));
    s.G = o;
    o = al16(o + 2 * sizeof(float) * (size_t)(T.L + 1) * (T.L + 1));
    s.rad = o;
    o = al16(o + sizeof(float) * (size_t)T.pairs);
    s.total = o;
    return s;
}

template <int RPT, int NPC>
__global__ void __launch_bounds__(kThreads, BMB_EXPAND_PAIR_MINB)
    expand_pair_kernel(FactoredTables T, const float* __restrict__ vols, long long vol_stride,
                       const int* __restrict__ win_vol, const int* __restrict__ win_shift, int n_win,
                       float* __restrict__ out, int ldo, const float2* __restrict__ pairs) {
    static_assert(NPC > 0 && NPC <= 64 && (NPC / 2) * (NPC / 2 + 1) / 2 <= kThreads, "specialised shapes only");
    extern __shared__ __align__(16) unsigned char sm[];
    const SmemPair P = smem_plan_pair(T);
    const int n = T.n, nt = T.nt, np = NPC, nl = T.L + 1, nsamp = nt * np;
    float* samp = reinterpret_cast<float*>(sm + P.samp);          // [2][kRC][nsamp]
    float2* F = reinterpret_cast<float2*>(sm + P.F);              // [2][nt][nl]
    float* Gp = reinterpret_cast<float*>(sm + P.G);               // [2][nl^2]
    float* rad = reinterpret_cast<float*>(sm + P.rad);
    const int tid = threadIdx.x;
    const int wa = 2 * blockIdx.x;
    const bool two = wa + 1 < n_win;
    const int wb = two ? wa + 1 : wa;
    const float* __restrict__ v[2] = {vols + (long long)win_vol[wa] * vol_stride,
                                      vols + (long long)win_vol[wb] * vol_stride};
    const float2* __restrict__ vp[2] = {pairs ? pairs + win_vol[wa] * pair_volume_elems(n) : nullptr,
                                        pairs ? pairs + win_vol[wb] * pair_volume_elems(n) : nullptr};
    int sh[2][3];
#pragma unroll
    for (int q = 0; q < 3; ++q) sh[0][q] = win_shift[3 * wa + q], sh[1][q] = win_shift[3 * wb + q];
    float acc[2][RPT];
    int rpr[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        acc[0][q] = acc[1][q] = 0.0f;
        rpr[q] = tid + q * kThreads < T.coeffs ? T.rowpack[tid + q * kThreads] : 0;
    }
    float th_w[NPC / 2];
    int th_m = 0, th_base = 0;
    float th_sgn = 1.0f;
    if (tid < T.ntri) {
        const int2 lm = T.tri_lm[tid];
        th_m = lm.y;
        th_base = lm.x * lm.x;
        th_sgn = ((lm.x + lm.y) & 1) ? -1.0f : 1.0f;
#pragma unroll
        for (int t = 0; t < NPC / 2; ++t) th_w[t] = __ldg(T.ptab + (size_t)tid * NPC + t);
    }
    __syncthreads();
    for (int ir = 0; ir < T.nr; ++ir) {
        const int rc = ir % kRC;
        if (rc == 0) {
            const int nrc = min(kRC, T.nr - ir);
            const int items = nsamp * kRC;
            auto entry = [&](int it) {
                const int s = it / kRC, j = it - s * kRC;
                return (it < items && j < nrc) ? __ldg(T.samp + (size_t)s * T.nr + ir + j) : make_int4(0, 0, 0, 0);
            };
            int4 e_next = entry(tid);
            for (int it = tid; it < items; it += kThreads) {
                const int s = it / kRC, j = it - s * kRC;
                const int4 e = e_next;
                e_next = entry(it + kThreads);
                if (j >= nrc) continue;
                const int x0 = e.x & 1023, y0 = (e.x >> 10) & 1023, z0 = (e.x >> 20) & 1023;
                const float fx = __int_as_float(e.y), fy = __int_as_float(e.z), fz = __int_as_float(e.w);
                const bool gx0 = (unsigned)x0 < (unsigned)n, gx1 = (unsigned)(x0 + 1) < (unsigned)n;
                const bool gy0 = (unsigned)y0 < (unsigned)n, gy1 = (unsigned)(y0 + 1) < (unsigned)n;
                const bool gz0 = (unsigned)z0 < (unsigned)n, gz1 = (unsigned)(z0 + 1) < (unsigned)n;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int xs0 = x0 + sh[q][0], ys0 = y0 + sh[q][1], zs0 = z0 + sh[q][2];
                    const bool vx0 = gx0 && (unsigned)xs0 < (unsigned)n;
                    const bool vx1 = gx1 && (unsigned)(xs0 + 1) < (unsigned)n;
                    const bool vy0 = gy0 && (unsigned)ys0 < (unsigned)n;
                    const bool vy1 = gy1 && (unsigned)(ys0 + 1) < (unsigned)n;
                    const bool vz0 = gz0 && (unsigned)zs0 < (unsigned)n;
                    const bool vz1 = gz1 && (unsigned)(zs0 + 1) < (unsigned)n;
                    float val = 0.0f;
                    const bool inside = vx0 && vx1 && vy0 && vy1 && vz0 && vz1;
                    if (vp[q] && inside) {  // every tap inside both grids: no masks (same values and order)
                        const float2* b = vp[q] + ((zs0 * n + ys0) * (n + 1) + xs0 + 1);
                        const int rowp = n + 1, slab = n * (n + 1);
                        const float2 p0 = __ldg(b), p1 = __ldg(b + rowp), p2 = __ldg(b + slab), p3 = __ldg(b + slab + rowp);
                        val = fmaf((1.0f - fy) * (1.0f - fz), fmaf(fx, p0.y - p0.x, p0.x), val);
                        val = fmaf(fy * (1.0f - fz), fmaf(fx, p1.y - p1.x, p1.x), val);
                        val = fmaf((1.0f - fy) * fz, fmaf(fx, p2.y - p2.x, p2.x), val);
                        val = fmaf(fy * fz, fmaf(fx, p3.y - p3.x, p3.x), val);
                    } else if (vp[q]) {
                        const int o0 = (zs0 * n + ys0) * (n + 1) + xs0 + 1;  // within one volume: 32-bit
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const int bb = c & 1, aa = c >> 1;
                            const bool vr = (bb ? vy1 : vy0) && (aa ? vz1 : vz0);
                            const float2 pr = (vr && (vx0 || vx1))
                                                  ? __ldg(vp[q] + o0 + (bb ? n + 1 : 0) + (aa ? n * (n + 1) : 0))
                                                  : make_float2(0.0f, 0.0f);
                            const float v0 = vx0 ? pr.x : 0.0f;
                            const float v1 = vx1 ? pr.y : 0.0f;
                            const float wyz = (bb ? fy : 1.0f - fy) * (aa ? fz : 1.0f - fz);
                            val = fmaf(wyz, fmaf(fx, v1 - v0, v0), val);
                        }
                    } else {
                        const int o0 = (zs0 * n + ys0) * n + xs0;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const int bb = c & 1, aa = c >> 1;
                            const bool vr = (bb ? vy1 : vy0) && (aa ? vz1 : vz0);
                            const float* row = v[q] + o0 + (bb ? n : 0) + (aa ? n * n : 0);
                            const float v0 = (vr && vx0) ? __ldg(row) : 0.0f;
                            const float v1 = (vr && vx1) ? __ldg(row + 1) : 0.0f;
                            const float wyz = (bb ? fy : 1.0f - fy) * (aa ? fz : 1.0f - fz);
                            val = fmaf(wyz, fmaf(fx, v1 - v0, v0), val);
                        }
                    }
                    samp[(q * kRC + j) * nsamp + s] = val;
                }
            }
        }
        for (int i = tid; i < T.pairs; i += kThreads) rad[i] = T.radial_t[(size_t)ir * T.pairs + i];
        __syncthreads();
        {  // 2. phi-DFT: thread = (window, order group, ring)
            constexpr int MH = NPC / 2, MS = (MH + 1) / 2;
            const int q = tid >> 7, g = (tid >> 6) & 1, t = tid & 63;
            if (t < nt) {
                const float* f = samp + (q * kRC + rc) * nsamp + t * np;
                float2* Fr = F + (q * nt + t) * nl;
                if (g == 0) dft_ring<NPC, 0, MS>(f, Fr);
                else dft_ring<NPC, MS, MH>(f, Fr);
            }
        }
        __syncthreads();
        if (tid < T.ntri) {  // 3. theta, both windows with the same register weights
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const float2* Fq = F + q * nt * nl;
                float re = 0.0f, im = 0.0f;
#pragma unroll
                for (int t = 0; t < NPC / 2; ++t) {
                    const float2 a = Fq[t * nl + th_m], b = Fq[(NPC - 1 - t) * nl + th_m];
                    re = fmaf(th_w[t], fmaf(th_sgn, b.x, a.x), re);
                    im = fmaf(th_w[t], fmaf(th_sgn, b.y, a.y), im);
                }
                float* G = Gp + q * nl * nl;
                if (th_m == 0) {
                    G[th_base] = re;
                } else {
                    G[th_base + 2 * th_m - 1] = re;
                    G[th_base + 2 * th_m] = im;
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int qq = 0; qq < RPT; ++qq) {  // 4. radial
            const int row = tid + qq * kThreads;
            if (row < T.coeffs) {
                const int rp = rpr[qq];
                const float rv = rad[rp >> 16];
                acc[0][qq] = fmaf(rv, Gp[rp & 0xffff], acc[0][qq]);
                acc[1][qq] = fmaf(rv, Gp[nl * nl + (rp & 0xffff)], acc[1][qq]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int qq = 0; qq < RPT; ++qq) {
        const int row = tid + qq * kThreads;
        if (row < T.coeffs) {
            out[(long long)wa * ldo + row] = acc[0][qq];
            if (two) out[(long long)wb * ldo + row] = acc[1][qq];
        }
    }
}

template <int RPT, int NPC>
int launch_pair(const FactoredTables& T, const float* vols, long long vol_stride, const int* win_vol,
                const int* win_shift, int n_win, float* out, int ldo, cudaStream_t s, const float2* pairs) {
    const size_t smem = smem_plan_pair(T).total;
    if (smem > 220 * 1024) return 1;
    if (ensure_dynamic_smem(expand_pair_kernel<RPT, NPC>, (int)smem) != cudaSuccess) return 2;
    expand_pair_kernel<RPT, NPC><<<(n_win + 1) / 2, kThreads, smem, s>>>(T, vols, vol_stride, win_vol, win_shift,
                                                                           n_win, out, ldo, pairs);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}


// ---------------------------------------------------------------- phi-DFT on tcgen05
// K2t: the two-window kernel with stage 2 on the tensor cores.  Per pass of
// kTcRC radii the 2 * kTcRC * n_theta rings of the pair are the rows of one GEMM
//   D[ring][2m + c] = sum_kk A[ring][kk] * B[2m + c][kk],
// A = the ring's samples f[p] for p != 0, n_phi/2 (kk = p - 1 below n_phi/2,
// p - 2 above: K = n_phi - 2, a multiple of 8), B = cos / -sin(2 pi m p / n_phi).
// FP32 accuracy comes from the 3xTF32 split (hi = rna_tf32(x), lo = x - hi;
// hi.hi + hi.lo + lo.hi, FP32 accumulation in TMEM); the two samples every real
// part shares, f[0] and f[n_phi/2], stay in FP32 and are added when the rows are
// drained.  The gather threads write A straight into the K-major SWIZZLE_128B
// layout (no staging copy), one thread issues the MMAs (M = 128 row tiles,
// N = 16 ceil(2 (L+1) / 16), 3 x K/8 instructions per tile), and all warps drain
// TMEM into the F rows the theta stage reads.  Stages 3 and 4 are those of the
// pair kernel, batched over the radii of the pass.
#ifndef BMB_EXPAND_TC_MINB
#define BMB_EXPAND_TC_MINB 2
#endif
constexpr int kTcRC = 4;
struct SmemTc {
    size_t a_hi, a_lo, b_hi, b_lo, side, G, rad, bar, total;
    int rows, tiles, katoms, ncols;
};
__host__ __device__ inline SmemTc smem_plan_tc(const FactoredTables& T) {
    SmemTc s;
    const int nl = T.L + 1;
    s.rows = 2 * kTcRC * T.nt;
    s.tiles = (s.rows + 127) / 128;
    s.katoms = (T.np - 2 + 31) / 32;
    s.ncols = (2 * nl + 15) / 16 * 16;
    const size_t tile_bytes = (size_t)s.katoms * 128 * 128;
    // rows are laid out tile by tile; the last tile's unused rows read whatever
    // follows (their D rows are never drained), so A_lo's last tile must still lie
    // inside the allocation: the buffers behind it cover that
    const size_t a_bytes = (size_t)(s.tiles - 1) * tile_bytes + (size_t)(s.rows - 128 * (s.tiles - 1) + 7) / 8 * 1024 * s.katoms;
    size_t o = 0;
    s.a_hi = o;
    o += (a_bytes + 1023) / 1024 * 1024;
    s.a_lo = o;
    o += (a_bytes + 1023) / 1024 * 1024;
    const size_t f_bytes = sizeof(float2) * (size_t)s.rows * nl;  // F aliases A (dead once the MMAs retire)
    if (o < f_bytes) o = (f_bytes + 1023) / 1024 * 1024;
    s.b_hi = o;
    o += (size_t)s.katoms * s.ncols * 128;
    s.b_lo = o;
    o += (size_t)s.katoms * s.ncols * 128;
    s.side = o;
    o = al16(o + sizeof(float2) * (size_t)s.rows);
    s.G = o;
    o = al16(o + 2 * kTcRC * sizeof(float) * (size_t)nl * nl);
    s.rad = o;
    o = al16(o + 2 * kTcRC * sizeof(float) * (size_t)T.pairs);
    s.bar = o;
    o += 16;
    const size_t need = s.a_lo + (size_t)s.tiles * tile_bytes;  // A_lo's last full tile
    s.total = o > need ? o : need;
    return s;
}

template <int RPT, int NPC>
__global__ void __launch_bounds__(kThreads, BMB_EXPAND_TC_MINB)
    expand_tc_kernel(FactoredTables T, const float* __restrict__ vols, long long vol_stride,
                     const int* __restrict__ win_vol, const int* __restrict__ win_shift, int n_win,
                     float* __restrict__ out, int ldo, const float2* __restrict__ pairs) {
    static_assert(NPC > 0 && NPC <= 64 && (NPC - 2) % 8 == 0 && (NPC / 2) * (NPC / 2 + 1) / 2 <= kThreads,
                  "specialised shapes only");
    constexpr int RC = kTcRC, HALFP = NPC / 2, NL = NPC / 2, NL2 = NL * NL;
    constexpr int KA = (NPC - 2 + 31) / 32;          // 128-byte K atoms per row
    constexpr int KS = (NPC - 2) / 8;                // tcgen05.mma K steps
    constexpr int NCOL = (2 * NL + 15) / 16 * 16;    // GEMM N
    constexpr int TILE_BYTES = KA * 128 * 128;
    extern __shared__ unsigned char sm_raw[];
    // SWIZZLE_128B operand tiles need a 1024-byte aligned base
    unsigned char* sm = sm_raw + ((1024u - (ptx::smem_u32(sm_raw) & 1023u)) & 1023u);
    const SmemTc P = smem_plan_tc(T);
    const int n = T.n, nt = T.nt, nsamp = nt * NPC;
    unsigned char* a_hi = sm + P.a_hi;
    unsigned char* a_lo = sm + P.a_lo;
    float2* F = reinterpret_cast<float2*>(sm);                    // [2][RC][nt][NL], aliases A
    float2* side = reinterpret_cast<float2*>(sm + P.side);        // [row] (f[0], f[n_phi/2])
    float* Gp = reinterpret_cast<float*>(sm + P.G);               // [2][RC][NL2]
    float* rad = reinterpret_cast<float*>(sm + P.rad);            // [2 buffers][RC][pairs]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + P.bar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + P.bar + 8);
    const int tid = threadIdx.x;
    const uint32_t warp = tid >> 5, lane = tid & 31;
    const uint32_t tmem_cols = P.tiles * 64 <= 128 ? 128u : 256u;

    if (tid == 0) {
        ptx::mbar_init(bar, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) {
        ptx::tmem_alloc(tmem_slot, tmem_cols);
        ptx::tmem_relinquish();
    }
    // B: twiddle rows (2m: cos, 2m+1: -sin), hi / lo TF32 parts, K-major SWIZZLE_128B
    for (int i = tid; i < NCOL * KA * 32; i += kThreads) {
        const int row = i / (KA * 32), kk = i - row * (KA * 32);
        float val = 0.0f;
        const int m = row >> 1;
        if (m < NL && kk < NPC - 2) {
            const int p = kk < HALFP - 1 ? kk + 1 : kk + 2;
            const float2 t = p < HALFP ? T.tw[p * NL + m] : T.tw[(NPC - p) * NL + m];
            val = (row & 1) ? (p < HALFP ? t.y : -t.y) : t.x;
        }
        const float hi = ptx::to_tf32(val);
        const int atom = kk >> 5, k5 = kk & 31;
        const int off = atom * NCOL * 128 + (row >> 3) * 1024 + (row & 7) * 128 + (((k5 >> 2) ^ (row & 7)) << 4) + (k5 & 3) * 4;
        *reinterpret_cast<float*>(sm + P.b_hi + off) = hi;
        *reinterpret_cast<float*>(sm + P.b_lo + off) = ptx::to_tf32(val - hi);
    }
    const int wa = 2 * blockIdx.x;
    const bool two = wa + 1 < n_win;
    const int wb = two ? wa + 1 : wa;
    const float* __restrict__ v[2] = {vols + (long long)win_vol[wa] * vol_stride,
                                      vols + (long long)win_vol[wb] * vol_stride};
    const float2* __restrict__ vp[2] = {pairs ? pairs + win_vol[wa] * pair_volume_elems(n) : nullptr,
                                        pairs ? pairs + win_vol[wb] * pair_volume_elems(n) : nullptr};
    int sh[2][3];
#pragma unroll
    for (int q = 0; q < 3; ++q) sh[0][q] = win_shift[3 * wa + q], sh[1][q] = win_shift[3 * wb + q];
    float acc[2][RPT];
    int rpr[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        acc[0][q] = acc[1][q] = 0.0f;
        rpr[q] = tid + q * kThreads < T.coeffs ? T.rowpack[tid + q * kThreads] : 0;
    }
    float th_w[NPC / 2];
    int th_m = 0, th_base = 0;
    float th_sgn = 1.0f;
    if (tid < T.ntri) {
        const int2 lm = T.tri_lm[tid];
        th_m = lm.y;
        th_base = lm.x * lm.x;
        th_sgn = ((lm.x + lm.y) & 1) ? -1.0f : 1.0f;
#pragma unroll
        for (int t = 0; t < NPC / 2; ++t) th_w[t] = __ldg(T.ptab + (size_t)tid * NPC + t);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    uint32_t phase = 0;
    for (int ir = 0, pass = 0; ir < T.nr; ir += RC, ++pass) {
        const int nrc = min(RC, T.nr - ir);
        float* radb = rad + (pass & 1) * RC * T.pairs;
        {  // 1. trilinear samples -> A (hi, lo) and the two FP32 side samples of every ring
            const int items = nsamp * RC;
            auto entry = [&](int it) {
                const int s = it / RC, j = it - s * RC;
                return (it < items && j < nrc) ? __ldg(T.samp + (size_t)s * T.nr + ir + j) : make_int4(0, 0, 0, 0);
            };
            int4 e_next = entry(tid);
            for (int it = tid; it < items; it += kThreads) {
                const int s = it / RC, j = it - s * RC;
                const int4 e = e_next;
                e_next = entry(it + kThreads);
                if (j >= nrc) continue;
                const int t = s / NPC, p = s - t * NPC;
                const int x0 = e.x & 1023, y0 = (e.x >> 10) & 1023, z0 = (e.x >> 20) & 1023;
                const float fx = __int_as_float(e.y), fy = __int_as_float(e.z), fz = __int_as_float(e.w);
                const bool gx0 = (unsigned)x0 < (unsigned)n, gx1 = (unsigned)(x0 + 1) < (unsigned)n;
                const bool gy0 = (unsigned)y0 < (unsigned)n, gy1 = (unsigned)(y0 + 1) < (unsigned)n;
                const bool gz0 = (unsigned)z0 < (unsigned)n, gz1 = (unsigned)(z0 + 1) < (unsigned)n;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int xs0 = x0 + sh[q][0], ys0 = y0 + sh[q][1], zs0 = z0 + sh[q][2];
                    const bool vx0 = gx0 && (unsigned)xs0 < (unsigned)n;
                    const bool vx1 = gx1 && (unsigned)(xs0 + 1) < (unsigned)n;
                    const bool vy0 = gy0 && (unsigned)ys0 < (unsigned)n;
                    const bool vy1 = gy1 && (unsigned)(ys0 + 1) < (unsigned)n;
                    const bool vz0 = gz0 && (unsigned)zs0 < (unsigned)n;
                    const bool vz1 = gz1 && (unsigned)(zs0 + 1) < (unsigned)n;
                    float val = 0.0f;
                    const bool inside = vx0 && vx1 && vy0 && vy1 && vz0 && vz1;
                    if (vp[q] && inside) {
                        const float2* b = vp[q] + ((zs0 * n + ys0) * (n + 1) + xs0 + 1);
                        const int rowp = n + 1, slab = n * (n + 1);
                        const float2 p0 = __ldg(b), p1 = __ldg(b + rowp), p2 = __ldg(b + slab), p3 = __ldg(b + slab + rowp);
                        val = fmaf((1.0f - fy) * (1.0f - fz), fmaf(fx, p0.y - p0.x, p0.x), val);
                        val = fmaf(fy * (1.0f - fz), fmaf(fx, p1.y - p1.x, p1.x), val);
                        val = fmaf((1.0f - fy) * fz, fmaf(fx, p2.y - p2.x, p2.x), val);
                        val = fmaf(fy * fz, fmaf(fx, p3.y - p3.x, p3.x), val);
                    } else if (vp[q]) {
                        const int o0 = (zs0 * n + ys0) * (n + 1) + xs0 + 1;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const int bb = c & 1, aa = c >> 1;
                            const bool vr = (bb ? vy1 : vy0) && (aa ? vz1 : vz0);
                            const float2 pr = (vr && (vx0 || vx1))
                                                  ? __ldg(vp[q] + o0 + (bb ? n + 1 : 0) + (aa ? n * (n + 1) : 0))
                                                  : make_float2(0.0f, 0.0f);
                            const float v0 = vx0 ? pr.x : 0.0f;
                            const float v1 = vx1 ? pr.y : 0.0f;
                            const float wyz = (bb ? fy : 1.0f - fy) * (aa ? fz : 1.0f - fz);
                            val = fmaf(wyz, fmaf(fx, v1 - v0, v0), val);
                        }
                    } else {
                        const int o0 = (zs0 * n + ys0) * n + xs0;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const int bb = c & 1, aa = c >> 1;
                            const bool vr = (bb ? vy1 : vy0) && (aa ? vz1 : vz0);
                            const float* row = v[q] + o0 + (bb ? n : 0) + (aa ? n * n : 0);
                            const float v0 = (vr && vx0) ? __ldg(row) : 0.0f;
                            const float v1 = (vr && vx1) ? __ldg(row + 1) : 0.0f;
                            const float wyz = (bb ? fy : 1.0f - fy) * (aa ? fz : 1.0f - fz);
                            val = fmaf(wyz, fmaf(fx, v1 - v0, v0), val);
                        }
                    }
                    const int r = (q * RC + j) * nt + t;
                    if (p == 0) {
                        side[r].x = val;
                    } else if (p == HALFP) {
                        side[r].y = val;
                    } else {
                        const int kk = p < HALFP ? p - 1 : p - 2;
                        const int atom = kk >> 5, k5 = kk & 31, rr = r & 127;
                        const int off = (r >> 7) * TILE_BYTES + atom * (128 * 128) + (rr >> 3) * 1024 + (rr & 7) * 128 +
                                        (((k5 >> 2) ^ (rr & 7)) << 4) + (k5 & 3) * 4;
                        const float hi = ptx::to_tf32(val);
                        *reinterpret_cast<float*>(a_hi + off) = hi;
                        *reinterpret_cast<float*>(a_lo + off) = ptx::to_tf32(val - hi);
                    }
                }
            }
        }
        for (int i = tid; i < nrc * T.pairs; i += kThreads) radb[i] = T.radial_t[(size_t)ir * T.pairs + i];
        ptx::fence_proxy_async_smem();
        __syncthreads();
        // 2. phi-DFT of every ring of the pass: 3xTF32 on the tensor cores
        if (warp == 0) {
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
                constexpr uint32_t idesc = ptx::make_idesc(2, 128, NCOL);
                for (int tile = 0; tile < P.tiles; ++tile) {
                    const uint32_t d = tmem_base + tile * 64;
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) {
                        const int atom = ks >> 2;
                        const uint64_t koff = (uint64_t)((ks & 3) * 32) >> 4;
                        const uint64_t ah = ptx::smem_desc_k_sw128(a_hi + tile * TILE_BYTES + atom * (128 * 128)) + koff;
                        const uint64_t al = ptx::smem_desc_k_sw128(a_lo + tile * TILE_BYTES + atom * (128 * 128)) + koff;
                        const uint64_t bh = ptx::smem_desc_k_sw128(sm + P.b_hi + atom * NCOL * 128) + koff;
                        const uint64_t bl = ptx::smem_desc_k_sw128(sm + P.b_lo + atom * NCOL * 128) + koff;
                        ptx::mma_tf32(d, al, bh, idesc, ks > 0 ? 1u : 0u);
                        ptx::mma_tf32(d, ah, bl, idesc, 1u);
                        ptx::mma_tf32(d, ah, bh, idesc, 1u);
                    }
                }
                ptx::tc_commit(bar);
            }
            __syncwarp();
        }
        ptx::mbar_wait(bar, phase);
        phase ^= 1;
        ptx::tc_fence_after();
        // drain: warp w owns the TMEM lanes 32 (w % 4) ..; tiles alternate between the two warp groups
        for (int tile = warp >> 2; tile < P.tiles; tile += 2) {
            const int r = tile * 128 + (warp & 3) * 32 + lane;
            if (tile * 128 + (int)(warp & 3) * 32 >= P.rows) continue;  // warp-uniform
            const float2 sd = r < P.rows ? side[r] : make_float2(0.0f, 0.0f);
            const float ev = sd.x + sd.y, od = sd.x - sd.y;
#pragma unroll
            for (int c = 0; c < NCOL / 16; ++c) {
                uint32_t d[16];
                ptx::tmem_ld_32x32b_x16(tmem_base + (((warp & 3) * 32u) << 16) + tile * 64 + c * 16, d);
                ptx::tmem_ld_wait();
                if (r < P.rows) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int m = c * 8 + i;
                        if (m < NL)
                            F[r * NL + m] = make_float2(__uint_as_float(d[2 * i]) + ((m & 1) ? od : ev), __uint_as_float(d[2 * i + 1]));
                    }
                }
            }
        }
        ptx::tc_fence_before();
        __syncthreads();
        if (tid < T.ntri) {  // 3. theta, every (window, radius) of the pass with the same register weights
            for (int qj = 0; qj < 2 * RC; ++qj) {
                if (qj % RC >= nrc) continue;
                const float2* Fq = F + qj * nt * NL;
                float re = 0.0f, im = 0.0f;
#pragma unroll
                for (int t = 0; t < NPC / 2; ++t) {
                    const float2 a = Fq[t * NL + th_m], b = Fq[(NPC - 1 - t) * NL + th_m];
                    re = fmaf(th_w[t], fmaf(th_sgn, b.x, a.x), re);
                    im = fmaf(th_w[t], fmaf(th_sgn, b.y, a.y), im);
                }
                float* G = Gp + qj * NL2;
                if (th_m == 0) {
                    G[th_base] = re;
                } else {
                    G[th_base + 2 * th_m - 1] = re;
                    G[th_base + 2 * th_m] = im;
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int qq = 0; qq < RPT; ++qq) {  // 4. radial, radius ascending (the order of the other kernels)
            const int row = tid + qq * kThreads;
            if (row < T.coeffs) {
                const int rp = rpr[qq];
                for (int j = 0; j < nrc; ++j) {
                    const float rv = radb[j * T.pairs + (rp >> 16)];
                    acc[0][qq] = fmaf(rv, Gp[j * NL2 + (rp & 0xffff)], acc[0][qq]);
                    acc[1][qq] = fmaf(rv, Gp[(RC + j) * NL2 + (rp & 0xffff)], acc[1][qq]);
                }
            }
        }
        // the next pass writes A / F, the side samples and the other rad buffer; G is
        // rewritten only after the next two barriers
    }
#pragma unroll
    for (int qq = 0; qq < RPT; ++qq) {
        const int row = tid + qq * kThreads;
        if (row < T.coeffs) {
            out[(long long)wa * ldo + row] = acc[0][qq];
            if (two) out[(long long)wb * ldo + row] = acc[1][qq];
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, tmem_cols);
    }
}

template <int RPT, int NPC>
int launch_tc(const FactoredTables& T, const float* vols, long long vol_stride, const int* win_vol,
              const int* win_shift, int n_win, float* out, int ldo, cudaStream_t s, const float2* pairs) {
    const size_t smem = smem_plan_tc(T).total + 1024;  // + alignment slack
    if (smem > 113 * 1024) return 1;
    if (ensure_dynamic_smem(expand_tc_kernel<RPT, NPC>, (int)smem) != cudaSuccess) return 2;
    expand_tc_kernel<RPT, NPC><<<(n_win + 1) / 2, kThreads, smem, s>>>(T, vols, vol_stride, win_vol, win_shift, n_win,
                                                                         out, ldo, pairs);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}


// ---------------------------------------------------------------- quad gathers
// K2q: the two-window kernel gathering from a zero-padded quad copy of each
// volume, quads[z + M][y + M][x + M] = (v[x], v[x+1], v[x+2], v[x+3]) (zero
// outside the grid, M = kQuadPad).  The padding removes every bound check on the
// shifted source for |shift| <= M; a footprint that leaves the window grid
// itself (bit 30 of the table entry, the outermost samples) keeps the masked
// taps.  CTAs follow a pair list: windows of one volume whose shifts differ by
// 1 or 2 in x only share ONE 16-byte load per footprint row (mode = the x
// difference); other pairs (mode 0) load 8 bytes per row and window.  Per
// window the FP32 values and FMA order are those of the other kernels
// (bit-identical coefficients).
template <int NG>
struct QuadGeom {
    int np_, rw_;
    __device__ __forceinline__ QuadGeom(int n) : np_(n + 2 * kQuadPad), rw_(n + 2 * kQuadPad) {}
    __device__ __forceinline__ int row() const { return NG > 0 ? NG + 2 * kQuadPad : rw_; }
    __device__ __forceinline__ int slab() const { return NG > 0 ? (NG + 2 * kQuadPad) * (NG + 2 * kQuadPad) : np_ * rw_; }
};

template <int RPT, int NPC, int NG>
__global__ void __launch_bounds__(kThreads, BMB_EXPAND_PAIR_MINB)
    expand_quad_kernel(FactoredTables T, const float4* __restrict__ quads, const int* __restrict__ win_vol,
                       const int* __restrict__ win_shift, const int4* __restrict__ pair_list,
                       float* __restrict__ out, int ldo) {
    static_assert(NPC > 0 && NPC <= 64 && (NPC / 2) * (NPC / 2 + 1) / 2 <= kThreads, "specialised shapes only");
    extern __shared__ __align__(16) unsigned char sm[];
    const SmemPair P = smem_plan_pair(T);
    const int n = T.n, nt = T.nt, np = NPC, nl = T.L + 1, nsamp = nt * np;
    float* samp = reinterpret_cast<float*>(sm + P.samp);          // [2][kRC][nsamp]
    float2* F = reinterpret_cast<float2*>(sm + P.F);              // [2][nt][nl]
    float* Gp = reinterpret_cast<float*>(sm + P.G);               // [2][nl^2]
    float* rad = reinterpret_cast<float*>(sm + P.rad);
    const int tid = threadIdx.x;
    const int4 pl = pair_list[blockIdx.x];
    const int wa = pl.x, wb = pl.y, mode = pl.z;
    const bool two = wb != wa;
    const QuadGeom<NG> geo(n);
    const int ROW = geo.row(), SLAB = geo.slab();
    const float4* __restrict__ vq[2] = {quads + win_vol[wa] * quad_volume_elems(n),
                                        quads + win_vol[wb] * quad_volume_elems(n)};
    int cb[2];  // offset of the shifted origin inside the padded copy
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int w = q ? wb : wa;
        cb[q] = ((win_shift[3 * w + 2] + kQuadPad) * ROW + win_shift[3 * w + 1] + kQuadPad) * ROW + win_shift[3 * w] + kQuadPad;
    }
    // the row map of the radial stage: in registers while the accumulators leave room
    constexpr bool RP_REG = RPT <= 12;
    float acc[2][RPT];
    int rpr[RP_REG ? RPT : 1];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        acc[0][q] = acc[1][q] = 0.0f;
        if constexpr (RP_REG) rpr[q] = tid + q * kThreads < T.coeffs ? T.rowpack[tid + q * kThreads] : 0;
    }
    float th_w[NPC / 2];
    int th_m = 0, th_base = 0;
    float th_sgn = 1.0f;
    if (tid < T.ntri) {
        const int2 lm = T.tri_lm[tid];
        th_m = lm.y;
        th_base = lm.x * lm.x;
        th_sgn = ((lm.x + lm.y) & 1) ? -1.0f : 1.0f;
#pragma unroll
        for (int t = 0; t < NPC / 2; ++t) th_w[t] = __ldg(T.ptab + (size_t)tid * NPC + t);
    }
    __syncthreads();
    // one pass of trilinear samples; MODE: 0 independent windows, 1 / 2 the x distance of the pair
    auto gather = [&](auto mode_tag, int ir) {
        constexpr int MODE = decltype(mode_tag)::value;
        const int nrc = min(kRC, T.nr - ir);
        const int items = nsamp * kRC;
        auto entry = [&](int it) {
            const int s = it / kRC, j = it - s * kRC;
            return (it < items && j < nrc) ? __ldg(T.samp + (size_t)s * T.nr + ir + j) : make_int4(0, 0, 0, 0);
        };
        int4 e_next = entry(tid);
        for (int it = tid; it < items; it += kThreads) {
            const int s = it / kRC, j = it - s * kRC;
            const int4 e = e_next;
            e_next = entry(it + kThreads);
            if (j >= nrc) continue;
            const int x0 = e.x & 1023, y0 = (e.x >> 10) & 1023, z0 = (e.x >> 20) & 1023;
            const float fx = __int_as_float(e.y), fy = __int_as_float(e.z), fz = __int_as_float(e.w);
            const int o0 = (z0 * ROW + y0) * ROW + x0;
            const float w0 = (1.0f - fy) * (1.0f - fz), w1 = fy * (1.0f - fz), w2 = (1.0f - fy) * fz, w3 = fy * fz;
            float va = 0.0f, vb = 0.0f;
            if (!(e.x >> 30)) {  // the footprint lies inside the window grid: the padding does the rest
                if constexpr (MODE == 0) {
                    const float2* a = reinterpret_cast<const float2*>(vq[0] + o0 + cb[0]);
                    const float2* b = reinterpret_cast<const float2*>(vq[1] + o0 + cb[1]);
                    const float2 a0 = __ldg(a), a1 = __ldg(a + 2 * ROW), a2 = __ldg(a + 2 * SLAB), a3 = __ldg(a + 2 * (SLAB + ROW));
                    const float2 b0 = __ldg(b), b1 = __ldg(b + 2 * ROW), b2 = __ldg(b + 2 * SLAB), b3 = __ldg(b + 2 * (SLAB + ROW));
                    va = fmaf(w0, fmaf(fx, a0.y - a0.x, a0.x), va);
                    va = fmaf(w1, fmaf(fx, a1.y - a1.x, a1.x), va);
                    va = fmaf(w2, fmaf(fx, a2.y - a2.x, a2.x), va);
                    va = fmaf(w3, fmaf(fx, a3.y - a3.x, a3.x), va);
                    vb = fmaf(w0, fmaf(fx, b0.y - b0.x, b0.x), vb);
                    vb = fmaf(w1, fmaf(fx, b1.y - b1.x, b1.x), vb);
                    vb = fmaf(w2, fmaf(fx, b2.y - b2.x, b2.x), vb);
                    vb = fmaf(w3, fmaf(fx, b3.y - b3.x, b3.x), vb);
                } else {
                    const float4* a = vq[0] + o0 + cb[0];
                    const float4 q0 = __ldg(a), q1 = __ldg(a + ROW), q2 = __ldg(a + SLAB), q3 = __ldg(a + SLAB + ROW);
                    va = fmaf(w0, fmaf(fx, q0.y - q0.x, q0.x), va);
                    va = fmaf(w1, fmaf(fx, q1.y - q1.x, q1.x), va);
                    va = fmaf(w2, fmaf(fx, q2.y - q2.x, q2.x), va);
                    va = fmaf(w3, fmaf(fx, q3.y - q3.x, q3.x), va);
                    if constexpr (MODE == 1) {
                        vb = fmaf(w0, fmaf(fx, q0.z - q0.y, q0.y), vb);
                        vb = fmaf(w1, fmaf(fx, q1.z - q1.y, q1.y), vb);
                        vb = fmaf(w2, fmaf(fx, q2.z - q2.y, q2.y), vb);
                        vb = fmaf(w3, fmaf(fx, q3.z - q3.y, q3.y), vb);
                    } else {
                        vb = fmaf(w0, fmaf(fx, q0.w - q0.z, q0.z), vb);
                        vb = fmaf(w1, fmaf(fx, q1.w - q1.z, q1.z), vb);
                        vb = fmaf(w2, fmaf(fx, q2.w - q2.z, q2.z), vb);
                        vb = fmaf(w3, fmaf(fx, q3.w - q3.z, q3.z), vb);
                    }
                }
            } else {  // taps that leave the window grid are zero whatever the source holds there
                const bool gx1 = x0 + 1 < n, gy1 = y0 + 1 < n, gz1 = z0 + 1 < n;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const float2* b = reinterpret_cast<const float2*>(vq[q] + o0 + cb[q]);
                    float val = 0.0f;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int bb = c & 1, aa = c >> 1;
                        const bool vr = (bb ? gy1 : true) && (aa ? gz1 : true);
                        const float2 pr = vr ? __ldg(b + 2 * ((bb ? ROW : 0) + (aa ? SLAB : 0))) : make_float2(0.0f, 0.0f);
                        const float v1 = gx1 ? pr.y : 0.0f;
                        const float wyz = (bb ? fy : 1.0f - fy) * (aa ? fz : 1.0f - fz);
                        val = fmaf(wyz, fmaf(fx, v1 - pr.x, pr.x), val);
                    }
                    if (q == 0) va = val;
                    else vb = val;
                }
            }
            samp[j * nsamp + s] = va;
            samp[(kRC + j) * nsamp + s] = vb;
        }
    };
    for (int ir = 0; ir < T.nr; ++ir) {
        const int rc = ir % kRC;
        if (rc == 0) {
            if (mode == 1) gather(std::integral_constant<int, 1>{}, ir);
            else if (mode == 2) gather(std::integral_constant<int, 2>{}, ir);
            else gather(std::integral_constant<int, 0>{}, ir);
        }
        for (int i = tid; i < T.pairs; i += kThreads) rad[i] = T.radial_t[(size_t)ir * T.pairs + i];
        __syncthreads();
        {  // 2. phi-DFT: thread = (window, order group, ring)
            constexpr int MH = NPC / 2, MS = (MH + 1) / 2;
            const int q = tid >> 7, g = (tid >> 6) & 1, t = tid & 63;
            if (t < nt) {
                const float* f = samp + (q * kRC + rc) * nsamp + t * np;
                float2* Fr = F + (q * nt + t) * nl;
                if (g == 0) dft_ring<NPC, 0, MS>(f, Fr);
                else dft_ring<NPC, MS, MH>(f, Fr);
            }
        }
        __syncthreads();
        if (tid < T.ntri) {  // 3. theta, both windows with the same register weights
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const float2* Fq = F + q * nt * nl;
                float re = 0.0f, im = 0.0f;
#pragma unroll
                for (int t = 0; t < NPC / 2; ++t) {
                    const float2 a = Fq[t * nl + th_m], b = Fq[(NPC - 1 - t) * nl + th_m];
                    re = fmaf(th_w[t], fmaf(th_sgn, b.x, a.x), re);
                    im = fmaf(th_w[t], fmaf(th_sgn, b.y, a.y), im);
                }
                float* G = Gp + q * nl * nl;
                if (th_m == 0) {
                    G[th_base] = re;
                } else {
                    G[th_base + 2 * th_m - 1] = re;
                    G[th_base + 2 * th_m] = im;
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int qq = 0; qq < RPT; ++qq) {  // 4. radial
            const int row = tid + qq * kThreads;
            if (row < T.coeffs) {
                int rp;
                if constexpr (RP_REG) rp = rpr[qq];
                else rp = __ldg(T.rowpack + row);
                const float rv = rad[rp >> 16];
                acc[0][qq] = fmaf(rv, Gp[rp & 0xffff], acc[0][qq]);
                acc[1][qq] = fmaf(rv, Gp[nl * nl + (rp & 0xffff)], acc[1][qq]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int qq = 0; qq < RPT; ++qq) {
        const int row = tid + qq * kThreads;
        if (row < T.coeffs) {
            out[(long long)wa * ldo + row] = acc[0][qq];
            if (two) out[(long long)wb * ldo + row] = acc[1][qq];
        }
    }
}

template <int RPT, int NPC>
int launch_quad(const FactoredTables& T, const float4* quads, const int* win_vol, const int* win_shift,
                const int4* pair_list, int n_pairs, float* out, int ldo, cudaStream_t s) {
    const size_t smem = smem_plan_pair(T).total;
    if (smem > 220 * 1024) return 1;
    if (T.n == 64) {
        if (ensure_dynamic_smem(expand_quad_kernel<RPT, NPC, 64>, (int)smem) != cudaSuccess) return 2;
        expand_quad_kernel<RPT, NPC, 64><<<n_pairs, kThreads, smem, s>>>(T, quads, win_vol, win_shift, pair_list, out, ldo);
    } else {
        if (ensure_dynamic_smem(expand_quad_kernel<RPT, NPC, 0>, (int)smem) != cudaSuccess) return 2;
        expand_quad_kernel<RPT, NPC, 0><<<n_pairs, kThreads, smem, s>>>(T, quads, win_vol, win_shift, pair_list, out, ldo);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

template <int HALF, int RPT, int NPC = 0>
int launch_t(const FactoredTables& T, size_t smem, const float* vols, long long vol_stride, const int* win_vol,
             const int* win_shift, int n_win, float* out, int ldo, cudaStream_t s, const float2* pairs) {
    if (ensure_dynamic_smem(expand_factored_kernel<HALF, RPT, NPC>, (int)smem) != cudaSuccess) return 2;
    expand_factored_kernel<HALF, RPT, NPC><<<n_win, kThreads, smem, s>>>(T, vols, vol_stride, win_vol, win_shift, out,
                                                                         ldo, pairs);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace

size_t factored_smem_bytes(const FactoredTables& T) { return smem_plan(T).total; }

namespace {
// one thread per output pair; rows of n + 1 pairs (x = -1 .. n-1)
__global__ void pair_volumes_kernel(const float* __restrict__ vols, long long vol_stride, int n, long long total,
                                    float2* __restrict__ pairs) {
    const long long per = pair_volume_elems(n);
    const int w = n + 1;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long vol = i / per, r = i - vol * per;
        const long long row = r / w;
        const int x = (int)(r - row * w) - 1;
        const float* src = vols + vol * vol_stride + row * n;
        pairs[i] = make_float2(x >= 0 ? __ldg(src + x) : 0.0f, x + 1 < n ? __ldg(src + x + 1) : 0.0f);
    }
}
}  // namespace

namespace {
// one thread per quad of the padded copy (rows of n + 2M quads, x = i - M)
__global__ void quad_volumes_kernel(const float* __restrict__ vols, long long vol_stride, int n, long long total,
                                    float4* __restrict__ quads) {
    const int e = n + 2 * kQuadPad;
    const long long per = quad_volume_elems(n);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long vol = i / per;
        const int r = (int)(i - vol * per);
        const int x = r % e - kQuadPad, y = (r / e) % e - kQuadPad, z = r / (e * e) - kQuadPad;
        float4 q = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if ((unsigned)y < (unsigned)n && (unsigned)z < (unsigned)n) {
            const float* src = vols + vol * vol_stride + ((long long)z * n + y) * n;
            if ((unsigned)x < (unsigned)n) q.x = __ldg(src + x);
            if ((unsigned)(x + 1) < (unsigned)n) q.y = __ldg(src + x + 1);
            if ((unsigned)(x + 2) < (unsigned)n) q.z = __ldg(src + x + 2);
            if ((unsigned)(x + 3) < (unsigned)n) q.w = __ldg(src + x + 3);
        }
        quads[i] = q;
    }
}
}  // namespace

void launch_quad_volumes(const float* vols, long long vol_stride, int n_vol, int n, float4* quads, cudaStream_t s) {
    const long long total = quad_volume_elems(n) * n_vol;
    if (total <= 0) return;
    const long long blocks = std::min<long long>((total + 255) / 256, 148LL * 32);
    quad_volumes_kernel<<<(int)blocks, 256, 0, s>>>(vols, vol_stride, n, total, quads);
}

bool expand_quads_supported(const FactoredTables& T) {
    const int rpt = (T.coeffs + kThreads - 1) / kThreads;
    if (!(T.L + 1 == T.np / 2 && T.nt == T.np && T.ntri <= kThreads)) return false;
    return (T.np == 18 && rpt <= 4) || (T.np == 34 && rpt <= 12) || (T.np == 42 && rpt <= 24);
}

int launch_expand_quads(const FactoredTables& T, const float4* quads, const int* win_vol, const int* win_shift,
                        const int4* pair_list, int n_pairs, float* out, int ldo, cudaStream_t s) {
    if (n_pairs <= 0) return 0;
    if (!expand_quads_supported(T)) return 1;
    if (T.np == 18) return launch_quad<4, 18>(T, quads, win_vol, win_shift, pair_list, n_pairs, out, ldo, s);
    if (T.np == 34) return launch_quad<12, 34>(T, quads, win_vol, win_shift, pair_list, n_pairs, out, ldo, s);
    return launch_quad<24, 42>(T, quads, win_vol, win_shift, pair_list, n_pairs, out, ldo, s);
}

void launch_pair_volumes(const float* vols, long long vol_stride, int n_vol, int n, float2* pairs, cudaStream_t s) {
    const long long total = pair_volume_elems(n) * n_vol;
    if (total <= 0) return;
    const long long blocks = std::min<long long>((total + 255) / 256, 148LL * 16);
    pair_volumes_kernel<<<(int)blocks, 256, 0, s>>>(vols, vol_stride, n, total, pairs);
}

int launch_expand_factored(const FactoredTables& T, const float* vols, long long vol_stride, const int* win_vol,
                           const int* win_shift, int n_win, float* out, int ldo, cudaStream_t s,
                           const float2* pairs, bool same_volume_pairs) {
    if (n_win <= 0) return 0;
    const size_t smem = factored_smem_bytes(T);
    const char* force = std::getenv("BMB_EXPAND_SPLIT");  // tests: the large-basis path at any size
    if (smem > 220 * 1024 || T.L + 1 > kThreads || (force && std::atoi(force) != 0))
        return launch_split(T, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
    const int half = T.np / 2, rpt = (T.coeffs + kThreads - 1) / kThreads;
    if (T.L + 1 > kThreads) return 1;
    static const bool cdft = [] {
        const char* e = std::getenv("BMB_EXPAND_CDFT");
        return !(e && std::atoi(e) == 0);
    }();
    // BMB_EXPAND_PAIRWIN: 0 off, 1 (default) when consecutive windows share volumes,
    // 2 always (tests: bit-identity of the two kernels); read per launch
    const char* pw = std::getenv("BMB_EXPAND_PAIRWIN");
    const int pair_mode = pw ? std::atoi(pw) : 1;
    const bool pair_windows = pair_mode == 2 || (pair_mode == 1 && same_volume_pairs);
    // BMB_EXPAND_TC=1 runs the phi-DFT of the two-window kernel on the tensor cores
    // (3xTF32); default off: measured slower than the FP32 pipe (K2t); read per launch
    const char* tc = std::getenv("BMB_EXPAND_TC");
    const bool use_tc = tc && std::atoi(tc) != 0;
    if (use_tc && cdft && pair_windows && n_win >= 2 && T.L + 1 == T.np / 2 && T.nt == T.np && T.ntri <= kThreads) {
        if (T.np == 18 && rpt <= 4) return launch_tc<4, 18>(T, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
        if (T.np == 34 && rpt <= 12) return launch_tc<12, 34>(T, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
    }
    if (cdft && pair_windows && n_win >= 2 && T.L + 1 == T.np / 2 && T.ntri <= kThreads) {
        if (T.np == 18 && rpt <= 4) return launch_pair<4, 18>(T, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
        if (T.np == 34 && rpt <= 12) return launch_pair<12, 34>(T, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
    }
    if (cdft && T.L + 1 == T.np / 2) {  // n_phi = 2L + 2 with compile-time twiddles
        if (T.np == 18 && rpt <= 4) return launch_t<9, 4, 18>(T, smem, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
        if (T.np == 34 && rpt <= 12) return launch_t<17, 12, 34>(T, smem, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
        if (T.np == 42 && rpt <= 24) return launch_t<21, 24, 42>(T, smem, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
        if (T.np == 50 && rpt <= 40) return launch_t<25, 40, 50>(T, smem, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
    }
    if (half <= 9 && rpt <= 4) return launch_t<9, 4>(T, smem, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
    if (half <= 17 && rpt <= 12) return launch_t<17, 12>(T, smem, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
    if (half <= 21 && rpt <= 24) return launch_t<21, 24>(T, smem, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
    if (half <= 25 && rpt <= 40) return launch_t<25, 40>(T, smem, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
    if (half <= 33 && rpt <= 72) return launch_t<33, 72>(T, smem, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
    return launch_split(T, vols, vol_stride, win_vol, win_shift, n_win, out, ldo, s, pairs);
}

}  // namespace bmb
