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
#include <vector>

#include "smem_attr.hpp"
#include "expand_factored.hpp"

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
