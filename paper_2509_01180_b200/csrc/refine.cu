// Rotate-score-gradient evaluation and the bulk-synchronous damped Newton
// refinement (kernels K4, K5, K7).
//
// K4+K5 (warp_eval): C(g) = Re sum_l sum_{m,m'} xi_l[m,m'] e^{-i m a}
// d^l_{m,m'}(b) e^{-i m' g} with its Euler gradient and Hessian
// (correlation_derivatives, src/xcorr.cpp:52-105).  One warp per evaluation;
// each lane owns half-plane (m,m') chains and marches the three-term Wigner-d
// recursion over l in registers (src/steer.cpp:101-141), so every d value is
// produced once, used for the correlation AND the wedge-power kernel (same
// angles and band, Objective::eval, src/optimize.cpp:106-130) and never stored.
// The (-m,-m') half follows from the real-volume symmetry
// xi_{-m,-m'} D_{-m,-m'} = conj(xi_{m,m'} D_{m,m'}).  FP32 recursion and lane
// accumulation, FP64 phases / cross-lane reduction.
//
// K7 (refine()): the damped-Newton iteration of src/optimize.cpp:255-357
// (Levenberg lambda, <= 3 retries x10, one-radian trust cap, FullPivLU
// semantics, re-anchoring within 0.05 of the gimbal poles through the composed
// kernel xi~ = xi D(a)^T, xcorr.cpp:149-155) run bulk-synchronously over every
// candidate of every window: per iteration, small kernels for the chart /
// re-anchor decision (thread per candidate), the chart-kernel composition
// (warp per re-anchored candidate), the order-2 evaluation (warp per candidate,
// CTA per window), the FP64 Newton step (thread per candidate: objective
// quotient, 3x3 full-pivot LU, trial rotation) and up to three order-0 trial
// evaluations with their acceptance tests.  The host raises L between bands
// (frequency marching) and relaunches the iteration until no candidate is
// active.
#include <cfloat>
#include <cstdlib>

#include <cstddef>

#include "smem_attr.hpp"
#include "refine.cuh"
#include "rotation.cuh"

namespace bmb {

namespace {

constexpr double kPiD = 3.14159265358979323846;

// STEP: shared-memory bank offset (4-byte words mod 32) between consecutive
// scratch sets.  The slices of a warp look up the same item positions in their
// own sets, so sets STEP banks apart keep those lookups conflict-free
// (16 for two 16-lane slices, 8 for four 8-lane slices).
#ifndef BMB_WS_BANK_PAD
#define BMB_WS_BANK_PAD 1
#endif
template <int ML, int STEP>
struct WarpScratchT {
    float2 ua[ML + 1];
    float2 ug[ML + 1];
    float cp[2 * ML + 3];
    float sp[2 * ML + 3];
    double res[20];     // reduced (value, grad[3], hess aa ab ag bb bg gg) x (corr, wedge)
    double red[32];     // reduce-scatter staging (first scratch set of a warp)
    double cs_half[8];  // cos, sin of beta/2, beta, alpha, gamma
    static constexpr int kWords = 4 * (ML + 1) + 2 * (2 * ML + 3) + 2 * (20 + 32 + 8);
    static constexpr int kPad = BMB_WS_BANK_PAD ? ((STEP - kWords % 32 + 31) % 32) + 1 : 2;
    float pad[kPad];
};
using WarpScratch = WarpScratchT<kMaxL, 16>;

// single out-of-line copies of the FP64 math-library routines
__device__ __noinline__ void sincos_d(double x, double* s, double* c) { sincos(x, s, c); }

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__host__ __device__ __forceinline__ int xi_off(int l) { return l * (2 * l - 1) * (2 * l + 1) / 3; }

// One evaluation job: correlation kernel, wedge-power kernel (null: no wedge)
// and the ZYZ angles.
struct EvalJob {
    const float4* xi;
    const float4* wx;
    double a, b, g;
};

__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
// warp-cooperative L1 prefetch of the contiguous rows [r0, r1) of a band-layout
// kernel (512 B per row): one 128-byte line per lane and pass
__device__ __forceinline__ void prefetch_rows(const float4* k, int r0, int r1, int lane) {
    const char* base = reinterpret_cast<const char*>(k + (size_t)r0 * 32);
    const int bytes = (r1 - r0) * 512;
    for (int off = lane * 128; off < bytes; off += 32 * 128) prefetch_l1(base + off);
}

// products with explicit rounding so that every evaluation runs the identical
// FP32 sequence whichever slot k of a K-way warp it occupies
__device__ __forceinline__ float2 cmul_x(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -__fmul_rn(a.y, b.y)), fmaf(a.x, b.y, __fmul_rn(a.y, b.x)));
}

// order-dependent accumulators of one (kernel, entry) of a chain
template <int ORDER>
struct Chain3 {
    float2 v0, v1, v2;
    __device__ __forceinline__ void init(float2 x, float d, float dp, float dpp) {
        v0 = make_float2(__fmul_rn(x.x, d), __fmul_rn(x.y, d));
        v1 = make_float2(__fmul_rn(x.x, dp), __fmul_rn(x.y, dp));
        v2 = make_float2(__fmul_rn(x.x, dpp), __fmul_rn(x.y, dpp));
    }
    __device__ __forceinline__ void step(float2 x, float d, float dp, float dpp) {
        v0.x = fmaf(x.x, d, v0.x);
        v0.y = fmaf(x.y, d, v0.y);
        if (ORDER >= 1) {
            v1.x = fmaf(x.x, dp, v1.x);
            v1.y = fmaf(x.y, dp, v1.y);
        }
        if (ORDER >= 2) {
            v2.x = fmaf(x.x, dpp, v2.x);
            v2.y = fmaf(x.y, dpp, v2.y);
        }
    }
};

// C += wgt Re(z(m,m') ch) and its derivatives (alpha: -i m, gamma: -i m', beta: d', d'')
template <int ORDER, int NV>
__device__ __forceinline__ void phase_acc(float* ac, const Chain3<ORDER>& ch, float2 z, float wgt, int m, int mp) {
    const float fm = (float)m, fmp = (float)mp;
    const float wm = wgt * fm, wmp = wgt * fmp;
    const float2 v0 = cmul_x(z, ch.v0);
    ac[0] = fmaf(wgt, v0.x, ac[0]);
    if (ORDER >= 1) {
        const float2 v1 = cmul_x(z, ch.v1);
        ac[NV > 1 ? 1 : 0] = fmaf(wm, v0.y, ac[NV > 1 ? 1 : 0]);
        ac[NV > 2 ? 2 : 0] = fmaf(wgt, v1.x, ac[NV > 2 ? 2 : 0]);
        ac[NV > 3 ? 3 : 0] = fmaf(wmp, v0.y, ac[NV > 3 ? 3 : 0]);
        if (ORDER >= 2) {
            const float2 v2 = cmul_x(z, ch.v2);
            ac[NV > 4 ? 4 : 0] = fmaf(-__fmul_rn(wm, fm), v0.x, ac[NV > 4 ? 4 : 0]);
            ac[NV > 5 ? 5 : 0] = fmaf(wm, v1.y, ac[NV > 5 ? 5 : 0]);
            ac[NV > 6 ? 6 : 0] = fmaf(-__fmul_rn(wm, fmp), v0.x, ac[NV > 6 ? 6 : 0]);
            ac[NV > 7 ? 7 : 0] = fmaf(wgt, v2.x, ac[NV > 7 ? 7 : 0]);
            ac[NV > 8 ? 8 : 0] = fmaf(wmp, v1.y, ac[NV > 8 ? 8 : 0]);
            ac[NV > 9 ? 9 : 0] = fmaf(-__fmul_rn(wmp, fmp), v0.x, ac[NV > 9 ? 9 : 0]);
        }
    }
}

template <class WS>
__device__ __forceinline__ float2 phase_of(const WS& w, int m, int mp) {
    float2 pa = w.ua[abs(m)], pg = w.ug[abs(mp)];
    if (m < 0) pa.y = -pa.y;
    if (mp < 0) pg.y = -pg.y;
    return cmul_x(pa, pg);
}

// load-latency options of the evaluation (bit 0: refinement order 0, bit 1:
// refinement order 2, bit 2: sweep): L1 prefetch of the next group's kernel
// rows, and loads software-pipelined one chain step ahead
#ifndef BMB_PF_MASK
#define BMB_PF_MASK 2
#endif
#ifndef BMB_PIPE_MASK
#define BMB_PIPE_MASK 0
#endif
#ifndef BMB_PF_SMALL
#define BMB_PF_SMALL 1
#endif
#ifndef BMB_PF_MIN_GROUPS
#define BMB_PF_MIN_GROUPS 4
#endif
template <int ORDER, bool SWEEP>
struct EvalOpts {
    static constexpr int bit = SWEEP ? 4 : (ORDER == 2 ? 2 : 1);
    static constexpr bool PF = (BMB_PF_MASK & bit) != 0;
    static constexpr bool PIPE = (BMB_PIPE_MASK & bit) != 0;
};

// Sum NT per-lane values over the warp and publish sum i to out[i] (shared
// memory): recursive-halving reduce-scatter (P - 1 FP64 shuffles for P = next
// power of two >= NT, then plain butterfly rounds) instead of NT butterflies.
template <int NT>
__device__ __forceinline__ void warp_reduce_publish(double (&v)[NT], double* out) {
    constexpr int P = NT <= 1 ? 1 : NT <= 2 ? 2 : NT <= 4 ? 4 : NT <= 8 ? 8 : NT <= 16 ? 16 : 32;
    static_assert(NT <= 32, "reduce-scatter over at most 32 values");
    constexpr int LOGP = P == 1 ? 0 : P == 2 ? 1 : P == 4 ? 2 : P == 8 ? 3 : P == 16 ? 4 : 5;
    const int lane = threadIdx.x & 31;
    double w[P];
#pragma unroll
    for (int i = 0; i < P; ++i) w[i] = i < NT ? v[i] : 0.0;
#pragma unroll
    for (int r = 0; r < LOGP; ++r) {
        const int off = 16 >> r;
        const int half = P >> (r + 1);
        const bool low = (lane & off) == 0;
#pragma unroll
        for (int j = 0; j < half; ++j) {
            const double mine = low ? w[j] : w[j + half];
            const double send = low ? w[j + half] : w[j];
            w[j] = mine + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
#pragma unroll
    for (int r = LOGP; r < 5; ++r) w[0] += __shfl_xor_sync(0xffffffffu, w[0], 16 >> r);
    // lanes whose top LOGP bits equal i hold sum i
    int idx = 0;
#pragma unroll
    for (int r = 0; r < LOGP; ++r) idx = (idx << 1) | ((lane >> (4 - r)) & 1);
    if ((lane & ((32 >> LOGP) - 1)) == 0 && idx < NT) out[idx] = w[0];
}

// Evaluate K jobs at band T.L that share their kernels (job[k].xi == job[0].xi,
// job[k].wx == job[0].wx: rotations of one window, or of one particle in the
// sweep) — the correlation and, when WEDGE, the wedge-power kernel at the same
// angles.  Warp-cooperative; results in ws[k].res.  Each lane runs the
// Wigner-d recursion of its items (m, m'), m >= |m'|; one chain feeds both
// half-plane entries of an item (A and its partner B), and each table load
// feeds K chains.
template <int ORDER, int K, bool WEDGE, bool PF = false, bool PIPE = false>
__device__ __forceinline__ void warp_eval_k(const BandTables& T, const EvalJob (&job)[K], WarpScratch* ws) {
    const float4* __restrict__ xi = job[0].xi;
    const float4* __restrict__ wx = job[0].wx;
    const int lane = threadIdx.x & 31;
    const int L = T.L;
    // the kernels are streamed once per evaluation: group g+1's rows are pulled
    // into L1 while group g runs (L2 latency off the recursion's critical path)
    // (kernels staged in shared memory by the fused refinement are not prefetched)
    // (low bands: a group or two of short rows, nothing to hide the prefetch behind)
    const bool pf_x = PF && T.n_groups > BMB_PF_MIN_GROUPS && __isGlobal(xi);
    const bool pf_w = PF && WEDGE && T.n_groups > BMB_PF_MIN_GROUPS && __isGlobal(wx);
    if (T.n_groups > 0) {
        if (pf_x) prefetch_rows(xi, T.row_off[0], T.row_off[1], lane);
        if (pf_w) prefetch_rows(wx, T.row_off[0], T.row_off[1], lane);
    }
    __syncwarp();
    // four FP64 sincos per job on lanes 4k..4k+3 (beta/2, beta, alpha, gamma);
    // the phases e^{-i m alpha}, e^{-i m gamma} are binary powers of the bases
    if (lane < 4 * K) {
        const int c = lane & 3;
        double ang = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k)
            if ((lane >> 2) == k) ang = c == 0 ? 0.5 * job[k].b : (c == 1 ? job[k].b : (c == 2 ? job[k].a : job[k].g));
        double sn, co;
        sincos_d(ang, &sn, &co);
        ws[lane >> 2].cs_half[2 * c] = co;
        ws[lane >> 2].cs_half[2 * c + 1] = sn;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double car = ws[k].cs_half[4], cai = -ws[k].cs_half[5];  // e^{-i alpha}
        const double cgr = ws[k].cs_half[6], cgi = -ws[k].cs_half[7];  // e^{-i gamma}
        for (int m = lane; m <= L; m += 32) {
            double ar = 1.0, ai = 0.0, gr = 1.0, gi = 0.0;
            double br_ = car, bi_ = cai, hr = cgr, hi = cgi;
            for (int e = m; e; e >>= 1) {
                if (e & 1) {
                    const double t = ar * br_ - ai * bi_;
                    ai = ar * bi_ + ai * br_;
                    ar = t;
                    const double u = gr * hr - gi * hi;
                    gi = gr * hi + gi * hr;
                    gr = u;
                }
                const double t2 = br_ * br_ - bi_ * bi_;
                bi_ = 2.0 * br_ * bi_;
                br_ = t2;
                const double u2 = hr * hr - hi * hi;
                hi = 2.0 * hr * hi;
                hr = u2;
            }
            ws[k].ua[m] = make_float2((float)ar, (float)ai);
            ws[k].ug[m] = make_float2((float)gr, (float)gi);
        }
        const double ch = ws[k].cs_half[0], sh = ws[k].cs_half[1];
        for (int j = lane; j <= 2 * L + 2; j += 32) {
            double pc = 1.0, ps = 1.0, bc = ch, bs = sh;
            for (int e = j; e; e >>= 1) {
                if (e & 1) {
                    pc *= bc;
                    ps *= bs;
                }
                bc *= bc;
                bs *= bs;
            }
            ws[k].cp[j] = (float)pc;
            ws[k].sp[j] = (float)ps;
        }
    }
    __syncwarp();
    float cb[K], sb[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        cb[k] = (float)ws[k].cs_half[2];
        sb[k] = (float)ws[k].cs_half[3];
    }

    constexpr int NV = ORDER == 0 ? 1 : (ORDER == 1 ? 4 : 10);
    float acc[K][NV], accw[K][NV];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int i = 0; i < NV; ++i) acc[k][i] = accw[k][i] = 0.0f;

    for (int g = 0; g < T.n_groups; ++g) {
        const int item = g * 32 + lane;
        const int r0 = T.row_off[g];
        const int glen = T.row_off[g + 1] - r0;
        if ((pf_x || pf_w) && g + 1 < T.n_groups) {
            const int n0 = T.row_off[g + 1], n1 = T.row_off[g + 2];
            if (pf_x) prefetch_rows(xi, n0, n1, lane);
            if (pf_w) prefetch_rows(wx, n0, n1, lane);
        }
        const int be = T.bexp[item];
        const int ea = be & 0xff, ep = be >> 8;
        const float bf = T.bfac[item];
        float d[K], dp[K], dpp[K], d1[K], dp1[K], dpp1[K];
        Chain3<ORDER> CA[K], CB[K], WA[K], WB[K];
        const float4* __restrict__ pq = T.PQR + r0 * 32 + lane;
        const float4* __restrict__ xr = xi + r0 * 32 + lane;
        const float4* __restrict__ wr = WEDGE ? wx + r0 * 32 + lane : nullptr;
        const float4 x0 = xr[0];
        const float4 w0 = WEDGE ? wr[0] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            // closed-form border at l0 = m (cs_power, steer.cpp:19-31)
            const float* cp = ws[k].cp;
            const float* sp = ws[k].sp;
            d[k] = __fmul_rn(__fmul_rn(bf, cp[ea]), sp[ep]);
            dp[k] = dpp[k] = d1[k] = dp1[k] = dpp1[k] = 0.0f;
            if (ORDER >= 1) {
                const float tb = ep ? __fmul_rn(__fmul_rn((float)ep, cp[ea + 1]), sp[ep - 1]) : 0.0f;
                const float ta = ea ? __fmul_rn(__fmul_rn((float)ea, cp[ea - 1]), sp[ep + 1]) : 0.0f;
                dp[k] = __fmul_rn(__fmul_rn(0.5f, bf), __fsub_rn(tb, ta));
            }
            if (ORDER >= 2) {
                const float t2b = ep > 1 ? __fmul_rn(__fmul_rn(ep * (ep - 1.0f), cp[ea + 2]), sp[ep - 2]) : 0.0f;
                const float t2a = ea > 1 ? __fmul_rn(__fmul_rn(ea * (ea - 1.0f), cp[ea - 2]), sp[ep + 2]) : 0.0f;
                const float mid = __fmul_rn(__fmul_rn(2.0f * ea * ep + ea + ep, cp[ea]), sp[ep]);
                dpp[k] = __fmul_rn(__fmul_rn(0.25f, bf), __fsub_rn(__fadd_rn(t2b, t2a), mid));
            }
            CA[k].init(make_float2(x0.x, x0.y), d[k], dp[k], dpp[k]);
            CB[k].init(make_float2(x0.z, x0.w), d[k], dp[k], dpp[k]);
            if (WEDGE) {
                WA[k].init(make_float2(w0.x, w0.y), d[k], dp[k], dpp[k]);
                WB[k].init(make_float2(w0.z, w0.w), d[k], dp[k], dpp[k]);
            }
        }
        // optionally software-pipelined one step ahead
        float4 pqn = (PIPE && glen > 1) ? __ldg(pq + 32) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 xn = (PIPE && glen > 1) ? xr[32] : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 wn = (PIPE && WEDGE && glen > 1) ? wr[32] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 2
        for (int s = 1; s < glen; ++s) {
            float4 pqr, x, w;
            if (PIPE) {
                pqr = pqn;
                x = xn;
                w = wn;
                if (s + 1 < glen) {
                    pqn = __ldg(pq + (s + 1) * 32);
                    xn = xr[(s + 1) * 32];
                    if (WEDGE) wn = wr[(s + 1) * 32];
                }
            } else {
                pqr = __ldg(pq + s * 32);
                x = xr[s * 32];
                w = WEDGE ? wr[s * 32] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            const float P = pqr.x, Q = pqr.y, R = pqr.z;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                // three-term recursion (steer.cpp:101-141): t1 = P cos b + Q, t2 = R
                const float t1 = fmaf(P, cb[k], Q);
                const float dn = fmaf(t1, d[k], -__fmul_rn(R, d1[k]));
                float dpn = 0.0f, dppn = 0.0f;
                if (ORDER >= 1) {
                    const float t1p = __fmul_rn(-P, sb[k]);
                    dpn = fmaf(t1p, d[k], fmaf(t1, dp[k], -__fmul_rn(R, dp1[k])));
                    if (ORDER >= 2) {
                        const float t1pp = __fmul_rn(-P, cb[k]);
                        dppn = fmaf(t1pp, d[k], fmaf(2.0f * t1p, dp[k], fmaf(t1, dpp[k], -__fmul_rn(R, dpp1[k]))));
                    }
                }
                d1[k] = d[k];
                d[k] = dn;
                if (ORDER >= 1) {
                    dp1[k] = dp[k];
                    dp[k] = dpn;
                }
                if (ORDER >= 2) {
                    dpp1[k] = dpp[k];
                    dpp[k] = dppn;
                }
                CA[k].step(make_float2(x.x, x.y), d[k], dp[k], dpp[k]);
                CB[k].step(make_float2(x.z, x.w), d[k], dp[k], dpp[k]);
                if (WEDGE) {
                    WA[k].step(make_float2(w.x, w.y), d[k], dp[k], dpp[k]);
                    WB[k].step(make_float2(w.z, w.w), d[k], dp[k], dpp[k]);
                }
            }
        }
        const char2 mm = T.item_mm[item], pm = T.item_pm[item];
        const float2 iw = T.item_w[item];  // (weight A, sign * weight B)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            // phases e^{-i m a} e^{-i m' g}; conj for negative orders
            const float2 za = phase_of(ws[k], mm.x, mm.y), zb = phase_of(ws[k], pm.x, pm.y);
            phase_acc<ORDER, NV>(acc[k], CA[k], za, iw.x, mm.x, mm.y);
            phase_acc<ORDER, NV>(acc[k], CB[k], zb, iw.y, pm.x, pm.y);
            if (WEDGE) {
                phase_acc<ORDER, NV>(accw[k], WA[k], za, iw.x, mm.x, mm.y);
                phase_acc<ORDER, NV>(accw[k], WB[k], zb, iw.y, pm.x, pm.y);
            }
        }
    }
    // cross-lane reduction in FP64, published through shared memory
    constexpr int NW = WEDGE ? 2 : 1;
    constexpr int NT = NW * NV * K;
    double v[NT];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            v[NW * NV * k + i] = acc[k][i];
            if (WEDGE) v[NW * NV * k + (NW - 1) * NV + i] = accw[k][i];
        }
    if constexpr (NT <= 32) {
        double* red = ws[0].red;  // reduced sums, then scattered to the per-job results
        warp_reduce_publish<NT>(v, red);
        __syncwarp();
        if (lane < K * NV) {
            const int k = lane / NV, i = lane % NV;
            const double c = red[NW * NV * k + i];
            const double wv = WEDGE ? red[NW * NV * k + (NW - 1) * NV + i] : 0.0;
#pragma unroll
            for (int kk = 0; kk < K; ++kk)
                if (kk == k) {
                    ws[kk].res[i] = c;
                    ws[kk].res[10 + i] = wv;
                }
        }
    } else {
#pragma unroll
        for (int o = 16; o; o >>= 1)
#pragma unroll
            for (int i = 0; i < NT; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    ws[k].res[i] = v[NW * NV * k + i];
                    ws[k].res[10 + i] = WEDGE ? v[NW * NV * k + (NW - 1) * NV + i] : 0.0;
                }
        }
    }
    __syncwarp();
}

// ---------------------------------------------------------------- half-warp jobs
// Two evaluations per warp, one per 16-lane half.  At low bands a job's chains
// are short (L = 4: 25 items in one group of 32 lanes), and the per-job work
// around them -- four FP64 sincos, the phase powers, the FP64 reduction of 20
// sums -- costs as much as the chains.  A half-warp walks each 32-lane group of
// the band layout in two passes of 16 items (each pass only as long as its
// longest chain: items are sorted by chain length), and the per-job work runs
// on both halves at once.  Same tables, same per-item FP32 sequence as the
// full-warp kernel; only the lane partition of the items (hence the FP32
// partial sums) differs.
template <int NT, int LANES>
__device__ __forceinline__ void sub_reduce_publish(double (&v)[NT], double* out) {
    constexpr int P = NT <= 1 ? 1 : NT <= 2 ? 2 : NT <= 4 ? 4 : NT <= 8 ? 8 : NT <= 16 ? 16 : 32;
    static_assert(NT <= 32, "reduce-scatter over at most 32 values");
    static_assert(LANES == 8 || LANES == 16, "8- or 16-lane jobs");
    constexpr int LOGP = P == 1 ? 0 : P == 2 ? 1 : P == 4 ? 2 : P == 8 ? 3 : P == 16 ? 4 : 5;
    constexpr int LB = LANES == 16 ? 4 : 3;  // lane bits of a job
    constexpr int R = LOGP < LB ? LOGP : LB;  // halving rounds over the job's lanes
    constexpr int KEEP = P >> R;              // sums left per lane
    const int ls = threadIdx.x & (LANES - 1);
    double w[P];
#pragma unroll
    for (int i = 0; i < P; ++i) w[i] = i < NT ? v[i] : 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int off = (LANES / 2) >> r;
        const int half = P >> (r + 1);
        const bool low = (ls & off) == 0;
#pragma unroll
        for (int j = 0; j < half; ++j) {
            const double mine = low ? w[j] : w[j + half];
            const double send = low ? w[j + half] : w[j];
            w[j] = mine + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
#pragma unroll
    for (int r = R; r < LB; ++r) w[0] += __shfl_xor_sync(0xffffffffu, w[0], (LANES / 2) >> r);
    // position j of this lane holds sum j + sum_r b_r P / 2^(r+1), b_r = lane bit (LB - 1 - r)
    int base = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) base += ((ls >> (LB - 1 - r)) & 1) * (P >> (r + 1));
    if ((ls & ((LANES >> R) - 1)) == 0) {
#pragma unroll
        for (int j = 0; j < KEEP; ++j)
            if (base + j < NT) out[base + j] = w[j];
    }
}

#ifndef BMB_SUB_PIPE
#define BMB_SUB_PIPE 0
#endif
template <int ORDER, bool WEDGE, bool PF, int LANES, class WS>
__device__ __forceinline__ void warp_eval_sub(const BandTables& T, const EvalJob& job, WS* ws) {
    constexpr int PASSES = 32 / LANES;
    constexpr bool SUB_PIPE = BMB_SUB_PIPE != 0;
    const float4* __restrict__ xi = job.xi;
    const float4* __restrict__ wx = job.wx;
    const int l16 = threadIdx.x & (LANES - 1);
    const int L = T.L;
    const bool pf_x = PF && T.n_groups > BMB_PF_MIN_GROUPS && __isGlobal(xi);
    const bool pf_w = PF && WEDGE && T.n_groups > BMB_PF_MIN_GROUPS && __isGlobal(wx);
    // L1 prefetch of rows [r0, r1) of this half's kernel: 16 lanes, one line each per pass
    auto prefetch_half = [&](const float4* k, int r0, int r1) {
        const char* b = reinterpret_cast<const char*>(k + (size_t)r0 * 32);
        const int bytes = (r1 - r0) * 512;
        for (int off = l16 * 128; off < bytes; off += LANES * 128) prefetch_l1(b + off);
    };
    if (T.n_groups > 0) {
        if (pf_x) prefetch_half(xi, T.row_off[0], T.row_off[1]);
        if (pf_w) prefetch_half(wx, T.row_off[0], T.row_off[1]);
        // low bands: the job's whole window kernel is a few KB; request it now so that
        // it arrives behind the sincos and the phase powers (BMB_PF_SMALL=0: off)
        if (BMB_PF_SMALL && PF && !pf_x && __isGlobal(xi)) prefetch_half(xi, T.row_off[0], T.row_off[T.n_groups]);
    }
    // four FP64 sincos per job on lanes 0..3 of its half (beta/2, beta, alpha, gamma)
    if (l16 < 4) {
        const double ang = l16 == 0 ? 0.5 * job.b : (l16 == 1 ? job.b : (l16 == 2 ? job.a : job.g));
        double sn, co;
        sincos_d(ang, &sn, &co);
        ws->cs_half[2 * l16] = co;
        ws->cs_half[2 * l16 + 1] = sn;
    }
    __syncwarp();
    {
        const double car = ws->cs_half[4], cai = -ws->cs_half[5];  // e^{-i alpha}
        const double cgr = ws->cs_half[6], cgi = -ws->cs_half[7];  // e^{-i gamma}
        for (int m = l16; m <= L; m += LANES) {
            double ar = 1.0, ai = 0.0, gr = 1.0, gi = 0.0;
            double br_ = car, bi_ = cai, hr = cgr, hi = cgi;
            for (int e = m; e; e >>= 1) {
                if (e & 1) {
                    const double t = ar * br_ - ai * bi_;
                    ai = ar * bi_ + ai * br_;
                    ar = t;
                    const double u = gr * hr - gi * hi;
                    gi = gr * hi + gi * hr;
                    gr = u;
                }
                const double t2 = br_ * br_ - bi_ * bi_;
                bi_ = 2.0 * br_ * bi_;
                br_ = t2;
                const double u2 = hr * hr - hi * hi;
                hi = 2.0 * hr * hi;
                hr = u2;
            }
            ws->ua[m] = make_float2((float)ar, (float)ai);
            ws->ug[m] = make_float2((float)gr, (float)gi);
        }
        const double ch = ws->cs_half[0], sh = ws->cs_half[1];
        for (int j = l16; j <= 2 * L + 2; j += LANES) {
            double pc = 1.0, ps = 1.0, bc = ch, bs = sh;
            for (int e = j; e; e >>= 1) {
                if (e & 1) {
                    pc *= bc;
                    ps *= bs;
                }
                bc *= bc;
                bs *= bs;
            }
            ws->cp[j] = (float)pc;
            ws->sp[j] = (float)ps;
        }
    }
    __syncwarp();
    const float cb = (float)ws->cs_half[2], sb = (float)ws->cs_half[3];
    const float* cp = ws->cp;
    const float* sp = ws->sp;

    constexpr int NV = ORDER == 0 ? 1 : (ORDER == 1 ? 4 : 10);
    float acc[NV], accw[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = accw[i] = 0.0f;

    for (int g = 0; g < T.n_groups; ++g) {
        const int r0 = T.row_off[g];
        if ((pf_x || pf_w) && g + 1 < T.n_groups) {
            const int n0 = T.row_off[g + 1], n1 = T.row_off[g + 2];
            if (pf_x) prefetch_half(xi, n0, n1);
            if (pf_w) prefetch_half(wx, n0, n1);
        }
#pragma unroll 1
        for (int p = 0; p < PASSES; ++p) {
            const int slot = p * LANES + l16;
            const int item = g * 32 + slot;
            const int plen = T.item_len[g * 32 + p * LANES];  // the pass's longest chain (0: padding)
            if (plen == 0) break;
            const int be = T.bexp[item];
            const int ea = be & 0xff, ep = be >> 8;
            const float bf = T.bfac[item];
            const float4* __restrict__ pq = T.PQR + r0 * 32 + slot;
            const float4* __restrict__ xr = xi + r0 * 32 + slot;
            const float4* __restrict__ wr = WEDGE ? wx + r0 * 32 + slot : nullptr;
            const float4 x0 = xr[0];
            const float4 w0 = WEDGE ? wr[0] : make_float4(0.f, 0.f, 0.f, 0.f);
            float d = __fmul_rn(__fmul_rn(bf, cp[ea]), sp[ep]);
            float dp = 0.0f, dpp = 0.0f, d1 = 0.0f, dp1 = 0.0f, dpp1 = 0.0f;
            if (ORDER >= 1) {
                const float tb = ep ? __fmul_rn(__fmul_rn((float)ep, cp[ea + 1]), sp[ep - 1]) : 0.0f;
                const float ta = ea ? __fmul_rn(__fmul_rn((float)ea, cp[ea - 1]), sp[ep + 1]) : 0.0f;
                dp = __fmul_rn(__fmul_rn(0.5f, bf), __fsub_rn(tb, ta));
            }
            if (ORDER >= 2) {
                const float t2b = ep > 1 ? __fmul_rn(__fmul_rn(ep * (ep - 1.0f), cp[ea + 2]), sp[ep - 2]) : 0.0f;
                const float t2a = ea > 1 ? __fmul_rn(__fmul_rn(ea * (ea - 1.0f), cp[ea - 2]), sp[ep + 2]) : 0.0f;
                const float mid = __fmul_rn(__fmul_rn(2.0f * ea * ep + ea + ep, cp[ea]), sp[ep]);
                dpp = __fmul_rn(__fmul_rn(0.25f, bf), __fsub_rn(__fadd_rn(t2b, t2a), mid));
            }
            Chain3<ORDER> CA, CB, WA, WB;
            CA.init(make_float2(x0.x, x0.y), d, dp, dpp);
            CB.init(make_float2(x0.z, x0.w), d, dp, dpp);
            if (WEDGE) {
                WA.init(make_float2(w0.x, w0.y), d, dp, dpp);
                WB.init(make_float2(w0.z, w0.w), d, dp, dpp);
            }
            float4 pqn = (SUB_PIPE && plen > 1) ? __ldg(pq + 32) : make_float4(0.f, 0.f, 0.f, 0.f);
            float4 xn = (SUB_PIPE && plen > 1) ? xr[32] : make_float4(0.f, 0.f, 0.f, 0.f);
            float4 wn = (SUB_PIPE && WEDGE && plen > 1) ? wr[32] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 2
            for (int s = 1; s < plen; ++s) {
                float4 pqr, x, w;
                if (SUB_PIPE) {
                    pqr = pqn;
                    x = xn;
                    w = wn;
                    if (s + 1 < plen) {
                        pqn = __ldg(pq + (s + 1) * 32);
                        xn = xr[(s + 1) * 32];
                        if (WEDGE) wn = wr[(s + 1) * 32];
                    }
                } else {
                    pqr = __ldg(pq + s * 32);
                    x = xr[s * 32];
                    w = WEDGE ? wr[s * 32] : make_float4(0.f, 0.f, 0.f, 0.f);
                }
                const float P = pqr.x, Q = pqr.y, R = pqr.z;
                const float t1 = fmaf(P, cb, Q);
                const float dn = fmaf(t1, d, -__fmul_rn(R, d1));
                float dpn = 0.0f, dppn = 0.0f;
                if (ORDER >= 1) {
                    const float t1p = __fmul_rn(-P, sb);
                    dpn = fmaf(t1p, d, fmaf(t1, dp, -__fmul_rn(R, dp1)));
                    if (ORDER >= 2) {
                        const float t1pp = __fmul_rn(-P, cb);
                        dppn = fmaf(t1pp, d, fmaf(2.0f * t1p, dp, fmaf(t1, dpp, -__fmul_rn(R, dpp1))));
                    }
                }
                d1 = d;
                d = dn;
                if (ORDER >= 1) {
                    dp1 = dp;
                    dp = dpn;
                }
                if (ORDER >= 2) {
                    dpp1 = dpp;
                    dpp = dppn;
                }
                CA.step(make_float2(x.x, x.y), d, dp, dpp);
                CB.step(make_float2(x.z, x.w), d, dp, dpp);
                if (WEDGE) {
                    WA.step(make_float2(w.x, w.y), d, dp, dpp);
                    WB.step(make_float2(w.z, w.w), d, dp, dpp);
                }
            }
            const char2 mm = T.item_mm[item], pm = T.item_pm[item];
            const float2 iw = T.item_w[item];
            const float2 za = phase_of(*ws, mm.x, mm.y), zb = phase_of(*ws, pm.x, pm.y);
            phase_acc<ORDER, NV>(acc, CA, za, iw.x, mm.x, mm.y);
            phase_acc<ORDER, NV>(acc, CB, zb, iw.y, pm.x, pm.y);
            if (WEDGE) {
                phase_acc<ORDER, NV>(accw, WA, za, iw.x, mm.x, mm.y);
                phase_acc<ORDER, NV>(accw, WB, zb, iw.y, pm.x, pm.y);
            }
        }
    }
    constexpr int NW = WEDGE ? 2 : 1;
    constexpr int NT = NW * NV;
    double v[NT];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        v[i] = acc[i];
        if (WEDGE) v[NV + i] = accw[i];
    }
    sub_reduce_publish<NT, LANES>(v, ws->red);
    __syncwarp();
    for (int i = l16; i < NV; i += LANES) {
        ws->res[i] = ws->red[i];
        ws->res[10 + i] = WEDGE ? ws->red[NV + i] : 0.0;
    }
    __syncwarp();
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// warp-aggregated ordered append: the predicated lanes append v in lane order
// (lists keep the candidate order of their producers, so the candidates of a
// window stay adjacent and can evaluate K-way)
__device__ __forceinline__ void wappend(bool pred, int v, int* list, int* count) {
    const unsigned m = __ballot_sync(0xffffffffu, pred);
    if (!m) return;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if ((threadIdx.x & 31) == leader) base = atomicAdd(count, __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (pred) list[base + __popc(m & lanemask_lt())] = v;
}

// xi_l[m,m'] = sum_k conj(f_klm) t_klm' from real-packed f and t
__device__ float2 xi_value(int l, int m, int mp, const float* f, const float* t, const int* block_off,
                           const int* radial_count) {
    const int nk = radial_count[l], base = block_off[l];
    const int am = abs(m), amp = abs(mp);
    const float sm = (m < 0 && (am & 1)) ? -1.0f : 1.0f;
    const float smp = (mp < 0 && (amp & 1)) ? -1.0f : 1.0f;
    float re = 0.0f, im = 0.0f;
    for (int k = 0; k < nk; ++k) {
        const float* fr = f + base + k * (2 * l + 1);
        const float* tr = t + base + k * (2 * l + 1);
        float fre = fr[am == 0 ? 0 : 2 * am - 1], fim = am == 0 ? 0.0f : fr[2 * am];
        if (m < 0) fre *= sm, fim *= -sm;
        float tre = tr[amp == 0 ? 0 : 2 * amp - 1], tim = amp == 0 ? 0.0f : tr[2 * amp];
        if (mp < 0) tre *= smp, tim *= -smp;
        re = fmaf(fre, tre, fmaf(fim, tim, re));  // conj(f) * t
        im = fmaf(fre, tim, fmaf(-fim, tre, im));
    }
    return make_float2(re, im);
}

// band-layout entry (row, lane): (xi_l[A], xi_l[B]) of the lane's item
__device__ float4 xi_entry(const BandTables& T, const int* row_group, const float* f, const float* t,
                           const int* block_off, const int* radial_count, int row, int lane) {
    const int2 dsc = T.at_desc[row * 32 + lane];  // degree and entries of the position
    if (!(dsc.x & 1)) return make_float4(0.f, 0.f, 0.f, 0.f);
    const int l = (dsc.x >> 2) & 63;
    const float2 xa = xi_value(l, ((dsc.x >> 8) & 255) - 64, ((dsc.x >> 16) & 255) - 64, f, t, block_off,
                               radial_count);
    const float2 xb = !(dsc.x & 2) ? make_float2(0.f, 0.f)
                                   : xi_value(l, (dsc.y & 255) - 64, ((dsc.y >> 8) & 255) - 64, f, t, block_off,
                                              radial_count);
    return make_float4(xa.x, xa.y, xb.x, xb.y);
}


// ---------------------------------------------------------------- scalar Newton
struct Derivs {
    double v;
    double g[3];
    double h[9];
};

__device__ void unpack(const double* res, int order, Derivs& c) {
    c.v = res[0];
    if (order >= 1) c.g[0] = res[1], c.g[1] = res[2], c.g[2] = res[3];
    if (order >= 2) {  // res: aa ab ag bb bg gg
        c.h[0] = res[4], c.h[1] = res[5], c.h[2] = res[6];
        c.h[3] = res[5], c.h[4] = res[7], c.h[5] = res[8];
        c.h[6] = res[6], c.h[7] = res[8], c.h[8] = res[9];
    }
}

// Objective::eval (src/optimize.cpp:106-130): C / sqrt(clamp(1 - rho, 0.02, 2))
__device__ void objective(const double* cr, const double* rr, bool wedge, int order, Derivs& f) {
    Derivs c, r;
    unpack(cr, order, c);
    if (!wedge) {
        f = c;
        return;
    }
    unpack(rr, order, r);
    const double v = fmin(fmax(1.0 - r.v, 0.02), 2.0);
    const double s = 1.0 / sqrt(v);
    f.v = c.v * s;
    if (order >= 1) {
        const double dv[3] = {-r.g[0], -r.g[1], -r.g[2]};
        const double v32 = s / v;
        for (int i = 0; i < 3; ++i) f.g[i] = c.g[i] * s - 0.5 * c.v * v32 * dv[i];
        if (order >= 2) {
            const double v52 = v32 / v;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    const double hv = -r.h[i * 3 + j];
                    f.h[i * 3 + j] = c.h[i * 3 + j] * s -
                                     0.5 * v32 * (c.g[i] * dv[j] + dv[i] * c.g[j] + c.v * hv) +
                                     0.75 * c.v * v52 * dv[i] * dv[j];
                }
        }
    }
}

// Chart derivatives of an anchored candidate without a per-candidate kernel.
// The reference optimizes C~(e) = C(R(e) a) on the composed kernel
// xi~ = xi D(a)^T (xi_compose_right, src/xcorr.cpp:149-155; refine(),
// src/optimize.cpp:268-299).  The same function and its e-derivatives follow
// from the window's own kernels: the objective is evaluated at the global
// rotation g = R(e) a, either on the window kernel at Euler angles e' = E(g),
// or — when g itself is near a pole — on the window's side kernel
// xi' = xi D(K^-1)^T at e' = E(g K) (K = ZYZ(0, pi/2, 0); g and g K are never
// both within 45 degrees of a pole).  Derivatives then map to the chart by the
// chain rule through e -> e'.  With W(e) = [z, Rz(a) y, Rz(a) Ry(b) z] (the
// space-frame angular velocities of the ZYZ angles, dR/de_i = [w_i]x R), both
// parametrizations move g with the same angular velocity, so
//   J = de'/de = W(e')^-1 W(e),
//   d^2 e'_k / de_i de_j = (W(e')^-1 (dW(e)/de_j - sum_k J_kj dW(e')/de'_k J))_ki,
//   grad = J^T grad',  H = J^T H' J + sum_k grad'_k d^2 e'_k / de de.
// cs = (cos a, sin a, cos b, sin b) of the ZYZ angles of q (rotation.cpp:77-93:
// a = atan2(m12, m02), b = atan2(hypot(m02, m12), m22)), from the matrix entries
__device__ __forceinline__ void frame_trig(const Quat& q, double cs[4]) {
    const double m02 = 2 * (q.x * q.z + q.w * q.y), m12 = 2 * (q.y * q.z - q.w * q.x);
    const double m22 = 1 - 2 * (q.x * q.x + q.y * q.y);
    const double sb = hypot(m02, m12);
    cs[0] = m02 / sb, cs[1] = m12 / sb;
    cs[2] = m22, cs[3] = sb;
    const double rb = rhypot(m22, sb);  // the matrix of a unit quaternion has m22^2 + sb^2 = 1 up to rounding
    cs[2] *= rb, cs[3] *= rb;
}

__device__ void euler_frame(const double cs[4], double W[9], double dWa[9], double dWb[9]) {
    const double ca = cs[0], sa = cs[1], cb = cs[2], sb = cs[3];
    // columns: w_alpha = z, w_beta = (-sin a, cos a, 0), w_gamma = (cos a sin b, sin a sin b, cos b)
    W[0] = 0.0, W[1] = -sa, W[2] = ca * sb;
    W[3] = 0.0, W[4] = ca, W[5] = sa * sb;
    W[6] = 1.0, W[7] = 0.0, W[8] = cb;
    dWa[0] = 0.0, dWa[1] = -ca, dWa[2] = -sa * sb;
    dWa[3] = 0.0, dWa[4] = -sa, dWa[5] = ca * sb;
    dWa[6] = 0.0, dWa[7] = 0.0, dWa[8] = 0.0;
    dWb[0] = 0.0, dWb[1] = 0.0, dWb[2] = ca * cb;
    dWb[3] = 0.0, dWb[4] = 0.0, dWb[5] = sa * cb;
    dWb[6] = 0.0, dWb[7] = 0.0, dWb[8] = -sb;
}

__device__ void mat3_mul(const double* A, const double* B, double* C) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) C[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
}

// f: objective at e' (value, gradient, Hessian in e' = ev); rewritten in place
// as the derivatives with respect to the chart angles e (te, tv: the frames' trig)
__device__ void chart_transform(Derivs& f, const double* te, const double* tv) {
    double We[9], dWe_a[9], dWe_b[9], Wp[9], dWp_a[9], dWp_b[9];
    euler_frame(te, We, dWe_a, dWe_b);
    euler_frame(tv, Wp, dWp_a, dWp_b);
    // W(e')^-1 by the adjugate (det = -sin b' != 0: b' is at least 45 degrees from a pole)
    double Wi[9];
    Wi[0] = Wp[4] * Wp[8] - Wp[5] * Wp[7];
    Wi[1] = Wp[2] * Wp[7] - Wp[1] * Wp[8];
    Wi[2] = Wp[1] * Wp[5] - Wp[2] * Wp[4];
    Wi[3] = Wp[5] * Wp[6] - Wp[3] * Wp[8];
    Wi[4] = Wp[0] * Wp[8] - Wp[2] * Wp[6];
    Wi[5] = Wp[2] * Wp[3] - Wp[0] * Wp[5];
    Wi[6] = Wp[3] * Wp[7] - Wp[4] * Wp[6];
    Wi[7] = Wp[1] * Wp[6] - Wp[0] * Wp[7];
    Wi[8] = Wp[0] * Wp[4] - Wp[1] * Wp[3];
    const double det = Wp[0] * Wi[0] + Wp[1] * Wi[3] + Wp[2] * Wi[6];
    const double rdet = 1.0 / det;
    for (int i = 0; i < 9; ++i) Wi[i] *= rdet;
    double J[9];
    mat3_mul(Wi, We, J);
    double g[3], H[9];
    for (int i = 0; i < 3; ++i) g[i] = J[i] * f.g[0] + J[3 + i] * f.g[1] + J[6 + i] * f.g[2];
    double HJ[9];
    mat3_mul(f.h, J, HJ);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) H[3 * i + j] = J[i] * HJ[j] + J[3 + i] * HJ[3 + j] + J[6 + i] * HJ[6 + j];
    const double* dWe[3] = {dWe_a, dWe_b, nullptr};
    for (int j = 0; j < 3; ++j) {
        // M = dW(e)/de_j - (J_0j dW(e')/da' + J_1j dW(e')/db') J
        double T[9], TJ[9], M[9], dJ[9];
        for (int q = 0; q < 9; ++q) T[q] = J[j] * dWp_a[q] + J[3 + j] * dWp_b[q];
        mat3_mul(T, J, TJ);
        for (int q = 0; q < 9; ++q) M[q] = (dWe[j] ? dWe[j][q] : 0.0) - TJ[q];
        mat3_mul(Wi, M, dJ);  // dJ[k][i] = d^2 e'_k / de_i de_j
        for (int i = 0; i < 3; ++i) H[3 * i + j] += dJ[i] * f.g[0] + dJ[3 + i] * f.g[1] + dJ[6 + i] * f.g[2];
    }
    for (int i = 0; i < 3; ++i) f.g[i] = g[i];
    for (int q = 0; q < 9; ++q) f.h[q] = H[q];
}

// damped step from wk.f with wk.lam, trial chart rotation (optimize.cpp:313-328)
// The trial's order-0 evaluation needs only the objective VALUE, which is smooth
// through the gimbal pole: an anchored candidate is evaluated at the global trial
// rotation h_try * a on the window kernel (C~(h) = C(h a), xcorr.cpp:149-155)
// instead of streaming its private chart kernels; et holds those angles.
__device__ __forceinline__ Quat qload(const double* q);
__device__ __forceinline__ void choose_frame(const Quat& g, const Quat& koff, double* ev, int& side, double* tv);
__device__ void make_trial(CandWork& wk, const CandState& st, const Quat& koff) {
    double m[9];
    for (int i = 0; i < 9; ++i) m[i] = wk.f[4 + i];
    m[0] -= wk.lam;
    m[4] -= wk.lam;
    m[8] -= wk.lam;
    const double g[3] = {wk.f[1], wk.f[2], wk.f[3]};
    double p[3];
    LU3 lu;
    lu.factor(m);
    if (lu.invertible()) {
        double x[3];
        lu.solve(g, x);
        p[0] = -x[0], p[1] = -x[1], p[2] = -x[2];
    } else {
        p[0] = g[0] / wk.lam, p[1] = g[1] / wk.lam, p[2] = g[2] / wk.lam;
    }
    const double pn = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
    if (pn > 1.0) {
        const double sc = 1.0 / pn;
        p[0] *= sc, p[1] *= sc, p[2] *= sc;
    }
    const Quat h = q_from_euler(wk.e[0] + p[0], wk.e[1] + p[1], wk.e[2] + p[2]);
    wk.gt[0] = h.w, wk.gt[1] = h.x, wk.gt[2] = h.y, wk.gt[3] = h.z;
    // frame of the trial's order-2 evaluation: the global angles (unanchored: the
    // next iteration's chart angles exactly), or for an anchored candidate the
    // better-conditioned of g and g K (its global angles et are not needed)
    if (st.anchored) {
        choose_frame(q_mul(h, qload(st.anchor)), koff, wk.evt, wk.sidet, wk.tvt);
    } else {
        const Euler3 et = q_euler(h);
        wk.et[0] = et.a, wk.et[1] = et.b, wk.et[2] = et.g;
        wk.evt[0] = et.a, wk.evt[1] = et.b, wk.evt[2] = et.g;
        wk.sidet = 0;
    }
}

__device__ __forceinline__ Quat qload(const double* q) { return Quat{q[0], q[1], q[2], q[3]}; }
__device__ __forceinline__ void qstore(double* d, const Quat& q) {
    d[0] = q.w, d[1] = q.x, d[2] = q.y, d[3] = q.z;
}

__device__ __forceinline__ bool slot_of(const StageArgs& a, long long idx) {
    const int w = (int)(idx / a.max_cand), c = (int)(idx % a.max_cand);
    return w < a.n_win && c < a.cand_count[w];
}

// band start of candidate i (slot_of(a, i) holds)
__device__ __forceinline__ void band_begin_one(const StageArgs& a, long long i) {
    CandWork& wk = a.work[i];
    wk.iter = 0;
    wk.retry = 0;
    wk.fresh = 0;
    if (a.prm.band_index == 0) {  // the work slots are reused across stages
        wk.val_band = -1;
        for (int b = 0; b < kMaxBands; ++b) wk.band_evals[b] = 0;
    }
    wk.status = ST_DONE;
    CandState& st = a.cand[i];
    if (!st.active || st.diverged) return;
    wk.lambda = a.prm.step_damping;
    st.band_converged = 0;
    if (st.anchored && a.prm.band > st.anchor_limit) {  // re-anchor at the new band (optimize.cpp:289)
        const Quat koff{a.prm.koffset[0], a.prm.koffset[1], a.prm.koffset[2], a.prm.koffset[3]};
        qstore(st.anchor, q_mul(q_inv(koff), qload(st.g)));
        st.anchor_limit = a.prm.band;
    }
    wk.status = ST_START;
}

// band start of every candidate slot; the started candidates form the first
// iteration's start list (ordered appends, whole warps)
__global__ void band_begin_kernel(StageArgs a, int* start, int* start_count) {
    const long long n = (long long)a.n_win * a.max_cand;
    const long long n_pad = (n + 31) & ~31LL;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_pad;
         i += (long long)gridDim.x * blockDim.x) {
        bool st = false;
        if (i < n) {
            if (!slot_of(a, i)) {
                CandWork& wk = a.work[i];
                wk.iter = 0;
                wk.retry = 0;
                wk.fresh = 0;
                wk.status = ST_DONE;
            } else {
                band_begin_one(a, i);
                st = a.work[i].status == ST_START;
            }
        }
        wappend(st, (int)i, start, start_count);
    }
}

// order-2 evaluation frame of an anchored candidate at global rotation g: the
// window kernel at E(g), or the side kernels at E(g K), whichever is further from
// its gimbal pole (chart_transform)
__device__ __forceinline__ void choose_frame(const Quat& g, const Quat& koff, double* ev, int& side, double* tv) {
    // sin b of g and of g K straight from the matrices; only the chosen frame's angles are computed
    const Quat gk = q_mul(g, koff);
    const double sg = hypot(2 * (g.x * g.z + g.w * g.y), 2 * (g.y * g.z - g.w * g.x));
    const double sk = hypot(2 * (gk.x * gk.z + gk.w * gk.y), 2 * (gk.y * gk.z - gk.w * gk.x));
    const bool use_side = sk > sg;
    const Quat& q = use_side ? gk : g;
    const Euler3 e = q_euler(q);
    ev[0] = e.a, ev[1] = e.b, ev[2] = e.g;
    side = use_side ? 2 : 1;
    frame_trig(q, tv);
}
__device__ __forceinline__ void set_eval_frame(CandWork& wk, const Quat& g, const Quat& koff) {
    choose_frame(g, koff, wk.ev, wk.side, wk.tv);
}

// iteration start of candidate i (chart and re-anchor decision,
// optimize.cpp:292-298): 0 = no step, 1 = evaluate at order 2 first, 2 = step on
// the order-2 results of the accepted trial (already at g).  Anchored candidates
// pick the kernel and angles of their order-2 evaluation (chart_transform).
__device__ __forceinline__ int iter_begin_one(const StageArgs& a, CandWork& wk, CandState& st) {
    if (wk.status != ST_START) return 0;
    if (wk.iter >= a.prm.newton_max_iter) {
        wk.status = ST_DONE;
        return 0;
    }
    const Quat g = qload(st.g);
    const Quat koff{a.prm.koffset[0], a.prm.koffset[1], a.prm.koffset[2], a.prm.koffset[3]};
    const bool was_anchored = st.anchored != 0;
    // an unanchored candidate that just accepted its trial sits at the trial's
    // global angles (g = h_try exactly: the anchor is the identity)
    Quat h = g;
    Euler3 e;
    if (wk.fresh && !was_anchored) {
        e.a = wk.et[0], e.b = wk.et[1], e.g = wk.et[2];
    } else {
        h = q_mul(g, q_inv(qload(st.anchor)));
        e = q_euler(h);
    }
    bool reanchored = false;
    if (e.b < 0.05 || e.b > kPiD - 0.05) {
        qstore(st.anchor, q_mul(q_inv(koff), g));
        st.anchor_limit = a.prm.band;
        st.anchored = 1;
        reanchored = true;
        h = koff;
        e = q_euler(koff);
    }
    wk.e[0] = e.a, wk.e[1] = e.b, wk.e[2] = e.g;
    if (st.anchored) frame_trig(h, wk.te);  // the chart side of chart_transform
    wk.status = ST_EVAL2;
    ++wk.iter;
    // the accepted trial's derivatives are in its own frame: the global angles of g
    // (unanchored -- exactly this iteration's chart angles unless the candidate
    // anchors right now, when that frame sits at a pole) or a well-conditioned
    // anchored frame (any chart of g follows by chart_transform)
    if (wk.fresh && (was_anchored || !reanchored)) {
        wk.fresh = 0;
        return 2;
    }
    wk.fresh = 0;
    wk.side = 0;
    if (st.anchored) set_eval_frame(wk, g, koff);
    return 1;
}

__device__ __forceinline__ int iter_begin_one(const StageArgs& a, long long i) {
    return iter_begin_one(a, a.work[i], a.cand[i]);
}

// The Newton kernels are latency-bound dependent FP64 chains over one
// candidate's CandWork (about 580 bytes) and CandState: requesting all of their
// cache lines up front turns the chain's serialized DRAM round trips into one.
#ifndef BMB_PF_LEVEL
#define BMB_PF_LEVEL 1
#endif
__device__ __forceinline__ void prefetch_span(const void* p, size_t bytes) {
    const size_t b = reinterpret_cast<size_t>(p);
    for (size_t o = b & ~size_t(127); o < b + bytes; o += 128) {
        if (BMB_PF_LEVEL == 1) asm volatile("prefetch.global.L1 [%0];" ::"l"(o));
        if (BMB_PF_LEVEL == 2) asm volatile("prefetch.global.L2 [%0];" ::"l"(o));
    }
}
__device__ __forceinline__ void prefetch_cand(const StageArgs& a, long long i) {
    prefetch_span(a.work + i, sizeof(CandWork));
    prefetch_span(a.cand + i, sizeof(CandState));
}

// iteration start of the candidates on the start list (band start, or accepted
// trials of the previous iteration); appends to the order-2 list and the step list
__global__ void iter_begin_kernel(StageArgs a, const int* start, const int* start_count) {
    const int n = *start_count;
    const int n_pad = (n + 31) & ~31;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_pad; q += gridDim.x * blockDim.x) {
        const int i = q < n ? start[q] : -1;
        if (i >= 0) prefetch_cand(a, i);
        const int f = i >= 0 ? iter_begin_one(a, i) : 0;
        wappend(f == 1, i, a.list2, a.counts + CNT_L2);
    }
}

// warps per CTA of the evaluation kernels (K scratch sets per warp in static smem)
#ifndef BMB_EVAL_WARPS1
#define BMB_EVAL_WARPS1 8
#endif
template <int K>
struct EvalShape {
    static constexpr int WARPS = K >= 4 ? 4 : (K == 1 ? BMB_EVAL_WARPS1 : 8);
};

// K jobs of one warp, evaluated as runs of jobs that share their kernels
// (K-way when all K share, else pairs, else one at a time)
template <int ORDER, int K, bool WEDGE, bool SWEEP>
__device__ __forceinline__ void eval_group(const BandTables& T, const EvalJob (&job)[K], WarpScratch* ws) {
    using O = EvalOpts<ORDER, SWEEP>;
    if constexpr (K == 1) {
        warp_eval_k<ORDER, 1, WEDGE, O::PF, O::PIPE>(T, job, ws);
    } else {
        bool same[K];
        same[0] = false;
        bool all = true;
#pragma unroll
        for (int k = 1; k < K; ++k) {
            same[k] = job[k].xi == job[k - 1].xi && job[k].wx == job[k - 1].wx;
            all &= same[k];
        }
        if (all) {
            warp_eval_k<ORDER, K, WEDGE, O::PF, O::PIPE>(T, job, ws);
            return;
        }
#pragma unroll 1
        for (int k = 0; k < K;) {
            if (K > 2 && k + 1 < K && same[k + 1]) {
                const EvalJob two[2] = {job[k], job[k + 1]};
                warp_eval_k<ORDER, 2, WEDGE, O::PF, O::PIPE>(T, two, ws + k);
                k += 2;
            } else {
                const EvalJob one[1] = {job[k]};
                warp_eval_k<ORDER, 1, WEDGE, O::PF, O::PIPE>(T, one, ws + k);
                k += 1;
            }
        }
    }
}

// K listed candidates per warp
// resident CTAs per SM the evaluation kernels are compiled for (register cap):
// measured best 4 at order 2 (80 registers, small spills) and 3 at order 0
#ifndef BMB_EVAL_MINB0
#define BMB_EVAL_MINB0 3
#endif
#ifndef BMB_EVAL_MINB2
#define BMB_EVAL_MINB2 4
#endif
#define BMB_EVAL_MINB(order) ((order) == 2 ? BMB_EVAL_MINB2 : BMB_EVAL_MINB0)
template <int ORDER, int K, bool TRIAL = false>
__global__ void __launch_bounds__(EvalShape<K>::WARPS * 32, BMB_EVAL_MINB(ORDER)) eval_kernel(StageArgs a, const int* list,
                                                                                       const int* count) {
    constexpr int WARPS = EvalShape<K>::WARPS;
    __shared__ WarpScratch wsc[WARPS * K];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = *count;
    const int len = a.T.rows * 32;
    const bool wedge = a.prm.has_wedge != 0;
    if (a.eval_stats && blockIdx.x == 0 && threadIdx.x == 0)
        atomicAdd(a.eval_stats + ((size_t)a.T.L * 2 + (ORDER == 2)) * 2 + (wedge ? 1 : 0), (unsigned long long)n);
    const int q0 = (blockIdx.x * WARPS + warp) * K;
    if (q0 >= n) return;
    EvalJob job[K];
    int idx[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int q = q0 + k < n ? q0 + k : q0;  // tail: repeat the first job, results dropped
        const int i = list[q];
        idx[k] = q0 + k < n ? i : -1;
        const CandWork& wk = a.work[i];
        const int w = i / a.max_cand;
        // order 2 (status EVAL2): chart angles e, or for an anchored candidate the
        // angles ev of g (window kernel) or of g K (side kernels); order 0 (trials,
        // final scores): global angles et on the window kernel
        // (TRIAL: order 2 at the trial point in its frame evt / sidet)
        const int side = ORDER == 2 ? (TRIAL ? wk.sidet : wk.side) : 0;
        job[k].xi = (side == 2 ? a.xi_side : a.xi_win) + (size_t)w * len;
        job[k].wx = !wedge ? nullptr : (side == 2 ? a.T.wedge_side : a.T.wedge);
        const double* e = ORDER == 2 ? (TRIAL ? (side ? wk.evt : wk.et) : (side ? wk.ev : wk.e)) : wk.et;
        job[k].a = e[0], job[k].b = e[1], job[k].g = e[2];
    }
    WarpScratch* ws = wsc + warp * K;
    if (wedge) eval_group<ORDER, K, true, false>(a.T, job, ws);
    else eval_group<ORDER, K, false, false>(a.T, job, ws);
    constexpr int NV = ORDER == 0 ? 1 : 10;
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (idx[k] >= 0 && lane < NV) {
            CandWork& wk = a.work[idx[k]];
            wk.c[lane] = ws[k].res[lane];
            wk.r[lane] = ws[k].res[10 + lane];
        }
}

// 32 / LANES listed candidates per warp, one per LANES-lane slice (warp_eval_sub);
// the scratch sets are sized for the bands the slice width serves
#ifndef BMB_HALF_WARPS
#define BMB_HALF_WARPS 4
#endif
#ifndef BMB_SUB_WARPS_O2
#define BMB_SUB_WARPS_O2 28
#endif
#ifndef BMB_SUB_WARPS_OTHER
#define BMB_SUB_WARPS_OTHER 24
#endif
template <int LANES>
struct SubShape {
    static constexpr int ML = LANES == 8 ? 8 : kMaxL;  // 8-lane jobs serve L <= 8
    using WS = WarpScratchT<ML, LANES == 8 ? 8 : 16>;
};
// CTAs of four warps (measured 2.6% faster than eight: finer tail); resident warps per SM
// by register cap: 28 at order 2 with 16-lane jobs (72 registers: 4.6% faster than 32 warps
// at 64 registers with their spills, 24 warps slower again), 24 with 8-lane jobs and at
// order 0 (85 registers; 8-lane order 2 measured 3% faster than at 64 registers)
#define BMB_SUB_MINB(order, lanes) \
    (((order) == 2 && (lanes) == 16 ? BMB_SUB_WARPS_O2 : BMB_SUB_WARPS_OTHER) / BMB_HALF_WARPS)
template <int ORDER, bool TRIAL, int LANES>
__global__ void __launch_bounds__(BMB_HALF_WARPS * 32, BMB_SUB_MINB(ORDER, LANES)) eval_sub_kernel(StageArgs a, const int* list,
                                                                                         const int* count) {
    constexpr int WARPS = BMB_HALF_WARPS, JOBS = 32 / LANES;
    using WS = typename SubShape<LANES>::WS;
    __shared__ WS wsc[WARPS * JOBS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, h = lane / LANES, l16 = lane & (LANES - 1);
    const int n = *count;
    const int len = a.T.rows * 32;
    const bool wedge = a.prm.has_wedge != 0;
    if (a.eval_stats && blockIdx.x == 0 && threadIdx.x == 0)
        atomicAdd(a.eval_stats + ((size_t)a.T.L * 2 + (ORDER == 2)) * 2 + (wedge ? 1 : 0), (unsigned long long)n);
    const int q0 = (blockIdx.x * WARPS + warp) * JOBS;
    if (q0 >= n) return;
    const bool live = q0 + h < n;
    const int i = list[live ? q0 + h : q0];  // tail: idle slices repeat the first job, results dropped
    EvalJob job;
    {
        const CandWork& wk = a.work[i];
        const int w = i / a.max_cand;
        const int side = ORDER == 2 ? (TRIAL ? wk.sidet : wk.side) : 0;
        job.xi = (side == 2 ? a.xi_side : a.xi_win) + (size_t)w * len;
        job.wx = !wedge ? nullptr : (side == 2 ? a.T.wedge_side : a.T.wedge);
        const double* e = ORDER == 2 ? (TRIAL ? (side ? wk.evt : wk.et) : (side ? wk.ev : wk.e)) : wk.et;
        job.a = e[0], job.b = e[1], job.g = e[2];
    }
    WS* ws = wsc + warp * JOBS + h;
    using O = EvalOpts<ORDER, false>;
    if (wedge) warp_eval_sub<ORDER, true, O::PF, LANES>(a.T, job, ws);
    else warp_eval_sub<ORDER, false, O::PF, LANES>(a.T, job, ws);
    constexpr int NV = ORDER == 0 ? 1 : 10;
    for (int v = l16; v < NV; v += LANES)
        if (live) {
            CandWork& wk = a.work[i];
            wk.c[v] = ws->res[v];
            wk.r[v] = ws->res[10 + v];
        }
}

// Newton step of an order-2 evaluated candidate; true: a trial is due (made here
// unless the caller makes it: one inlined copy of make_trial per kernel)
template <bool MAKE = true>
__device__ __forceinline__ bool step_one(const StageArgs& a, CandWork& wk, CandState& st) {
    Derivs f;
    objective(wk.c, wk.r, a.prm.has_wedge != 0, 2, f);
    if (wk.side) chart_transform(f, wk.te, wk.tv);  // anchored: derivatives in the chart angles
    wk.val = f.v;  // the objective at g (any chart: the same function value)
    wk.val_band = a.prm.band_index;
    ++st.evals;
    ++wk.band_evals[a.prm.band_index];
    wk.f[0] = f.v;
    for (int k = 0; k < 3; ++k) wk.f[1 + k] = f.g[k];
    for (int k = 0; k < 9; ++k) wk.f[4 + k] = f.h[k];
    const double scale = fmax(fabs(f.v), 1e-300);
    const double gnorm = sqrt(f.g[0] * f.g[0] + f.g[1] * f.g[1] + f.g[2] * f.g[2]);
    if (f.v > st.best_score) {
        st.best_score = f.v;
        for (int k = 0; k < 4; ++k) st.best_g[k] = st.g[k];
    }
    if (gnorm <= a.prm.grad_tol * scale) {
        st.band_converged = 1;
        wk.status = ST_DONE;
        return false;
    }
    wk.lam = wk.lambda;
    wk.retry = 0;
    if (MAKE) make_trial(wk, st, Quat{a.prm.koffset[0], a.prm.koffset[1], a.prm.koffset[2], a.prm.koffset[3]});
    wk.status = ST_EVAL0;
    return true;
}

// Newton step of every order-2 evaluated candidate; appends trials to list_out
// resident CTAs per SM the thread-per-candidate Newton kernels are compiled for
// (0: no register cap; their FP64 chains are latency-bound)
#ifndef BMB_NEWTON_MINB
#define BMB_NEWTON_MINB 0
#endif
#if BMB_NEWTON_MINB > 0
#define BMB_NEWTON_BOUNDS __launch_bounds__(BMB_NEWTON_BLOCK_SIZE, BMB_NEWTON_MINB)
#else
#define BMB_NEWTON_BOUNDS
#endif
#ifndef BMB_NEWTON_PAD_BYTES
#define BMB_NEWTON_PAD_BYTES 0  // occupancy experiments: extra dynamic shared memory per CTA
#endif
#ifndef BMB_NEWTON_BLOCK_SIZE
#define BMB_NEWTON_BLOCK_SIZE 32
#endif
// A warp's candidates staged in shared memory for the Newton kernels: the
// thread-per-candidate chains read and update most of CandWork / CandState field
// by field, and every such access was a dependent global round trip (ncu: 78% of
// the stalls on long scoreboards, 13% issue).  The warp copies its 32 records in
// with coalesced, independent 8-byte loads (one memory latency for all of them),
// runs the chain on the shared copies and writes the records back.  Strides of
// an odd number of 8-byte words keep the per-lane records on distinct banks.
// CandWork in 16-byte chunks at a stride of an odd number of chunks, CandState in
// 8-byte words at an odd stride: the lanes' records fall on different banks.
constexpr int kWorkChunks = (int)(sizeof(CandWork) / 16), kCandWords = (int)(sizeof(CandState) / 8);
constexpr int kWorkStride = (kWorkChunks | 1) * 2, kCandStride = kCandWords | 1;  // in 8-byte words
static_assert(sizeof(CandWork) % 16 == 0 && sizeof(CandState) % 8 == 0, "record sizes the copies assume");
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
                 : "memory");
}
struct __align__(16) NewtonStage {
    unsigned long long work[32 * kWorkStride];
    unsigned long long cand[32 * kCandStride];
};
// the warp's 32 * kWorkChunks chunks (and 32 * kCandWords words) dealt round-robin to
// the lanes: every copy instruction moves 512 (256) contiguous-by-record bytes
__device__ __forceinline__ void stage_in(const StageArgs& a, int i, NewtonStage& sm) {
    const int lane = threadIdx.x & 31;
#pragma unroll 5
    for (int j = 0; j < kWorkChunks; ++j) {
        const int f = lane + 32 * j, c = f / kWorkChunks, k = f - c * kWorkChunks;
        const int ic = __shfl_sync(0xffffffffu, i, c);
        if (ic >= 0)
            cp_async16(sm.work + c * kWorkStride + 2 * k, reinterpret_cast<const uint4*>(a.work + ic) + k);
    }
#pragma unroll
    for (int j = 0; j < kCandWords; ++j) {
        const int f = lane + 32 * j, c = f / kCandWords, k = f - c * kCandWords;
        const int ic = __shfl_sync(0xffffffffu, i, c);
        if (ic >= 0)
            cp_async8(sm.cand + c * kCandStride + k, reinterpret_cast<const unsigned long long*>(a.cand + ic) + k);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
}
// the raw derivatives c / r are inputs of the Newton kernels only (the evaluation kernels
// write them): their chunks are not written back
constexpr int kRawChunk0 = (int)(offsetof(CandWork, c) / 16);
constexpr int kRawChunk1 = (int)((offsetof(CandWork, r) + sizeof(double) * 10) / 16);
static_assert(offsetof(CandWork, c) % 16 == 0 && (offsetof(CandWork, r) + sizeof(double) * 10) % 16 == 0 &&
                  offsetof(CandWork, r) == offsetof(CandWork, c) + sizeof(double) * 10,
              "c and r form one 16-byte aligned span of CandWork");
__device__ __forceinline__ void stage_out(const StageArgs& a, int i, const NewtonStage& sm) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    constexpr int kBack = kWorkChunks - (kRawChunk1 - kRawChunk0);  // chunks written back per record
#pragma unroll 5
    for (int j = 0; j < kBack; ++j) {
        const int f = lane + 32 * j, c = f / kBack, kk = f - c * kBack;
        const int k = kk < kRawChunk0 ? kk : kk + (kRawChunk1 - kRawChunk0);
        const int ic = __shfl_sync(0xffffffffu, i, c);
        if (ic >= 0)
            reinterpret_cast<uint4*>(a.work + ic)[k] = *reinterpret_cast<const uint4*>(sm.work + c * kWorkStride + 2 * k);
    }
#pragma unroll
    for (int j = 0; j < kCandWords; ++j) {
        const int f = lane + 32 * j, c = f / kCandWords, k = f - c * kCandWords;
        const int ic = __shfl_sync(0xffffffffu, i, c);
        if (ic >= 0) reinterpret_cast<unsigned long long*>(a.cand + ic)[k] = sm.cand[c * kCandStride + k];
    }
    __syncwarp();
}

__global__ void BMB_NEWTON_BOUNDS step_kernel(StageArgs a, const int* list_in, const int* count_in, int* list_out, int* count_out) {
    extern __shared__ __align__(16) unsigned char newton_smem[];
    NewtonStage& sm = reinterpret_cast<NewtonStage*>(newton_smem)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const int n = *count_in;
    const int n_pad = (n + 31) & ~31;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_pad; q += gridDim.x * blockDim.x) {
        const int i = q < n ? list_in[q] : -1;
        stage_in(a, i, sm);
        CandWork& wk = *reinterpret_cast<CandWork*>(sm.work + lane * kWorkStride);
        CandState& st = *reinterpret_cast<CandState*>(sm.cand + lane * kCandStride);
        const bool t = i >= 0 && step_one(a, wk, st);
        stage_out(a, i, sm);
        wappend(t, i, list_out, count_out);
    }
}

// acceptance test of a trial; true: it failed with retries left (re-queue after
// the caller makes the damped trial)
__device__ __forceinline__ bool accept_one(const StageArgs& a, CandWork& wk, CandState& st) {
    Derivs t;
    objective(wk.c, wk.r, a.prm.has_wedge != 0, 0, t);  // the value (the trial ran at order 2)
    ++st.evals;
    ++wk.band_evals[a.prm.band_index];
    const double scale = fmax(fabs(wk.f[0]), 1e-300);
    // tolerant acceptance (optimize.cpp:330-341)
    if (t.v > wk.f[0] - a.prm.accept_tol * scale) {
        qstore(st.g, q_mul(qload(wk.gt), qload(st.anchor)));
        wk.val = t.v;  // the trial point is the new g
        wk.val_band = a.prm.band_index;
        wk.lambda = fmax(wk.lam / 10.0, 1e-12);
        // the trial's order-2 results are the next iteration's evaluation at g
        wk.ev[0] = wk.evt[0], wk.ev[1] = wk.evt[1], wk.ev[2] = wk.evt[2];
        for (int k = 0; k < 4; ++k) wk.tv[k] = wk.tvt[k];
        wk.side = wk.sidet;
        wk.fresh = 1;
        if (t.v > st.best_score) {
            st.best_score = t.v;
            for (int k = 0; k < 4; ++k) st.best_g[k] = st.g[k];
        }
        wk.status = ST_START;
        return false;
    }
    ++wk.retry;
    wk.lam *= 10.0;
    if (wk.retry == 3) {  // three damped retries failed to ascend
        st.diverged = 1;
        wk.status = ST_DONE;
        return false;
    }
    return true;
}

// One Newton round of every pending trial: the acceptance test; an accepted
// trial starts the candidate's next iteration right away (iter_begin_one) and,
// with the trial's own order-2 results, takes its Newton step (step_one) -- the
// new trial joins trial_out; a candidate whose iteration needs a fresh order-2
// evaluation (it just anchored) joins fresh_out; a rejected trial with retries
// left is re-queued with its damped retry.  The per-candidate sequence is the
// reference's (optimize.cpp:291-346); only the interleaving across candidates
// differs from a lock-step iteration.
__global__ void BMB_NEWTON_BOUNDS advance_kernel(StageArgs a, const int* list_in, const int* count_in, int* trial_out, int* trial_count,
                               int* fresh_out, int* fresh_count) {
    extern __shared__ __align__(16) unsigned char newton_smem[];
    NewtonStage& sm = reinterpret_cast<NewtonStage*>(newton_smem)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const int n = *count_in;
    const int n_pad = (n + 31) & ~31;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_pad; q += gridDim.x * blockDim.x) {
        const int i = q < n ? list_in[q] : -1;
        bool trial = false, fresh = false;
        stage_in(a, i, sm);
        if (i >= 0) {
            CandWork& wk = *reinterpret_cast<CandWork*>(sm.work + lane * kWorkStride);
            CandState& st = *reinterpret_cast<CandState*>(sm.cand + lane * kCandStride);
            if (accept_one(a, wk, st)) {
                trial = true;  // damped retry
            } else if (wk.status == ST_START) {
                const int f = iter_begin_one(a, wk, st);
                if (f == 2) trial = step_one<false>(a, wk, st);
                else fresh = f == 1;
            }
            if (trial)
                make_trial(wk, st, Quat{a.prm.koffset[0], a.prm.koffset[1], a.prm.koffset[2], a.prm.koffset[3]});
        }
        stage_out(a, i, sm);
        wappend(trial, i, trial_out, trial_count);
        wappend(fresh, i, fresh_out, fresh_count);
    }
}

// final unanchored score of candidate i at the top band: true if it is scored
__device__ __forceinline__ bool final_prep_one(const StageArgs& a, long long i) {
    CandWork& wk = a.work[i];
    wk.status = ST_DONE;
    if (!a.cand[i].active) return false;
    CandState& st = a.cand[i];
    // the final score is Objective::eval at g at this band (optimize.cpp:349-352): a
    // candidate whose last evaluation at g ran at this band already has that value
    // (the evaluation is still counted, as in the reference)
    if (!st.diverged && wk.val_band == a.prm.band_index) {
        st.score = wk.val;
        ++st.evals;
        ++wk.band_evals[a.prm.band_index];
        return false;
    }
    const Euler3 e = q_euler(qload(st.diverged ? st.best_g : st.g));
    wk.et[0] = e.a, wk.et[1] = e.b, wk.et[2] = e.g;
    wk.status = ST_FINAL;
    return true;
}

__device__ __forceinline__ void final_score_one(const StageArgs& a, long long i) {
    CandWork& wk = a.work[i];
    Derivs t;
    objective(wk.c, wk.r, a.prm.has_wedge != 0, 0, t);
    a.cand[i].score = t.v;
    ++a.cand[i].evals;
    ++wk.band_evals[a.prm.band_index];
    wk.status = ST_DONE;
}

__global__ void final_prep_kernel(StageArgs a) {
    const long long n = (long long)a.n_win * a.max_cand;
    const long long n_pad = (n + 31) & ~31LL;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_pad;
         i += (long long)gridDim.x * blockDim.x) {
        bool f = false;
        if (i < n) {
            if (!slot_of(a, i)) a.work[i].status = ST_DONE;
            else f = final_prep_one(a, i);
        }
        wappend(f, (int)i, a.list2, a.counts + CNT_L2);
    }
}

__global__ void final_score_kernel(StageArgs a) {
    const int n = a.counts[CNT_L2];
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const int i = a.list2[q];
        prefetch_cand(a, i);
        final_score_one(a, i);
    }
}

// prune_after_band (optimize.cpp:391-403): after the first band every candidate
// has its unanchored band-0 score; each window keeps its best (first on ties) and
// restarts it as a fresh refine() from that result for the remaining bands
__device__ void prune_window(const StageArgs& a, int w) {
    const int nc = a.cand_count[w];
    CandState* cs = a.cand + (size_t)w * a.max_cand;
    int best = -1;
    for (int c = 0; c < nc; ++c)
        if (cs[c].active && (best < 0 || cs[c].score > cs[best].score)) best = c;
    for (int c = 0; c < nc; ++c)
        if (c != best) cs[c].active = 0;
    if (best < 0) return;
    CandState& st = cs[best];
    const double* q = st.diverged ? st.best_g : st.g;
    const double g0 = q[0], g1 = q[1], g2 = q[2], g3 = q[3];
    st.g[0] = st.best_g[0] = g0;
    st.g[1] = st.best_g[1] = g1;
    st.g[2] = st.best_g[2] = g2;
    st.g[3] = st.best_g[3] = g3;
    st.anchor[0] = 1.0;
    st.anchor[1] = st.anchor[2] = st.anchor[3] = 0.0;
    st.anchored = 0;
    st.anchor_limit = -1;
    st.diverged = 0;
    st.band_converged = 0;
    a.work[(size_t)w * a.max_cand + best].val_band = -1;
    st.best_score = -DBL_MAX * 2.0;  // -inf
}

__global__ void prune_kernel(StageArgs a) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w < a.n_win) prune_window(a, w);
}

__global__ void window_reduce_kernel(ReduceArgs a) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= a.n_win) return;
    const int nc = a.cand_count[w];
    const CandState* cs = a.cand + (size_t)w * a.max_cand;
    WindowOutcome o;
    o.particle = a.win_particle[w];
    o.shift[0] = a.win_shift[3 * w];
    o.shift[1] = a.win_shift[3 * w + 1];
    o.shift[2] = a.win_shift[3 * w + 2];
    o.n_cand = nc + (nc > 0 ? a.extra_candidates : 0);
    o.sub_norm = a.sub_norm[w];
    o.valid = (nc > 0 && o.sub_norm > 0.0) ? 1 : 0;
    o.evals = a.grid_evals;
    for (int b = 0; b < kMaxBands; ++b) o.band_evals[b] = b == 0 ? a.grid_evals : 0;
    int best = -1;
    double bs = 0.0, ba = 0.0;
    for (int c = 0; c < nc; ++c) {
        const CandState& st = cs[c];
        o.evals += st.evals;
        const CandWork& wk = a.work[(size_t)w * a.max_cand + c];
        for (int b = 0; b < kMaxBands; ++b) o.band_evals[b] += wk.band_evals[b];
        if (!st.active) continue;  // pruned after the first band
        const double ang = q_angle(qload(st.diverged ? st.best_g : st.g));
        // search_one_shift tie rule (optimize.cpp:405-412)
        if (best < 0 || st.score > bs || (st.score == bs && ang < ba)) {
            best = c;
            bs = st.score;
            ba = ang;
        }
    }
    o.best_cand = best;
    if (best >= 0) {
        const CandState& st = cs[best];
        const double* q = st.diverged ? st.best_g : st.g;
        for (int i = 0; i < 4; ++i) o.quat[i] = q[i];
        o.raw_score = st.score;
        o.converged = (!st.diverged && st.band_converged) ? 1 : 0;
        o.norm_score = o.valid ? st.score / (a.t_norm * o.sub_norm) : -DBL_MAX;
    } else {
        o.quat[0] = 1.0, o.quat[1] = o.quat[2] = o.quat[3] = 0.0;
        o.raw_score = 0.0;
        o.converged = 0;
        o.norm_score = -DBL_MAX;
    }
    a.out[w] = o;
}

// ---------------------------------------------------------------- objective probe
// bm_objective_eval: the refinement's evaluation of Objective::eval
// (src/optimize.cpp:102-131) at given chart angles and anchors, through the same
// frame choice, evaluation kernels and chart transform as the Newton loop
__global__ void objective_setup_kernel(StageArgs a, const double* euler, const double* anchors, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) a.counts[CNT_L2] = n;
    if (i >= n) return;
    CandState& st = a.cand[i];
    CandWork& wk = a.work[i];
    const Quat koff{a.prm.koffset[0], a.prm.koffset[1], a.prm.koffset[2], a.prm.koffset[3]};
    const double* e = euler + 3 * i;
    const Quat anchor = anchors ? qload(anchors + 4 * i) : Quat{1.0, 0.0, 0.0, 0.0};
    const Quat g = anchors ? q_mul(q_from_euler(e[0], e[1], e[2]), anchor) : q_from_euler(e[0], e[1], e[2]);
    qstore(st.g, g);
    qstore(st.anchor, anchor);
    st.anchored = anchors ? 1 : 0;
    wk.e[0] = e[0], wk.e[1] = e[1], wk.e[2] = e[2];
    frame_trig(q_from_euler(e[0], e[1], e[2]), wk.te);
    wk.side = 0;
    if (anchors) set_eval_frame(wk, g, koff);
    // order 0: the value at the global rotation on the window kernel (make_trial)
    const Euler3 eg = q_euler(g);
    wk.et[0] = anchors ? eg.a : e[0];
    wk.et[1] = anchors ? eg.b : e[1];
    wk.et[2] = anchors ? eg.g : e[2];
    a.list2[i] = i;
}

__global__ void objective_finalize_kernel(StageArgs a, int n, int order, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    CandWork& wk = a.work[i];
    Derivs f;
    objective(wk.c, wk.r, a.prm.has_wedge != 0, order, f);
    if (order == 2 && wk.side) chart_transform(f, wk.te, wk.tv);
    double* o = out + 13 * (size_t)i;
    o[0] = f.v;
    for (int k = 0; k < 3; ++k) o[1 + k] = order == 2 ? f.g[k] : 0.0;
    for (int k = 0; k < 9; ++k) o[4 + k] = order == 2 ? f.h[k] : 0.0;
}

// ---------------------------------------------------------------- sweep
template <int ORDER, int K>
__global__ void __launch_bounds__(EvalShape<K>::WARPS * 32) eval_sweep_kernel(EvalArgs a) {
    constexpr int WARPS = EvalShape<K>::WARPS;
    __shared__ WarpScratch wsc[WARPS * K];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpScratch* ws = wsc + warp * K;
    const long long total = (long long)a.n_xi * a.n_rot;
    for (long long u0 = ((long long)blockIdx.x * WARPS + warp) * K; u0 < total;
         u0 += (long long)gridDim.x * WARPS * K) {
        EvalJob job[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const long long u = u0 + k < total ? u0 + k : u0;
            const int p = (int)(u / a.n_rot), gi = (int)(u % a.n_rot);
            job[k].xi = a.xi + (size_t)p * a.T.rows * 32;
            job[k].wx = nullptr;
            const double* e = a.euler + 3 * gi;
            job[k].a = e[0], job[k].b = e[1], job[k].g = e[2];
        }
        eval_group<ORDER, K, false, true>(a.T, job, ws);
        if (lane < K && u0 + lane < total) {
            const double* r = ws[lane].res;
            double* o = a.out + 4 * (u0 + lane);
            o[0] = r[0];
            o[1] = ORDER >= 1 ? r[1] : 0.0;
            o[2] = ORDER >= 1 ? r[2] : 0.0;
            o[3] = ORDER >= 1 ? r[3] : 0.0;
        }
        __syncwarp();
    }
}

__global__ void build_xi_kernel(XiArgs a) {
    const float* f = a.f + (long long)blockIdx.y * a.ldf;
    const float* t = a.t + (long long)blockIdx.y * a.ldt;
    float4* out = a.out + (size_t)blockIdx.y * a.T.rows * 32;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < a.T.rows * 32; e += gridDim.x * blockDim.x)
        out[e] = xi_entry(a.T, a.row_group, f, t, a.block_off, a.radial_count, e >> 5, e & 31);
}

// one CTA per coefficient set: its rows (and the template's) staged in shared
// memory, entries computed from there
__global__ void __launch_bounds__(256) build_xi_staged_kernel(XiArgs a) {
    extern __shared__ __align__(16) float xs[];
    float* fs = xs;
    float* ts = xs + ((a.nf + 3) & ~3);
    const float* f = a.f + (long long)blockIdx.x * a.ldf;
    const float* t = a.t + (long long)blockIdx.x * a.ldt;
    for (int i = threadIdx.x; i < a.nf; i += blockDim.x) {
        fs[i] = f[i];
        ts[i] = t[i];
    }
    __syncthreads();
    float4* out = a.out + (size_t)blockIdx.x * a.T.rows * 32;
    for (int e = threadIdx.x; e < a.T.rows * 32; e += blockDim.x)
        out[e] = xi_entry(a.T, a.row_group, fs, ts, a.block_off, a.radial_count, e >> 5, e & 31);
}

// xi_l[m,m'] against two templates (t and the side template u) at once: the
// f loads are shared and the sign/conjugation of negative orders is applied to
// the four raw k-sums after the loop:
//   f_m = s_m (fr + i c_m fi), t_m' = s_m' (tr + i c_m' ti)  (s = (-1)^|m| for m < 0, c = -1 for m < 0)
//   conj(f) t = s_m s_m' [(S_rr + c_m c_m' S_ii) + i (c_m' S_ri - c_m S_ir)]
__device__ __forceinline__ void xi_value2(int l, int m, int mp, const float* f, const float* t, const float* u,
                                          const int* block_off, const int* radial_count, float2& xt, float2& xu) {
    const int nk = radial_count[l], base = block_off[l], w = 2 * l + 1;
    const int am = abs(m), amp = abs(mp);
    const int fo = base + (am ? 2 * am - 1 : 0), to = base + (amp ? 2 * amp - 1 : 0);
    float rr = 0.f, ii = 0.f, ri = 0.f, ir = 0.f, urr = 0.f, uii = 0.f, uri = 0.f, uir = 0.f;
    for (int k = 0; k < nk; ++k) {
        const float fr = f[fo + k * w], fi = am ? f[fo + 1 + k * w] : 0.f;
        const float tr = t[to + k * w], ti = amp ? t[to + 1 + k * w] : 0.f;
        const float vr = u[to + k * w], vi = amp ? u[to + 1 + k * w] : 0.f;
        rr = fmaf(fr, tr, rr);
        ii = fmaf(fi, ti, ii);
        ri = fmaf(fr, ti, ri);
        ir = fmaf(fi, tr, ir);
        urr = fmaf(fr, vr, urr);
        uii = fmaf(fi, vi, uii);
        uri = fmaf(fr, vi, uri);
        uir = fmaf(fi, vr, uir);
    }
    const float sg = ((m < 0 && (am & 1)) ? -1.f : 1.f) * ((mp < 0 && (amp & 1)) ? -1.f : 1.f);
    const float cm = m < 0 ? -1.f : 1.f, cp = mp < 0 ? -1.f : 1.f;
    xt = make_float2(sg * fmaf(cm * cp, ii, rr), sg * (cp * ri - cm * ir));
    xu = make_float2(sg * fmaf(cm * cp, uii, urr), sg * (cp * uri - cm * uir));
}

// the same on staged complex pairs: fp[pair] = (Re, Im) of f and tu[pair] = (Re t,
// Im t, Re u, Im u), a row (l, k) holding its l + 1 orders (order 0 with a zero
// imaginary part), so one 8-byte and one 16-byte load feed the eight FMAs of a k
// step.  Same products and order as xi_value2.
__device__ __forceinline__ void xi_value2s(int l, int m, int mp, const float2* fp, const float4* tu, int nk,
                                           float2& xt, float2& xu) {
    const int am = abs(m), amp = abs(mp), st = l + 1;
    const float2* pf = fp + am;
    const float4* pt = tu + amp;
    float rr = 0.f, ii = 0.f, ri = 0.f, ir = 0.f, urr = 0.f, uii = 0.f, uri = 0.f, uir = 0.f;
#pragma unroll 4
    for (int k = 0; k < nk; ++k) {
        const float2 fv = pf[k * st];
        const float4 tv = pt[k * st];
        rr = fmaf(fv.x, tv.x, rr);
        ii = fmaf(fv.y, tv.y, ii);
        ri = fmaf(fv.x, tv.y, ri);
        ir = fmaf(fv.y, tv.x, ir);
        urr = fmaf(fv.x, tv.z, urr);
        uii = fmaf(fv.y, tv.w, uii);
        uri = fmaf(fv.x, tv.w, uri);
        uir = fmaf(fv.y, tv.z, uir);
    }
    const float sg = ((m < 0 && (am & 1)) ? -1.f : 1.f) * ((mp < 0 && (amp & 1)) ? -1.f : 1.f);
    const float cm = m < 0 ? -1.f : 1.f, cp = mp < 0 ? -1.f : 1.f;
    xt = make_float2(sg * fmaf(cm * cp, ii, rr), sg * (cp * ri - cm * ir));
    xu = make_float2(sg * fmaf(cm * cp, uii, urr), sg * (cp * uri - cm * uir));
}

// window and side kernels of one coefficient set per CTA, written to out and out2.
// STAGED: f, t and the side template staged in shared memory as complex pairs
// (a.npairs of them); false: large bases read f and the templates from global memory
template <bool STAGED>
__global__ void __launch_bounds__(256) build_xi_pair_kernel(XiArgs a) {
    extern __shared__ __align__(16) float xs[];
    const float* f = a.f + (long long)blockIdx.x * a.ldf;
    const size_t off = (size_t)blockIdx.x * a.T.rows * 32;
    if constexpr (STAGED) {
        const int np2 = (a.npairs + 1) & ~1;
        float2* fp = reinterpret_cast<float2*>(xs);
        float4* tu = reinterpret_cast<float4*>(xs + 2 * np2);
        int* poff = reinterpret_cast<int*>(tu + np2);  // [L + 1] first pair of degree l
        int* nks = poff + a.T.L + 1;                   // [L + 1] radial count of degree l
        if (threadIdx.x <= a.T.L) {
            int sum = 0;
            for (int l = 0; l < threadIdx.x; ++l) sum += a.radial_count[l] * (l + 1);
            poff[threadIdx.x] = sum;
            nks[threadIdx.x] = a.radial_count[threadIdx.x];
        }
        __syncthreads();
        int l = 0;  // degree of pair p: monotone in p, so the scan resumes where it stopped
        for (int p = threadIdx.x; p < a.npairs; p += blockDim.x) {  // independent loads: one latency for all
            while (l < a.T.L && poff[l + 1] <= p) ++l;
            const int st = l + 1, q = p - poff[l];
            const int k = q / st, am = q - k * st;
            const int src = a.block_off[l] + k * (2 * l + 1) + (am ? 2 * am - 1 : 0);
            fp[p] = make_float2(f[src], am ? f[src + 1] : 0.f);
            tu[p] = make_float4(a.t[src], am ? a.t[src + 1] : 0.f, a.t2[src], am ? a.t2[src + 1] : 0.f);
        }
        __syncthreads();
        for (int e = threadIdx.x; e < a.T.rows * 32; e += blockDim.x) {
            const int2 dsc = a.T.at_desc[e];
            float4 o1 = make_float4(0.f, 0.f, 0.f, 0.f), o2 = o1;
            if (dsc.x & 1) {
                const int l = (dsc.x >> 2) & 63;
                const float2* fl = fp + poff[l];
                const float4* tl = tu + poff[l];
                const int nk = nks[l];
                float2 x, y;
                xi_value2s(l, ((dsc.x >> 8) & 255) - 64, ((dsc.x >> 16) & 255) - 64, fl, tl, nk, x, y);
                o1.x = x.x, o1.y = x.y, o2.x = y.x, o2.y = y.y;
                if (dsc.x & 2) {
                    xi_value2s(l, (dsc.y & 255) - 64, ((dsc.y >> 8) & 255) - 64, fl, tl, nk, x, y);
                    o1.z = x.x, o1.w = x.y, o2.z = y.x, o2.w = y.y;
                }
            }
            a.out[off + e] = o1;
            a.out2[off + e] = o2;
        }
    } else {
        for (int e = threadIdx.x; e < a.T.rows * 32; e += blockDim.x) {
            const int2 dsc = a.T.at_desc[e];
            float4 o1 = make_float4(0.f, 0.f, 0.f, 0.f), o2 = o1;
            if (dsc.x & 1) {
                const int l = (dsc.x >> 2) & 63;
                float2 x, y;
                xi_value2(l, ((dsc.x >> 8) & 255) - 64, ((dsc.x >> 16) & 255) - 64, f, a.t, a.t2, a.block_off,
                          a.radial_count, x, y);
                o1.x = x.x, o1.y = x.y, o2.x = y.x, o2.y = y.y;
                if (dsc.x & 2) {
                    xi_value2(l, (dsc.y & 255) - 64, ((dsc.y >> 8) & 255) - 64, f, a.t, a.t2, a.block_off,
                              a.radial_count, x, y);
                    o1.z = x.x, o1.w = x.y, o2.z = y.x, o2.w = y.y;
                }
            }
            a.out[off + e] = o1;
            a.out2[off + e] = o2;
        }
    }
}

}  // namespace

double eval_flops(int L, int order, bool wedge) {
    const double nxi = (L + 1.0) * (2.0 * L + 1.0) * (2.0 * L + 3.0) / 3.0;
    const double plane = (2.0 * L + 1.0) * (2.0 * L + 1.0);
    const int nd = order + 1;                                  // d, d', d''
    const int nv = order == 0 ? 1 : (order == 1 ? 4 : 10);     // reduced values
    const double per_kernel = 4.0 * nd * nxi + 6.0 * nv * plane;
    return 6.0 * nd * nxi + per_kernel * (wedge ? 2.0 : 1.0);
}

// thread-per-candidate bookkeeping kernels: small CTAs so that a few thousand
// candidates still spread over every SM (these kernels are latency-bound)
constexpr int kNB = BMB_NEWTON_BLOCK_SIZE;
static int thread_grid(long long n) {
    long long b = (n + kNB - 1) / kNB;
    return (int)(b < 1 ? 1 : (b > 16384 ? 16384 : b));
}

void launch_band_begin(const StageArgs& a, int* start, int* start_count, cudaStream_t s) {
    band_begin_kernel<<<thread_grid((long long)a.n_win * a.max_cand), kNB, 0, s>>>(a, start, start_count);
}
void launch_iter_begin(const StageArgs& a, const int* start, const int* start_count, int max_n, cudaStream_t s) {
    iter_begin_kernel<<<thread_grid(max_n), kNB, 0, s>>>(a, start, start_count);
}
// jobs per warp in the refinement: 1 (measured fastest; K-way over runs of
// same-window candidates in the ordered lists is slower at every order):
// BMB_EVAL_K0 / BMB_EVAL_K2 (1, 2, 4) for A/B runs
static int eval_k_for(int order, int /*max_n*/) {
    static const int k0 = [] {
        const char* e = std::getenv("BMB_EVAL_K0");
        return e ? std::atoi(e) : 1;
    }();
    static const int k2 = [] {
        const char* e = std::getenv("BMB_EVAL_K2");
        return e ? std::atoi(e) : 1;
    }();
    return order == 2 ? k2 : k0;
}

template <int ORDER, int K, bool TRIAL = false>
static void launch_eval_k(const StageArgs& a, const int* list, const int* count, int max_n, cudaStream_t s) {
    constexpr int per = K * EvalShape<K>::WARPS;
    eval_kernel<ORDER, K, TRIAL><<<(max_n + per - 1) / per, EvalShape<K>::WARPS * 32, 0, s>>>(a, list, count);
}

// bands evaluated two or four jobs per warp (eval_sub_kernel): BMB_HALF_MAX_L (default: all;
// measured: config 2 2870 -> 3067 subtomograms/s, config 5 (L = 20) 1253 -> 1272
// against full-warp jobs; -1 disables) for A/B runs
static int half_max_l() {
    static const int v = [] {
        const char* e = std::getenv("BMB_HALF_MAX_L");
        return e ? std::atoi(e) : kMaxL;
    }();
    return v;
}
// bands evaluated 8 lanes per job, four jobs per warp: BMB_QUARTER_MAX_L (default
// 8, measured: config 2 3067 -> 3120 subtomograms/s against 16-lane jobs at L = 4, 8,
// and 8-lane jobs at L = 16 were slower (3050); at most 8, the scratch size; -1 disables)
static int quarter_max_l() {
    static const int v = [] {
        const char* e = std::getenv("BMB_QUARTER_MAX_L");
        const int q = e ? std::atoi(e) : 8;
        return q > 8 ? 8 : q;
    }();
    return v;
}
template <int ORDER, bool TRIAL, int LANES>
static void launch_eval_sub_w(const StageArgs& a, const int* list, const int* count, int max_n, cudaStream_t s) {
    constexpr int per = (32 / LANES) * BMB_HALF_WARPS;
    eval_sub_kernel<ORDER, TRIAL, LANES><<<(max_n + per - 1) / per, BMB_HALF_WARPS * 32, 0, s>>>(a, list, count);
}
template <int ORDER, bool TRIAL = false>
static void launch_eval_half(const StageArgs& a, const int* list, const int* count, int max_n, cudaStream_t s) {
    if (a.T.L <= quarter_max_l()) launch_eval_sub_w<ORDER, TRIAL, 8>(a, list, count, max_n, s);
    else launch_eval_sub_w<ORDER, TRIAL, 16>(a, list, count, max_n, s);
}

void launch_eval(const StageArgs& a, int order, const int* list, const int* count, int max_n, cudaStream_t s,
                 bool trial) {
    if (max_n <= 0) return;
    if (a.T.L <= half_max_l()) {
        if (order == 2 && trial) launch_eval_half<2, true>(a, list, count, max_n, s);
        else if (order == 2) launch_eval_half<2>(a, list, count, max_n, s);
        else launch_eval_half<0>(a, list, count, max_n, s);
        return;
    }
    const int k = eval_k_for(order, max_n);
    if (order == 2 && trial) {
        launch_eval_k<2, 1, true>(a, list, count, max_n, s);
    } else if (order == 2) {
        if (k >= 2) launch_eval_k<2, 2>(a, list, count, max_n, s);
        else launch_eval_k<2, 1>(a, list, count, max_n, s);
    } else {
        if (k == 4) launch_eval_k<0, 4>(a, list, count, max_n, s);
        else if (k == 2) launch_eval_k<0, 2>(a, list, count, max_n, s);
        else launch_eval_k<0, 1>(a, list, count, max_n, s);
    }
}
void launch_step(const StageArgs& a, const int* list_in, const int* count_in, int* list_out, int* count_out,
                 int max_n, cudaStream_t s) {
    constexpr int smem = (kNB / 32) * (int)sizeof(NewtonStage) + BMB_NEWTON_PAD_BYTES;
    if (smem > 48 * 1024) ensure_dynamic_smem(step_kernel, smem);
    step_kernel<<<thread_grid(max_n), kNB, smem, s>>>(a, list_in, count_in, list_out, count_out);
}
void launch_advance(const StageArgs& a, const int* list_in, const int* count_in, int* trial_out, int* trial_count,
                    int* fresh_out, int* fresh_count, int max_n, cudaStream_t s) {
    constexpr int smem = (kNB / 32) * (int)sizeof(NewtonStage) + BMB_NEWTON_PAD_BYTES;
    if (smem > 48 * 1024) ensure_dynamic_smem(advance_kernel, smem);
    advance_kernel<<<thread_grid(max_n), kNB, smem, s>>>(a, list_in, count_in, trial_out, trial_count, fresh_out,
                                                         fresh_count);
}
void launch_final_prep(const StageArgs& a, cudaStream_t s) {
    final_prep_kernel<<<thread_grid((long long)a.n_win * a.max_cand), kNB, 0, s>>>(a);
}
void launch_final_score(const StageArgs& a, int max_n, cudaStream_t s) {
    final_score_kernel<<<thread_grid(max_n), kNB, 0, s>>>(a);
}
void launch_prune(const StageArgs& a, cudaStream_t s) {
    prune_kernel<<<(a.n_win + 127) / 128, 128, 0, s>>>(a);
}
void launch_window_reduce(const ReduceArgs& a, cudaStream_t s) {
    window_reduce_kernel<<<(a.n_win + 127) / 128, 128, 0, s>>>(a);
}

int launch_objective_eval(const StageArgs& a, const double* euler, const double* anchors, int n, int order,
                          double* out, cudaStream_t s) {
    if (n <= 0) return 0;
    objective_setup_kernel<<<(n + 127) / 128, 128, 0, s>>>(a, euler, anchors, n);
    launch_eval(a, order == 2 ? 2 : 0, a.list2, a.counts + CNT_L2, n, s);
    objective_finalize_kernel<<<(n + 127) / 128, 128, 0, s>>>(a, n, order, out);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int launch_eval_sweep(const EvalArgs& a, cudaStream_t s) {
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const char* e = std::getenv("BMB_SWEEP_K");
    const int k = e ? std::atoi(e) : 4;
    const int grid = sms * 8;
    if (a.order >= 1) {
        if (k == 1) eval_sweep_kernel<1, 1><<<grid, EvalShape<1>::WARPS * 32, 0, s>>>(a);
        else if (k == 2) eval_sweep_kernel<1, 2><<<grid, EvalShape<2>::WARPS * 32, 0, s>>>(a);
        else eval_sweep_kernel<1, 4><<<grid, EvalShape<4>::WARPS * 32, 0, s>>>(a);
    } else {
        if (k == 1) eval_sweep_kernel<0, 1><<<grid, EvalShape<1>::WARPS * 32, 0, s>>>(a);
        else if (k == 2) eval_sweep_kernel<0, 2><<<grid, EvalShape<2>::WARPS * 32, 0, s>>>(a);
        else eval_sweep_kernel<0, 4><<<grid, EvalShape<4>::WARPS * 32, 0, s>>>(a);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int launch_build_xi(const XiArgs& a, cudaStream_t s) {
    if (a.n <= 0) return 0;
    if (a.t2) {  // window + side kernels in one pass
        // staged complex pairs: 8 B of f and 16 B of (t, u) per pair, + per-degree offsets and counts
        const size_t smem = 24 * (size_t)((a.npairs + 1) & ~1) + 2 * sizeof(int) * (size_t)(a.T.L + 1);
        if (a.ldt != 0 || a.nf <= 0 || !a.out2) return 1;
        if (a.npairs > 0 && a.T.L < 256 && smem <= 200 * 1024) {
            if (ensure_dynamic_smem(build_xi_pair_kernel<true>, (int)smem) != cudaSuccess) return 2;
            build_xi_pair_kernel<true><<<a.n, 256, smem, s>>>(a);
        } else {
            build_xi_pair_kernel<false><<<a.n, 256, 0, s>>>(a);
        }
        return cudaGetLastError() == cudaSuccess ? 0 : 2;
    }
    const size_t smem = sizeof(float) * 2 * (size_t)((a.nf + 3) & ~3);
    if (a.nf > 0 && smem <= 200 * 1024) {
        if (ensure_dynamic_smem(build_xi_staged_kernel, (int)smem) != cudaSuccess) return 2;
        build_xi_staged_kernel<<<a.n, 256, smem, s>>>(a);
        return cudaGetLastError() == cudaSuccess ? 0 : 2;
    }
    dim3 grid((a.T.rows * 32 + 255) / 256, a.n);
    build_xi_kernel<<<grid, 256, 0, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace bmb
