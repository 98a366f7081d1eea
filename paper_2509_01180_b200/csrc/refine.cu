// Rotate-score-gradient evaluation and the device Newton state machine.
//
// Kernel K4+K5 (warp_eval): C(g) = Re sum_l sum_{m,m'} xi_l[m,m'] e^{-i m a}
// d^l_{m,m'}(b) e^{-i m' g} with its Euler gradient and Hessian
// (correlation_derivatives, src/xcorr.cpp:52-105).  One warp per evaluation;
// each lane owns half-plane (m,m') chains and marches the three-term Wigner-d
// recursion over l in registers (src/steer.cpp:101-141), so every d value is
// produced once, used for the correlation AND the wedge-power kernel (same
// angles and band, Objective::eval, src/optimize.cpp:106-130) and never stored.
// The (-m,-m') half follows from the real-volume symmetry
// xi_{-m,-m'} D_{-m,-m'} = conj(xi_{m,m'} D_{m,m'}).  FP32 recursion and lane
// accumulation, FP64 phases / cross-lane reduction / Newton algebra.
//
// Kernel K7 (refine_kernel): one CTA per shift window (persistent), xi of the
// window built in shared memory in the band layout, one warp per candidate
// running the damped-Newton iteration of refine() (src/optimize.cpp:255-357):
// Levenberg lambda, <= 3 retries x10, one-radian trust cap, FullPivLU
// semantics, re-anchoring near the gimbal poles with the composed kernel
// xi~ = xi D(a)^T (xcorr.cpp:149-155) in per-warp scratch, final unanchored
// score at the top band, best-candidate selection per window.
#include <cfloat>

#include "refine.cuh"
#include "rotation.cuh"

namespace bmb {

namespace {

constexpr int kWarps = 8;
constexpr double kPiD = 3.14159265358979323846;

struct WarpScratch {
    float2 ua[kMaxL + 1];
    float2 ug[kMaxL + 1];
    float cp[2 * kMaxL + 3];
    float sp[2 * kMaxL + 3];
};

struct Derivs {
    double v;
    double g[3];
    double h[9];
};

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// Evaluate the correlation (and the wedge-power kernel when WEDGE) at ZYZ
// angles (alpha, beta, gamma), band T.L.  Warp-cooperative; all lanes return
// the same (FP64) results.
template <int ORDER, bool WEDGE>
__device__ __noinline__ void warp_eval(const BandTables& T, const float2* xi, const float2* wx, double alpha,
                          double beta, double gamma, WarpScratch& ws, Derivs& c, Derivs& r) {
    const int lane = threadIdx.x & 31;
    const int L = T.L;
    __syncwarp();
    for (int m = lane; m <= L; m += 32) {
        double s, co;
        sincos(m * alpha, &s, &co);
        ws.ua[m] = make_float2((float)co, (float)-s);
        sincos(m * gamma, &s, &co);
        ws.ug[m] = make_float2((float)co, (float)-s);
    }
    const double ch = cos(0.5 * beta), sh = sin(0.5 * beta);
    for (int j = lane; j <= 2 * L + 2; j += 32) {
        double pc = 1.0, ps = 1.0, bc = ch, bs = sh;  // binary exponentiation
        for (int e = j; e; e >>= 1) {
            if (e & 1) {
                pc *= bc;
                ps *= bs;
            }
            bc *= bc;
            bs *= bs;
        }
        ws.cp[j] = (float)pc;
        ws.sp[j] = (float)ps;
    }
    __syncwarp();
    const float cb = (float)cos(beta), sb = (float)sin(beta);

    float acc[10], accw[10];
#pragma unroll
    for (int i = 0; i < 10; ++i) acc[i] = accw[i] = 0.0f;

    for (int g = 0; g < T.n_groups; ++g) {
        const int item = g * 32 + lane;
        const char2 mm = T.item_mm[item];
        const int m = mm.x, mp = mm.y;
        const int r0 = T.row_off[g];
        const int glen = T.row_off[g + 1] - r0;
        const int be = T.bexp[item];
        const int ea = be & 0xff, ep = be >> 8;
        const float bf = T.bfac[item];
        // closed-form border at l0 (cs_power, steer.cpp:19-31)
        float d = bf * ws.cp[ea] * ws.sp[ep];
        float dp = 0.0f, dpp = 0.0f;
        if (ORDER >= 1) {
            const float tb = ep ? ep * ws.cp[ea + 1] * ws.sp[ep - 1] : 0.0f;
            const float ta = ea ? ea * ws.cp[ea - 1] * ws.sp[ep + 1] : 0.0f;
            dp = 0.5f * bf * (tb - ta);
        }
        if (ORDER >= 2) {
            const float t2b = ep > 1 ? ep * (ep - 1.0f) * ws.cp[ea + 2] * ws.sp[ep - 2] : 0.0f;
            const float t2a = ea > 1 ? ea * (ea - 1.0f) * ws.cp[ea - 2] * ws.sp[ep + 2] : 0.0f;
            dpp = 0.25f * bf * (t2b + t2a - (2.0f * ea * ep + ea + ep) * ws.cp[ea] * ws.sp[ep]);
        }
        float d1 = 0.0f, dp1 = 0.0f, dpp1 = 0.0f;  // degree l-1 (none at the border)
        const float2 x0 = xi[r0 * 32 + lane];
        float2 A0 = make_float2(x0.x * d, x0.y * d), A1 = make_float2(x0.x * dp, x0.y * dp),
               A2 = make_float2(x0.x * dpp, x0.y * dpp);
        float2 W0 = make_float2(0.f, 0.f), W1 = W0, W2 = W0;
        if (WEDGE) {
            const float2 w0 = wx[r0 * 32 + lane];
            W0 = make_float2(w0.x * d, w0.y * d);
            W1 = make_float2(w0.x * dp, w0.y * dp);
            W2 = make_float2(w0.x * dpp, w0.y * dpp);
        }
#pragma unroll 2
        for (int s = 1; s < glen; ++s) {
            const int at = (r0 + s) * 32 + lane;
            const float4 pqr = __ldg(T.PQR + at);
            const float P = pqr.x, Q = pqr.y, R = pqr.z;
            const float t1 = fmaf(P, cb, Q);
            const float dn = t1 * d - R * d1;
            float dpn = 0.0f, dppn = 0.0f;
            if (ORDER >= 1) {
                const float t1p = -P * sb;
                dpn = t1p * d + t1 * dp - R * dp1;
                if (ORDER >= 2) {
                    const float t1pp = -P * cb;
                    dppn = t1pp * d + 2.0f * t1p * dp + t1 * dpp - R * dpp1;
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
            const float2 x = xi[at];
            A0.x = fmaf(x.x, d, A0.x);
            A0.y = fmaf(x.y, d, A0.y);
            if (ORDER >= 1) {
                A1.x = fmaf(x.x, dp, A1.x);
                A1.y = fmaf(x.y, dp, A1.y);
            }
            if (ORDER >= 2) {
                A2.x = fmaf(x.x, dpp, A2.x);
                A2.y = fmaf(x.y, dpp, A2.y);
            }
            if (WEDGE) {
                const float2 w = wx[at];
                W0.x = fmaf(w.x, d, W0.x);
                W0.y = fmaf(w.y, d, W0.y);
                if (ORDER >= 1) {
                    W1.x = fmaf(w.x, dp, W1.x);
                    W1.y = fmaf(w.y, dp, W1.y);
                }
                if (ORDER >= 2) {
                    W2.x = fmaf(w.x, dpp, W2.x);
                    W2.y = fmaf(w.y, dpp, W2.y);
                }
            }
        }
        // phases e^{-i m a} e^{-i m' g}; conj for negative orders
        float2 pa = ws.ua[abs(m)], pg = ws.ug[abs(mp)];
        if (m < 0) pa.y = -pa.y;
        if (mp < 0) pg.y = -pg.y;
        const float2 z = cmul(pa, pg);
        const float wgt = (m == 0 && mp == 0) ? 1.0f : 2.0f;  // half-plane symmetry
        const float fm = (float)m, fmp = (float)mp;
        {
            const float2 v0 = cmul(z, A0);
            acc[0] += wgt * v0.x;
            if (ORDER >= 1) {
                const float2 v1 = cmul(z, A1);
                acc[1] += wgt * fm * v0.y;
                acc[2] += wgt * v1.x;
                acc[3] += wgt * fmp * v0.y;
                if (ORDER >= 2) {
                    const float2 v2 = cmul(z, A2);
                    acc[4] -= wgt * fm * fm * v0.x;
                    acc[5] += wgt * fm * v1.y;
                    acc[6] -= wgt * fm * fmp * v0.x;
                    acc[7] += wgt * v2.x;
                    acc[8] += wgt * fmp * v1.y;
                    acc[9] -= wgt * fmp * fmp * v0.x;
                }
            }
        }
        if (WEDGE) {
            const float2 v0 = cmul(z, W0);
            accw[0] += wgt * v0.x;
            if (ORDER >= 1) {
                const float2 v1 = cmul(z, W1);
                accw[1] += wgt * fm * v0.y;
                accw[2] += wgt * v1.x;
                accw[3] += wgt * fmp * v0.y;
                if (ORDER >= 2) {
                    const float2 v2 = cmul(z, W2);
                    accw[4] -= wgt * fm * fm * v0.x;
                    accw[5] += wgt * fm * v1.y;
                    accw[6] -= wgt * fm * fmp * v0.x;
                    accw[7] += wgt * v2.x;
                    accw[8] += wgt * fmp * v1.y;
                    accw[9] -= wgt * fmp * fmp * v0.x;
                }
            }
        }
    }
    // cross-lane reduction in FP64; hess index map: aa ab ag / ab bb bg / ag bg gg
    c.v = warp_sum(acc[0]);
    if (WEDGE) r.v = warp_sum(accw[0]);
    if (ORDER >= 1) {
        for (int i = 0; i < 3; ++i) c.g[i] = warp_sum(acc[1 + i]);
        if (WEDGE)
            for (int i = 0; i < 3; ++i) r.g[i] = warp_sum(accw[1 + i]);
    }
    if (ORDER >= 2) {
        double h[6], hw[6];
        for (int i = 0; i < 6; ++i) h[i] = warp_sum(acc[4 + i]);
        // acc order: aa, ab, ag, bb, bg, gg
        c.h[0] = h[0], c.h[1] = h[1], c.h[2] = h[2];
        c.h[3] = h[1], c.h[4] = h[3], c.h[5] = h[4];
        c.h[6] = h[2], c.h[7] = h[4], c.h[8] = h[5];
        if (WEDGE) {
            for (int i = 0; i < 6; ++i) hw[i] = warp_sum(accw[4 + i]);
            r.h[0] = hw[0], r.h[1] = hw[1], r.h[2] = hw[2];
            r.h[3] = hw[1], r.h[4] = hw[3], r.h[5] = hw[4];
            r.h[6] = hw[2], r.h[7] = hw[4], r.h[8] = hw[5];
        }
    }
}

// Objective::eval (src/optimize.cpp:106-130): C / sqrt(clamp(1 - rho, 0.02, 2))
__device__ void objective(const Derivs& c, const Derivs& r, bool wedge, int order, Derivs& f) {
    if (!wedge) {
        f = c;
        return;
    }
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

template <int ORDER>
__device__ void eval_objective(const BandTables& T, const float2* xi, const float2* wx,
                               bool wedge, const Euler3& e, WarpScratch& ws, Derivs& f) {
    Derivs c, r;
    if (wedge) warp_eval<ORDER, true>(T, xi, wx, e.a, e.b, e.g, ws, c, r);
    else warp_eval<ORDER, false>(T, xi, wx, e.a, e.b, e.g, ws, c, r);
    objective(c, r, wedge, ORDER, f);
}

// ---------------------------------------------------------------- anchoring
__host__ __device__ __forceinline__ int xi_off(int l) { return l * (2 * l - 1) * (2 * l + 1) / 3; }

// xi~_l = xi_l D^l(a)^T  (xi_compose_right, src/xcorr.cpp:149-155), with
// D^l_{m'n}(a) = e^{-i m' a} d^l_{m'n}(b) e^{-i n g}:
//   xi~_l[m,m'] = e^{-i m' a} sum_n (xi_l[m,n] e^{-i n g}) d^l_{m'n}(b).
// The full-plane d^l(b) comes from the same band tables as the evaluation
// (half-plane chains + d_{-m,-m'} = (-1)^{m-m'} d_{m,m'}); xi is unpacked into a
// dense, phase-folded scratch so the n-sum runs over contiguous rows.  The
// wedge-power kernel is rank one (conj(chi_lm) q_lm' / total), so its
// composition only rotates q: q~_l = D^l(a) q_l  (O(l^2) per degree).
__device__ void compose_kernels(const BandTables& T, const float2* src, const RefineArgs& a,
                                const Quat& anchor, float* scratch, float2* out, float2* out_w,
                                WarpScratch& ws) {
    const int lane = threadIdx.x & 31;
    const int L = T.L;
    const int nxi = xi_off(L + 1);
    float* dtab = scratch;                                                  // nxi floats
    float2* xd = reinterpret_cast<float2*>(scratch + ((nxi + 1) & ~1));    // nxi complex
    float2* qt = xd + nxi;                                                  // (L+1)^2 complex
    const Euler3 e = q_euler(anchor);
    __syncwarp();
    for (int m = lane; m <= L; m += 32) {
        double sn, co;
        sincos(m * e.a, &sn, &co);
        ws.ua[m] = make_float2((float)co, (float)-sn);
        sincos(m * e.g, &sn, &co);
        ws.ug[m] = make_float2((float)co, (float)-sn);
    }
    const double ch = cos(0.5 * e.b), sh = sin(0.5 * e.b);
    for (int j = lane; j <= 2 * L + 2; j += 32) {
        double pc = 1.0, ps = 1.0, bc = ch, bs = sh;
        for (int q = j; q; q >>= 1) {
            if (q & 1) {
                pc *= bc;
                ps *= bs;
            }
            bc *= bc;
            bs *= bs;
        }
        ws.cp[j] = (float)pc;
        ws.sp[j] = (float)ps;
    }
    __syncwarp();
    const float cb = (float)cos(e.b);
    // full-plane d^l_{m,m'}(b_a): half-plane chains + mirror
    for (int g = 0; g < T.n_groups; ++g) {
        const int item = g * 32 + lane;
        const int len = T.item_len[item];
        const int m = T.item_mm[item].x, mp = T.item_mm[item].y;
        const int l0 = max(abs(m), abs(mp));
        const int be = T.bexp[item];
        float d = T.bfac[item] * ws.cp[be & 0xff] * ws.sp[be >> 8], d1 = 0.0f;
        const float mir = ((m - mp) & 1) ? -1.0f : 1.0f;
        const int r0 = T.row_off[g];
        for (int s = 0; s < len; ++s) {
            if (s > 0) {
                const float4 pqr = __ldg(T.PQR + (r0 + s) * 32 + lane);
                const float dn = fmaf(pqr.x, cb, pqr.y) * d - pqr.z * d1;
                d1 = d;
                d = dn;
            }
            const int l = l0 + s, w = 2 * l + 1, o = xi_off(l);
            dtab[o + (m + l) * w + (mp + l)] = d;
            dtab[o + (-m + l) * w + (-mp + l)] = mir * d;
        }
    }
    // dense xi'_l[m,n] = xi_l[m,n] e^{-i n g} (both half-planes)
    for (int at = lane; at < T.rows * 32; at += 32) {
        const int row = at >> 5, j = at & 31;
        const int g = a.row_group[row];
        const int item = g * 32 + j;
        const int s = row - T.row_off[g];
        if (s >= T.item_len[item]) continue;
        const int m = T.item_mm[item].x, mp = T.item_mm[item].y;
        const int l = max(abs(m), abs(mp)) + s, w = 2 * l + 1, o = xi_off(l);
        const float2 x = src[at];
        float2 eg = ws.ug[abs(mp)];
        if (mp < 0) eg.y = -eg.y;
        xd[o + (m + l) * w + (mp + l)] = cmul(x, eg);
        const float sg = ((m + mp) & 1) ? -1.0f : 1.0f;
        const float2 xm = make_float2(sg * x.x, -sg * x.y);  // xi[-m,-m']
        xd[o + (-m + l) * w + (-mp + l)] = cmul(xm, make_float2(eg.x, -eg.y));
    }
    // wedge: q~_l[m'] = e^{-i m' a} sum_n d_{m'n} e^{-i n g} q_ln
    const bool wedge = out_w != nullptr;
    if (wedge) {
        for (int idx = lane; idx < (L + 1) * (L + 1); idx += 32) {
            int l = 0;
            while ((l + 1) * (l + 1) <= idx) ++l;
            const int mp = idx - l * l - l;
            const int w = 2 * l + 1, o = xi_off(l);
            float re = 0.0f, im = 0.0f;
            for (int n = -l; n <= l; ++n) {
                const int an = abs(n);
                double2 qv = a.q_hat[l * (l + 1) / 2 + an];
                if (n < 0) {
                    const double sgn = (an & 1) ? -1.0 : 1.0;
                    qv = make_double2(sgn * qv.x, -sgn * qv.y);
                }
                float2 eg = ws.ug[an];
                if (n < 0) eg.y = -eg.y;
                const float2 t = cmul(make_float2((float)qv.x, (float)qv.y), eg);
                const float dv = dtab[o + (mp + l) * w + (n + l)];
                re = fmaf(dv, t.x, re);
                im = fmaf(dv, t.y, im);
            }
            float2 ea = ws.ua[abs(mp)];
            if (mp < 0) ea.y = -ea.y;
            qt[idx] = cmul(ea, make_float2(re, im));
        }
    }
    __syncwarp();
    // xi~ in band layout
    const float inv_total = (float)(1.0 / a.wp_total);
    for (int at = lane; at < T.rows * 32; at += 32) {
        const int row = at >> 5, j = at & 31;
        const int g = a.row_group[row];
        const int item = g * 32 + j;
        const int s = row - T.row_off[g];
        if (s >= T.item_len[item]) {
            out[at] = make_float2(0.f, 0.f);
            if (wedge) out_w[at] = make_float2(0.f, 0.f);
            continue;
        }
        const int m = T.item_mm[item].x, mp = T.item_mm[item].y;
        const int l = max(abs(m), abs(mp)) + s, w = 2 * l + 1, o = xi_off(l);
        const float2* xr = xd + o + (m + l) * w;
        const float* dr = dtab + o + (mp + l) * w;
        float re = 0.0f, im = 0.0f;
        for (int n = 0; n < w; ++n) {
            const float2 x = xr[n];
            const float dv = dr[n];
            re = fmaf(x.x, dv, re);
            im = fmaf(x.y, dv, im);
        }
        float2 ea = ws.ua[abs(mp)];
        if (mp < 0) ea.y = -ea.y;
        out[at] = cmul(ea, make_float2(re, im));
        if (wedge) {
            const int am = abs(m);
            double2 c = a.chi_hat[l * (l + 1) / 2 + am];
            if (m < 0) {
                const double sgn = (am & 1) ? -1.0 : 1.0;
                c = make_double2(sgn * c.x, -sgn * c.y);
            }
            const float2 qv = qt[l * l + (mp + l)];
            // conj(chi_lm) q~_lm' / total
            const float cr = (float)c.x, ci = (float)-c.y;
            out_w[at] = make_float2((cr * qv.x - ci * qv.y) * inv_total, (cr * qv.y + ci * qv.x) * inv_total);
        }
    }
    __syncwarp();
}

// Damped-Newton band of one candidate (warp-redundant scalar state).
__device__ void newton_band(const RefineArgs& a, const float2* xi_s, CandState& st,
                            WarpScratch& ws, float* scratch) {
    const BandTables& T = a.T;
    const RefineParams& prm = a.prm;
    const bool wedge = prm.has_wedge != 0;
    const int band = prm.band;
    const Quat koff{prm.koffset[0], prm.koffset[1], prm.koffset[2], prm.koffset[3]};
    const int nxi = xi_off(T.L + 1);
    float2* xi_t = reinterpret_cast<float2*>(scratch + ((nxi + 1) & ~1)) + nxi + (T.L + 1) * (T.L + 1);
    float2* w_t = xi_t + (size_t)T.rows * 32;
    Quat g{st.g[0], st.g[1], st.g[2], st.g[3]};
    Quat anchor{st.anchor[0], st.anchor[1], st.anchor[2], st.anchor[3]};
    Quat best_g{st.best_g[0], st.best_g[1], st.best_g[2], st.best_g[3]};
    double best = st.best_score;

    auto reanchor = [&](const Quat& target) {
        anchor = q_mul(q_inv(koff), target);
        st.anchor_limit = band;
        compose_kernels(T, xi_s, a, anchor, scratch, xi_t, wedge ? w_t : nullptr, ws);
        st.anchored = 1;
    };

    double lambda = prm.step_damping;
    st.band_converged = 0;
    if (st.anchored && band > st.anchor_limit) reanchor(g);
    for (int iter = 0; iter < prm.newton_max_iter; ++iter) {
        Quat h = q_mul(g, q_inv(anchor));
        Euler3 e = q_euler(h);
        if (e.b < 0.05 || e.b > kPiD - 0.05) {
            reanchor(g);
            h = koff;
            e = q_euler(h);
        }
        const float2* xs = st.anchored ? xi_t : xi_s;
        const float2* wsrc = st.anchored ? w_t : T.wedge;
        Derivs d;
        eval_objective<2>(T, xs, wsrc, wedge, e, ws, d);
        ++st.evals;
        const double scale = fmax(fabs(d.v), 1e-300);
        const double gnorm = sqrt(d.g[0] * d.g[0] + d.g[1] * d.g[1] + d.g[2] * d.g[2]);
        if (d.v > best) {
            best = d.v;
            best_g = g;
        }
        if (gnorm <= prm.grad_tol * scale) {
            st.band_converged = 1;
            break;
        }
        bool accepted = false;
        double lam = lambda;
        for (int retry = 0; retry < 3 && !accepted; ++retry, lam *= 10.0) {
            double mtx[9];
            for (int i = 0; i < 9; ++i) mtx[i] = d.h[i];
            mtx[0] -= lam;
            mtx[4] -= lam;
            mtx[8] -= lam;
            LU3 lu;
            lu.factor(mtx);
            double p[3];
            if (lu.invertible()) {
                double x[3];
                lu.solve(d.g, x);
                p[0] = -x[0], p[1] = -x[1], p[2] = -x[2];
            } else {
                p[0] = d.g[0] / lam, p[1] = d.g[1] / lam, p[2] = d.g[2] / lam;
            }
            const double pn = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
            if (pn > 1.0) {
                const double sc = 1.0 / pn;
                p[0] *= sc, p[1] *= sc, p[2] *= sc;
            }
            const Quat h_try = q_from_euler(e.a + p[0], e.b + p[1], e.g + p[2]);
            Derivs tr;
            eval_objective<0>(T, xs, wsrc, wedge, q_euler(h_try), ws, tr);
            ++st.evals;
            if (tr.v > d.v - prm.accept_tol * scale) {
                g = q_mul(h_try, anchor);
                lambda = fmax(lam / 10.0, 1e-12);
                accepted = true;
                if (tr.v > best) {
                    best = tr.v;
                    best_g = g;
                }
            }
        }
        if (!accepted) {
            st.diverged = 1;
            break;
        }
    }
    st.g[0] = g.w, st.g[1] = g.x, st.g[2] = g.y, st.g[3] = g.z;
    st.anchor[0] = anchor.w, st.anchor[1] = anchor.x, st.anchor[2] = anchor.y,
    st.anchor[3] = anchor.z;
    st.best_g[0] = best_g.w, st.best_g[1] = best_g.x, st.best_g[2] = best_g.y,
    st.best_g[3] = best_g.z;
    st.best_score = best;
}

// xi_l[m,m'] for the table entry (row, lane) from real-packed f and t
__device__ float2 xi_entry(const BandTables& T, const int* row_group, const float* f,
                           const float* t, const int* block_off, const int* radial_count,
                           int row, int lane) {
    const int g = row_group[row];
    const int item = g * 32 + lane;
    const int s = row - T.row_off[g];
    if (s >= T.item_len[item]) return make_float2(0.f, 0.f);
    const int m = T.item_mm[item].x, mp = T.item_mm[item].y;
    const int l = max(abs(m), abs(mp)) + s;
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

constexpr int kRefineWarps = 16;
constexpr int kMaxBatch = 8;

// Persistent CTAs take batches of `a.batch` windows: their kernels are built in
// shared memory, then the CTA's 16 warps pull (window, candidate) items from
// one pooled queue, so the per-candidate Newton time imbalance averages over
// the whole batch instead of stalling every window at a barrier.
__global__ void __launch_bounds__(kRefineWarps * 32, 1) refine_kernel(RefineArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const BandTables& T = a.T;
    const int xi_len = T.rows * 32;
    float2* xib = reinterpret_cast<float2*>(sm);                               // batch * rows*32
    float* tbuf = reinterpret_cast<float*>(xib + (size_t)a.batch * xi_len);    // rows_band
    float* fbuf = tbuf + a.rows_band;                                          // rows_band
    WarpScratch* wsc = reinterpret_cast<WarpScratch*>(
        (reinterpret_cast<uintptr_t>(fbuf + a.rows_band) + 15) & ~uintptr_t(15));
    __shared__ int s_w0, s_next, s_nitems;
    __shared__ int s_start[kMaxBatch + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpScratch& ws = wsc[warp];
    float* scratch = a.scratch + (size_t)(blockIdx.x * kRefineWarps + warp) * a.scratch_per_warp;

    for (int r = threadIdx.x; r < a.rows_band; r += blockDim.x) tbuf[r] = a.t_hat[r];
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            s_w0 = atomicAdd(a.win_counter, a.batch);
            s_next = 0;
            int acc = 0;
            for (int b = 0; b < a.batch; ++b) {
                s_start[b] = acc;
                const int w = s_w0 + b;
                acc += w < a.n_win ? a.cand_count[w] : 0;
            }
            s_start[a.batch] = acc;
            s_nitems = acc;
        }
        __syncthreads();
        const int w0 = s_w0;
        if (w0 >= a.n_win) break;
        const int nb = min(a.batch, a.n_win - w0);
        // build the batch's kernels (windows without candidates are skipped)
        for (int b = 0; b < nb; ++b) {
            if (s_start[b + 1] == s_start[b]) continue;
            const float* cw = a.coef + (long long)(w0 + b) * a.ldc;
            for (int r = threadIdx.x; r < a.rows_band; r += blockDim.x) fbuf[r] = cw[r];
            __syncthreads();
            float2* xi = xib + (size_t)b * xi_len;
            for (int e = threadIdx.x; e < xi_len; e += blockDim.x)
                xi[e] = xi_entry(T, a.row_group, fbuf, tbuf, a.block_off, a.radial_count, e >> 5, e & 31);
            __syncthreads();
        }
        const int nitems = s_nitems;
        for (;;) {
            int it = 0;
            if (lane == 0) it = atomicAdd(&s_next, 1);
            it = __shfl_sync(0xffffffffu, it, 0);
            if (it >= nitems) break;
            int b = 0;
            while (it >= s_start[b + 1]) ++b;
            const int c = it - s_start[b];
            const float2* xi = xib + (size_t)b * xi_len;
            CandState* cs = a.cand + (size_t)(w0 + b) * a.max_cand;
            CandState st = cs[c];
            if (!st.diverged) newton_band(a, xi, st, ws, scratch);
            if (a.last_band) {
                // final unanchored score at the top band (optimize.cpp:349-352)
                const Quat rq = st.diverged ? Quat{st.best_g[0], st.best_g[1], st.best_g[2], st.best_g[3]}
                                            : Quat{st.g[0], st.g[1], st.g[2], st.g[3]};
                Derivs f;
                eval_objective<0>(T, xi, T.wedge, a.prm.has_wedge != 0, q_euler(rq), ws, f);
                st.score = f.v;
                ++st.evals;
            }
            if (lane == 0) cs[c] = st;
            __syncwarp();
        }
        __syncthreads();
        if (a.last_band && threadIdx.x < nb) {
            const int w = w0 + threadIdx.x;
            const int nc = a.cand_count[w];
            const CandState* cs = a.cand + (size_t)w * a.max_cand;
            WindowOutcome o;
            o.particle = a.win_particle[w];
            o.shift[0] = a.win_shift[3 * w];
            o.shift[1] = a.win_shift[3 * w + 1];
            o.shift[2] = a.win_shift[3 * w + 2];
            o.n_cand = nc;
            o.sub_norm = a.sub_norm[w];
            o.valid = (nc > 0 && o.sub_norm > 0.0) ? 1 : 0;
            o.evals = a.grid_evals;
            int best = -1;
            double bs = 0.0, ba = 0.0;
            for (int c = 0; c < nc; ++c) {
                const CandState& st = cs[c];
                o.evals += st.evals;
                const Quat rq = st.diverged ? Quat{st.best_g[0], st.best_g[1], st.best_g[2], st.best_g[3]}
                                            : Quat{st.g[0], st.g[1], st.g[2], st.g[3]};
                const double ang = q_angle(rq);
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
    }
}

// ---------------------------------------------------------------- sweep
__global__ void __launch_bounds__(kWarps * 32) eval_sweep_kernel(EvalArgs a) {
    __shared__ WarpScratch wsc[kWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long total = (long long)a.n_xi * a.n_rot;
    for (long long u = (long long)blockIdx.x * kWarps + warp; u < total;
         u += (long long)gridDim.x * kWarps) {
        const int p = (int)(u / a.n_rot), gi = (int)(u % a.n_rot);
        const float2* xi = a.xi + (size_t)p * a.T.rows * 32;
        Derivs c, r;
        const double* e = a.euler + 3 * gi;
        if (a.order >= 1) warp_eval<1, false>(a.T, xi, nullptr, e[0], e[1], e[2], wsc[warp], c, r);
        else warp_eval<0, false>(a.T, xi, nullptr, e[0], e[1], e[2], wsc[warp], c, r);
        if (lane == 0) {
            double* o = a.out + 4 * u;
            o[0] = c.v;
            o[1] = a.order >= 1 ? c.g[0] : 0.0;
            o[2] = a.order >= 1 ? c.g[1] : 0.0;
            o[3] = a.order >= 1 ? c.g[2] : 0.0;
        }
    }
}

__global__ void build_xi_kernel(XiArgs a) {
    const float* f = a.f + (long long)blockIdx.y * a.ldf;
    const float* t = a.t + (long long)blockIdx.y * a.ldt;
    float2* out = a.out + (size_t)blockIdx.y * a.T.rows * 32;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < a.T.rows * 32; e += gridDim.x * blockDim.x)
        out[e] = xi_entry(a.T, a.row_group, f, t, a.block_off, a.radial_count, e >> 5, e & 31);
}

}  // namespace

static size_t refine_fixed_bytes(int rows_band) {
    return sizeof(float) * 2 * rows_band + 16 + sizeof(WarpScratch) * kRefineWarps;
}

int refine_batch(const BandTables& T, int rows_band) {
    const size_t budget = 200 * 1024;
    const size_t fixed = refine_fixed_bytes(rows_band);
    const size_t per = sizeof(float2) * (size_t)T.rows * 32;
    int b = fixed + per <= budget ? (int)((budget - fixed) / per) : 1;
    return b < 1 ? 1 : (b > kMaxBatch ? kMaxBatch : b);
}

size_t refine_smem_bytes(const BandTables& T, int rows_band, int batch) {
    return sizeof(float2) * (size_t)T.rows * 32 * batch + refine_fixed_bytes(rows_band);
}

long long refine_scratch_floats(const BandTables& T) {
    // dtab (N_xi floats) + dense xi' (N_xi complex) + q~ ((L+1)^2 complex) + two band-layout kernels
    const long long nxi = xi_off(T.L + 1);
    return (nxi + 2) + 2 * nxi + 2LL * (T.L + 1) * (T.L + 1) + 4LL * T.rows * 32;
}

int refine_warps() { return kRefineWarps; }

int refine_resident_blocks(const BandTables& T, int rows_band, int batch, int device) {
    const size_t smem = refine_smem_bytes(T, rows_band, batch);
    cudaFuncSetAttribute(refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, refine_kernel, kRefineWarps * 32, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return (per_sm > 0 ? per_sm : 1) * sms;
}

int launch_refine(const RefineArgs& a, int blocks, cudaStream_t s) {
    if (a.n_win <= 0) return 0;
    const size_t smem = refine_smem_bytes(a.T, a.rows_band, a.batch);
    cudaFuncSetAttribute(refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    refine_kernel<<<blocks, kRefineWarps * 32, smem, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int launch_eval_sweep(const EvalArgs& a, cudaStream_t s) {
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    eval_sweep_kernel<<<sms * 4, kWarps * 32, 0, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int launch_build_xi(const XiArgs& a, cudaStream_t s) {
    if (a.n <= 0) return 0;
    dim3 grid((a.T.rows * 32 + 255) / 256, a.n);
    build_xi_kernel<<<grid, 256, 0, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace bmb
