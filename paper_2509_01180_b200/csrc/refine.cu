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
__device__ double sqrt_binom_d(int n, int k) {
    double r = 1.0;
    for (int i = 1; i <= k; ++i) r *= (double)(n - k + i) / i;
    return sqrt(r);
}
__device__ double ipow_d(double x, int e) {
    double r = 1.0;
    for (int i = 0; i < e; ++i) r *= x;
    return r;
}
__host__ __device__ __forceinline__ int xi_off(int l) { return l * (2 * l - 1) * (2 * l + 1) / 3; }

// value of a band-layout kernel at (l, m, n), any orders, via the item map and
// the real-volume symmetry
__device__ float2 band_at(const BandTables& T, const float2* src, int l, int m, int n) {
    const int L = T.L;
    const int v = T.item_of[(m + L) * (2 * L + 1) + (n + L)];
    const int i = v >= 0 ? v : -v - 1;
    const int l0 = max(abs(m), abs(n));
    const float2 x = src[(T.row_off[i >> 5] + l - l0) * 32 + (i & 31)];
    if (v >= 0) return x;
    const float sg = ((m + n) & 1) ? -1.0f : 1.0f;
    return make_float2(sg * x.x, -sg * x.y);
}

// xi~_l = xi_l D^l(a)^T  (xi_compose_right, src/xcorr.cpp:149-155) for the
// correlation kernel and the wedge-power kernel, written in band layout.
__device__ void compose_kernels(const BandTables& T, const float2* src, const float2* src_w,
                                const Quat& anchor, float* dtab, float2* out, float2* out_w,
                                WarpScratch& ws) {
    const int lane = threadIdx.x & 31;
    const int L = T.L, W = 2 * L + 1;
    const Euler3 e = q_euler(anchor);
    const double cb = cos(e.b), ch = cos(0.5 * e.b), sh = sin(0.5 * e.b);
    __syncwarp();
    // full-plane little-d^l(beta_a), FP64 chains (steer.cpp:43-144)
    for (int idx = lane; idx < W * W; idx += 32) {
        const int m = idx / W - L, n = idx % W - L;
        const int l0 = max(abs(m), abs(n));
        double fac;
        int pa, pp;
        if (l0 == 0) {
            fac = 1.0, pa = pp = 0;
        } else if (m == l0) {
            fac = (((l0 - n) & 1) ? -1.0 : 1.0) * sqrt_binom_d(2 * l0, l0 + n), pa = l0 + n, pp = l0 - n;
        } else if (m == -l0) {
            fac = sqrt_binom_d(2 * l0, l0 + n), pa = l0 - n, pp = l0 + n;
        } else if (n == l0) {
            fac = sqrt_binom_d(2 * l0, l0 + m), pa = l0 + m, pp = l0 - m;
        } else {
            fac = (((l0 + m) & 1) ? -1.0 : 1.0) * sqrt_binom_d(2 * l0, l0 + m), pa = l0 - m, pp = l0 + m;
        }
        double dcur = fac * (ipow_d(ch, pa) * ipow_d(sh, pp)), dprev = 0.0;
        dtab[xi_off(l0) + (m + l0) * (2 * l0 + 1) + (n + l0)] = (float)dcur;
        for (int l = l0 + 1; l <= L; ++l) {
            double dn;
            if (l == 1) {
                dn = cb;
            } else {
                const double a2 = sqrt(((double)l * l - (double)m * m) * ((double)l * l - (double)n * n));
                const double den = (l - 1.0) * a2;
                const double t1 = (2.0 * l - 1.0) * (l * (l - 1.0) * cb - (double)m * n) / den;
                const bool has2 = abs(m) <= l - 2 && abs(n) <= l - 2;
                const double b2 = has2 ? sqrt(((double)(l - 1) * (l - 1) - (double)m * m) *
                                              ((double)(l - 1) * (l - 1) - (double)n * n))
                                       : 0.0;
                dn = t1 * dcur - (has2 ? l * b2 / den * dprev : 0.0);
            }
            dprev = dcur;
            dcur = dn;
            dtab[xi_off(l) + (m + l) * (2 * l + 1) + (n + l)] = (float)dcur;
        }
    }
    for (int m = lane; m <= L; m += 32) {
        double s, co;
        sincos(m * e.a, &s, &co);
        ws.ua[m] = make_float2((float)co, (float)-s);
        sincos(m * e.g, &s, &co);
        ws.ug[m] = make_float2((float)co, (float)-s);
    }
    __syncwarp();
    for (int item = lane; item < T.n_items; item += 32) {
        const int m = T.item_mm[item].x, mp = T.item_mm[item].y;
        const int l0 = max(abs(m), abs(mp));
        float2 em = ws.ua[abs(mp)];
        if (mp < 0) em.y = -em.y;
        const int base = T.row_off[item >> 5] * 32 + (item & 31);
        for (int l = l0; l <= L; ++l) {
            float2 acc = make_float2(0.f, 0.f), accw = make_float2(0.f, 0.f);
            const float* drow = dtab + xi_off(l) + (mp + l) * (2 * l + 1) + l;  // d^l_{m',n}
            for (int n = -l; n <= l; ++n) {
                float2 eg = ws.ug[abs(n)];
                if (n < 0) eg.y = -eg.y;
                const float d = drow[n];
                const float2 x = cmul(band_at(T, src, l, m, n), eg);
                acc.x = fmaf(x.x, d, acc.x);
                acc.y = fmaf(x.y, d, acc.y);
                if (src_w) {
                    const float2 y = cmul(band_at(T, src_w, l, m, n), eg);
                    accw.x = fmaf(y.x, d, accw.x);
                    accw.y = fmaf(y.y, d, accw.y);
                }
            }
            out[base + (l - l0) * 32] = cmul(em, acc);
            if (src_w) out_w[base + (l - l0) * 32] = cmul(em, accw);
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
    float* dtab = scratch;
    float2* xi_t = reinterpret_cast<float2*>(scratch + ((xi_off(T.L + 1) + 1) & ~1));  // 8-byte aligned
    float2* w_t = xi_t + (size_t)T.rows * 32;
    Quat g{st.g[0], st.g[1], st.g[2], st.g[3]};
    Quat anchor{st.anchor[0], st.anchor[1], st.anchor[2], st.anchor[3]};
    Quat best_g{st.best_g[0], st.best_g[1], st.best_g[2], st.best_g[3]};
    double best = st.best_score;

    auto reanchor = [&](const Quat& target) {
        anchor = q_mul(q_inv(koff), target);
        st.anchor_limit = band;
        compose_kernels(T, xi_s, wedge ? T.wedge : nullptr, anchor, dtab, xi_t, w_t, ws);
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

__global__ void __launch_bounds__(kWarps * 32, 2) refine_kernel(RefineArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const BandTables& T = a.T;
    float2* xi = reinterpret_cast<float2*>(sm);                        // rows*32
    float* fbuf = reinterpret_cast<float*>(xi + (size_t)T.rows * 32);   // rows_band
    float* tbuf = fbuf + a.rows_band;
    WarpScratch* wsc = reinterpret_cast<WarpScratch*>(
        (reinterpret_cast<uintptr_t>(tbuf + a.rows_band) + 15) & ~uintptr_t(15));
    __shared__ int s_win, s_next;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpScratch& ws = wsc[warp];
    float* scratch = a.scratch + (size_t)(blockIdx.x * kWarps + warp) * a.scratch_per_warp;

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            s_win = atomicAdd(a.win_counter, 1);
            s_next = 0;
        }
        __syncthreads();
        const int w = s_win;
        if (w >= a.n_win) break;
        const int nc = a.cand_count[w];
        CandState* cs = a.cand + (size_t)w * a.max_cand;
        if (nc > 0) {
            const float* cw = a.coef + (long long)w * a.ldc;
            for (int r = threadIdx.x; r < a.rows_band; r += blockDim.x) {
                fbuf[r] = cw[r];
                tbuf[r] = a.t_hat[r];
            }
            __syncthreads();
            for (int e = threadIdx.x; e < T.rows * 32; e += blockDim.x)
                xi[e] = xi_entry(T, a.row_group, fbuf, tbuf, a.block_off, a.radial_count, e >> 5,
                                 e & 31);
            __syncthreads();
            for (;;) {
                int c = 0;
                if (lane == 0) c = atomicAdd(&s_next, 1);
                c = __shfl_sync(0xffffffffu, c, 0);
                if (c >= nc) break;
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
        }
        if (a.last_band && threadIdx.x == 0) {
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

size_t refine_smem_bytes(const BandTables& T, int rows_band, int max_cand) {
    (void)max_cand;
    return sizeof(float2) * (size_t)T.rows * 32 + sizeof(float) * 2 * rows_band + 16 +
           sizeof(WarpScratch) * kWarps;
}

long long refine_scratch_floats(const BandTables& T) {
    // dtab (N_xi(L) floats, +1 pad) + two band-layout complex kernels
    return (long long)(xi_off(T.L + 1) + 2) + 4LL * T.rows * 32;
}

int refine_resident_blocks(const BandTables& T, int rows_band, int max_cand, int device) {
    const size_t smem = refine_smem_bytes(T, rows_band, max_cand);
    cudaFuncSetAttribute(refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, refine_kernel, kWarps * 32, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return (per_sm > 0 ? per_sm : 1) * sms;
}

int launch_refine(const RefineArgs& a, int blocks, cudaStream_t s) {
    if (a.n_win <= 0) return 0;
    const size_t smem = refine_smem_bytes(a.T, a.rows_band, a.max_cand);
    cudaFuncSetAttribute(refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    refine_kernel<<<blocks, kWarps * 32, smem, s>>>(a);
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
