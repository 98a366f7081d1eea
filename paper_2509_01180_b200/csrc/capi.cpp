// extern "C" boundary of libballmatch_b200 (declared in include/ballmatch_b200.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>

#include "../../include/ballmatch_b200.h"
#include "bmb_internal.hpp"
#include "context.hpp"
#include "average.hpp"
#include "generate.hpp"
#include "ops.hpp"
#include "sweep_tc.hpp"
#include "refine.cuh"
#include "rotation.cuh"
#include "tables.hpp"
#include "wedge.hpp"

namespace {
// FP32 evaluation tolerances (the same values as kFp32AcceptTol / kFp32GradTol
// of include/ballmatch_b200.hpp and api.FP32_ACCEPT_TOL / FP32_GRAD_TOL)
constexpr double kFp32AcceptTolC = 1e-6;
constexpr double kFp32GradTolC = 1e-5;
}  // namespace

struct bm_context {
    std::unique_ptr<bmb::Context> impl;
};

namespace bmb {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace bmb

extern "C" {

const char* bm_last_error(void) { return bmb::g_last_error.c_str(); }

int bm_abi_version(void) { return BM_ABI_VERSION; }

int bm_split3_gemm(int fmt, int block_n, int kchunk, const void* a_hi, const void* a_lo, const void* b_hi,
                   const void* b_lo, float* out, long long ldo, long long m_pad, long long n_pad,
                   long long k_pad, int m_valid, int n_valid, const float* row_scale,
                   const float* col_scale, void* stream) {
    bmb::SplitGemmArgs a;
    a.fmt = fmt;
    a.block_n = block_n;
    a.kchunk = kchunk;
    a.a_hi = a_hi;
    a.a_lo = a_lo;
    a.b_hi = b_hi;
    a.b_lo = b_lo;
    a.out = out;
    a.ldo = ldo;
    a.m_pad = m_pad;
    a.n_pad = n_pad;
    a.k_pad = k_pad;
    a.m_valid = m_valid;
    a.n_valid = n_valid;
    a.row_scale = row_scale;
    a.col_scale = col_scale;
    const int rc = bmb::launch_split3_gemm(a, static_cast<cudaStream_t>(stream));
    if (rc != BM_OK) bmb::set_last_error("bm_split3_gemm: bad shape or launch failure");
    return rc;
}

}  // extern "C"

namespace {
// Map C++ exceptions to status codes (the reference's exception types:
// std::invalid_argument -> BM_ERR_ARG, std::domain_error -> BM_ERR_DOMAIN).
template <class F>
int guarded(const char* what, F&& f) {
    try {
        return f();
    } catch (const std::invalid_argument& e) {
        bmb::set_last_error(std::string(what) + ": " + e.what());
        return BM_ERR_ARG;
    } catch (const std::domain_error& e) {
        bmb::set_last_error(std::string(what) + ": " + e.what());
        return BM_ERR_DOMAIN;
    } catch (const std::bad_alloc&) {
        bmb::set_last_error(std::string(what) + ": out of device memory");
        return BM_ERR_NOMEM;
    } catch (const std::exception& e) {
        bmb::set_last_error(std::string(what) + ": " + e.what());
        return BM_ERR_CUDA;
    }
}
// The caller's stream (NULL = the legacy default stream) and the context's
// stream are joined with events: context work starts after the caller's prior
// work, and the caller's later work starts after the context's.
struct StreamJoin {
    cudaStream_t user, ctx;
    cudaEvent_t ev = nullptr;
    StreamJoin(bm_context* c, void* s)
        : user(s ? static_cast<cudaStream_t>(s) : cudaStreamLegacy), ctx(c->impl->stream) {
        cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        cudaEventRecord(ev, user);
        cudaStreamWaitEvent(ctx, ev, 0);
    }
    ~StreamJoin() {
        cudaEventRecord(ev, ctx);
        cudaStreamWaitEvent(user, ev, 0);
        cudaEventDestroy(ev);
    }
};
}  // namespace

extern "C" {

int bm_context_create(int device, int n, int l_max, double lambda_cut, bm_context** out) {
    return guarded("bm_context_create", [&] {
        if (!out) throw std::invalid_argument("null output handle");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw std::runtime_error("no CUDA device");
        if (device < 0 || device >= ndev) throw std::invalid_argument("bad device index");
        const double cut = lambda_cut > 0 ? lambda_cut : bmb::host::default_lambda_cut(n, l_max);
        auto* c = new bm_context;
        c->impl = std::make_unique<bmb::Context>(device, n, l_max, cut);
        *out = c;
        return BM_OK;
    });
}

int bm_context_destroy(bm_context* ctx) {
    delete ctx;
    return BM_OK;
}

int bm_context_info(const bm_context* ctx, long long* info) {
    if (!ctx || !info) return BM_ERR_STATE;
    const auto& c = *ctx->impl;
    long long v[10] = {c.n, c.basis.l_max, c.geo.coeffs, c.geo.support, c.geo.m_pad, c.geo.k_pad,
                       c.basis.n_r, c.basis.n_theta, c.basis.n_phi, 0};
    for (int l = 0; l <= c.basis.l_max; ++l) v[9] += c.basis.radial_count(l);
    std::memcpy(info, v, sizeof(v));
    return BM_OK;
}

double bm_context_lambda_cut(const bm_context* ctx) { return ctx ? ctx->impl->basis.lambda_cut : 0.0; }

int bm_context_roots(const bm_context* ctx, int l, double* roots, double* norms) {
    if (!ctx || l < 0 || l > ctx->impl->basis.l_max) return -1;
    const auto& b = ctx->impl->basis;
    for (int k = 0; k < b.radial_count(l); ++k) {
        if (roots) roots[k] = b.roots[l][k];
        if (norms) norms[k] = b.norms[l][k];
    }
    return b.radial_count(l);
}

double bm_default_lambda_cut(int n, int l_max) { return bmb::host::default_lambda_cut(n, l_max); }

int bm_basis_roots(int l_max, double lambda_cut, int l, double* roots, double* norms, int* count) {
    return guarded("bm_basis_roots", [&] {
        if (l < 0 || l > l_max) throw std::invalid_argument("degree outside [0, l_max]");
        if (!count) throw std::invalid_argument("null count");
        const bmb::host::Basis b = bmb::host::make_basis(l_max, lambda_cut);
        for (int k = 0; k < b.radial_count(l); ++k) {
            if (roots) roots[k] = b.roots[l][k];
            if (norms) norms[k] = b.norms[l][k];
        }
        *count = b.radial_count(l);
        return (int)BM_OK;
    });
}

int bm_expand(bm_context* ctx, const float* vols, int count, const int* shifts, double* out,
              void* stream) {
    return guarded("bm_expand", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (count < 0 || (count > 0 && (!vols || !out))) throw std::invalid_argument("bad buffers");
        auto& c = *ctx->impl;
        cudaSetDevice(c.device);
        std::vector<int> wv(count), ws(3 * count, 0);
        for (int i = 0; i < count; ++i) wv[i] = i;
        if (shifts) ws.assign(shifts, shifts + 3 * count);
        StreamJoin join(ctx, stream);
        const long long stride = (long long)c.n * c.n * c.n;
        c.expand_windows(vols, stride, count, wv, ws);
        bmb::launch_to_complex(c.coef.as<float>(), count, c.geo.m_pad, c.geo, out, c.stream);
        if (cudaGetLastError() != cudaSuccess) throw std::runtime_error("kernel launch failed");
        return (int)BM_OK;
    });
}


int bm_expand_windows(bm_context* ctx, const float* vols, int n_vol, const int* win_vol, const int* win_shift,
                      int n_win, double* out, void* stream) {
    return guarded("bm_expand_windows", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (n_vol < 0 || n_win < 0 || (n_win > 0 && (!vols || !out || !win_vol || !win_shift)))
            throw std::invalid_argument("bad buffers");
        for (int i = 0; i < n_win; ++i)
            if (win_vol[i] < 0 || win_vol[i] >= n_vol) throw std::invalid_argument("window volume index out of range");
        auto& c = *ctx->impl;
        cudaSetDevice(c.device);
        const std::vector<int> wv(win_vol, win_vol + n_win), ws(win_shift, win_shift + 3 * (size_t)n_win);
        StreamJoin join(ctx, stream);
        const long long stride = (long long)c.n * c.n * c.n;
        c.expand_windows(vols, stride, n_vol, wv, ws);
        bmb::launch_to_complex(c.coef.as<float>(), n_win, c.geo.m_pad, c.geo, out, c.stream);
        if (cudaGetLastError() != cudaSuccess) throw std::runtime_error("kernel launch failed");
        return (int)BM_OK;
    });
}

static bmb::AlignConfig cfg_of(const bm_align_config* c) {
    if (!c) throw std::invalid_argument("null config");
    if (c->n_bands < 0 || c->n_bands > 16) throw std::invalid_argument("config: at most 16 bands");
    if (c->n_thresholds < 0 || c->n_thresholds > 8) throw std::invalid_argument("config: at most 8 band thresholds");
    bmb::AlignConfig a;
    a.bands.assign(c->bands, c->bands + c->n_bands);
    a.auto_bands = c->auto_bands != 0;
    a.prune_after_band = c->prune_after_band != 0;
    if (c->n_thresholds > 0) a.band_thresholds.assign(c->thresholds, c->thresholds + c->n_thresholds);
    a.seed_grid_step = c->seed_grid_step;
    a.max_candidates = c->max_candidates;
    a.newton_max_iter = c->newton_max_iter;
    a.step_damping = c->step_damping;
    a.shift_radius = c->shift_radius;
    a.shift_step = c->shift_step;
    // accept_tol == 0 (e.g. a zero-initialised struct): the FP32 defaults of the
    // C++ and Python wrappers (slack 1e-6, gradient floor 1e-5);
    // negative or non-finite values reach validate() and are rejected there
    if (c->accept_tol == 0.0) {
        a.accept_tol = kFp32AcceptTolC;
        a.grad_tol = std::max(c->grad_tol, kFp32GradTolC);
    } else {
        a.accept_tol = c->accept_tol;
        a.grad_tol = c->grad_tol;
    }
    return a;
}

int bm_set_template(bm_context* ctx, const float* tmpl, double wedge_theta_deg, void* stream) {
    return guarded("bm_set_template", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (!tmpl) throw std::invalid_argument("null template");
        cudaSetDevice(ctx->impl->device);
        StreamJoin join(ctx, stream);
        ctx->impl->set_template(tmpl, wedge_theta_deg);
        return (int)BM_OK;
    });
}

double bm_template_norm(const bm_context* ctx) { return ctx ? ctx->impl->t_norm : 0.0; }

int bm_align_batch(bm_context* ctx, const float* particles, int count, const bm_align_config* cfg,
                   bm_align_result* out, void* stream) {
    return guarded("bm_align_batch", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (count < 0 || (count > 0 && (!particles || !out))) throw std::invalid_argument("bad buffers");
        cudaSetDevice(ctx->impl->device);
        StreamJoin join(ctx, stream);
        const auto res = ctx->impl->align_batch(particles, count, cfg_of(cfg));
        for (int i = 0; i < count; ++i) {
            const auto& r = res[i];
            bm_align_result& o = out[i];
            for (int j = 0; j < 3; ++j) o.shift[j] = r.shift[j];
            for (int j = 0; j < 4; ++j) o.quat[j] = r.quat[j];
            o.score = r.score;
            o.converged = r.converged;
            o.candidates = r.candidates;
            o.evaluations = r.evaluations;
            o.subtomo_norm = r.subtomo_norm;
            o.windows = r.windows;
            o.n_bands = (int)std::min<size_t>(r.bands.size(), 16);
            for (int j = 0; j < o.n_bands; ++j) o.bands[j] = r.bands[j];
            for (int j = 0; j < 16; ++j)
                o.evaluations_per_band[j] = j < (int)r.evaluations_per_band.size() ? r.evaluations_per_band[j] : 0;
            o.expand_template_s = r.expand_template_s;
            o.coarse_search_s = r.coarse_search_s;
            o.fine_search_s = r.fine_search_s;
        }
        return (int)BM_OK;
    });
}

int bm_search_windows(bm_context* ctx, const float* vols, int n_vol, const int* win_vol,
                      const int* win_shift, int n_win, const bm_align_config* cfg,
                      bm_window_result* out, void* stream) {
    return guarded("bm_search_windows", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (n_win < 0 || (n_win > 0 && (!vols || !win_vol || !win_shift || !out)))
            throw std::invalid_argument("bad buffers");
        for (int i = 0; i < n_win; ++i)
            if (win_vol[i] < 0 || win_vol[i] >= n_vol) throw std::invalid_argument("window volume index out of range");
        cudaSetDevice(ctx->impl->device);
        StreamJoin join(ctx, stream);
        std::vector<int> wv(win_vol, win_vol + n_win), ws(win_shift, win_shift + 3 * n_win);
        const auto res = ctx->impl->run_windows(vols, n_vol, wv, ws, cfg_of(cfg));
        for (int i = 0; i < n_win; ++i) {
            const auto& r = res[i];
            bm_window_result& o = out[i];
            o.volume = r.particle;
            for (int j = 0; j < 3; ++j) o.shift[j] = r.shift[j];
            o.valid = r.valid;
            o.n_candidates = r.n_cand;
            o.converged = r.converged;
            o.raw_score = r.raw_score;
            o.norm_score = r.norm_score;
            o.subtomo_norm = r.sub_norm;
            for (int j = 0; j < 4; ++j) o.quat[j] = r.quat[j];
            o.evaluations = r.evals;
        }
        return (int)BM_OK;
    });
}

int bm_eval_sweep(bm_context* ctx, const double* f, int n_f, const double* t, const double* euler,
                  int n_rot, int order, double* out, void* stream) {
    return guarded("bm_eval_sweep", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (n_f < 0 || n_rot < 0 || order < 0 || order > 1) throw std::invalid_argument("bad sizes/order");
        if (n_f == 0 || n_rot == 0) return (int)BM_OK;
        auto& c = *ctx->impl;
        cudaSetDevice(c.device);
        StreamJoin join(ctx, stream);
        const int ld = c.geo.m_pad;
        c.work_f.reserve(sizeof(float) * (size_t)(n_f + 1) * ld);
        float* fr = c.work_f.as<float>();
        float* tr = fr + (size_t)n_f * ld;
        bmb::launch_from_complex(f, n_f, c.geo, fr, ld, c.stream);
        bmb::launch_from_complex(t, 1, c.geo, tr, ld, c.stream);
        bmb::BandDev& bd = c.band(c.basis.l_max);
        bmb::XiArgs xa;
        xa.T = bd.view();
        xa.row_group = bd.row_group.as<int>();
        xa.f = fr;
        xa.ldf = ld;
        xa.t = tr;
        xa.ldt = 0;
        xa.block_off = c.geo.block_off;
        xa.radial_count = c.geo.radial_count;
        xa.n = n_f;
        c.work_xi.reserve(sizeof(float4) * (size_t)n_f * bd.rows * 32);
        xa.out = c.work_xi.as<float4>();
        if (bmb::launch_build_xi(xa, c.stream) != 0) throw std::runtime_error("build_xi launch failed");
        bmb::EvalArgs ea;
        ea.T = bd.view();
        ea.xi = xa.out;
        ea.euler = euler;
        ea.n_xi = n_f;
        ea.n_rot = n_rot;
        ea.order = order;
        ea.out = out;
        if (bmb::launch_eval_sweep(ea, c.stream) != 0) throw std::runtime_error("eval sweep launch failed");
        return (int)BM_OK;
    });
}

int bm_objective_eval(bm_context* ctx, const double* f, const double* t, const double* euler,
                      const double* anchors, int n, int L, int order, double* out, void* stream) {
    return guarded("bm_objective_eval", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (n < 0 || (n > 0 && (!f || !euler || !out))) throw std::invalid_argument("bad buffers");
        if (n == 0) return (int)BM_OK;
        auto& c = *ctx->impl;
        cudaSetDevice(c.device);
        StreamJoin join(ctx, stream);
        c.objective_eval(f, t, euler, anchors, n, L, order, out);
        return (int)BM_OK;
    });
}

int bm_seed_candidates(bm_context* ctx, const double* f, int n_f, int L_low, double step,
                       int max_candidates, double* quats, int* counts, double* scores, void* stream) {
    return guarded("bm_seed_candidates", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (n_f < 0 || (n_f > 0 && (!f || !quats || !counts))) throw std::invalid_argument("bad buffers");
        if (n_f == 0) return (int)BM_OK;
        auto& c = *ctx->impl;
        cudaSetDevice(c.device);
        StreamJoin join(ctx, stream);
        c.seed_candidates(f, n_f, L_low, step, max_candidates, quats, counts, scores);
        return (int)BM_OK;
    });
}

int bm_template_coeffs(bm_context* ctx, double* out, void* stream) {
    return guarded("bm_template_coeffs", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (!out) throw std::invalid_argument("null output");
        auto& c = *ctx->impl;
        if (!c.has_template) return (int)BM_ERR_STATE;
        cudaSetDevice(c.device);
        StreamJoin join(ctx, stream);
        bmb::launch_to_complex(c.t_hat.as<float>(), 1, c.geo.m_pad, c.geo, out, c.stream);
        return (int)BM_OK;
    });
}

int bm_wedge_power_kernel(bm_context* ctx, double* out) {
    return guarded("bm_wedge_power_kernel", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (!out) throw std::invalid_argument("null output");
        auto& c = *ctx->impl;
        if (!c.wedge_active()) return (int)BM_ERR_STATE;
        const int L = c.basis.l_max;
        auto coef = [&](const std::vector<std::complex<double>>& hat, int l, int m) {
            if (m >= 0) return hat[bmb::host::tri(l, m)];
            const std::complex<double> z = std::conj(hat[bmb::host::tri(l, -m)]);
            return ((-m) % 2) ? -z : z;
        };
        size_t o = 0;
        for (int l = 0; l <= L; ++l)
            for (int m = -l; m <= l; ++m)
                for (int mp = -l; mp <= l; ++mp, ++o) {
                    const std::complex<double> w = std::conj(coef(c.chi_hat, l, m)) * coef(c.q_hat, l, mp) / c.wp_total;
                    out[2 * o] = w.real();
                    out[2 * o + 1] = w.imag();
                }
        return (int)BM_OK;
    });
}

namespace {
bmb::Euler3 euler_of(const double* q) {
    return bmb::q_euler(bmb::q_normalized(q[0], q[1], q[2], q[3]));
}
// D^l(g) blocks on the device (scratch of the context)
const double* device_wigner(bmb::Context& c, int L, const double* quat) {
    const bmb::Euler3 e = euler_of(quat);
    const std::vector<std::complex<double>> D = bmb::wigner_D_blocks(L, e.a, e.b, e.g);
    c.work_xi.reserve(sizeof(double) * 2 * D.size());
    cudaMemcpyAsync(c.work_xi.p, D.data(), sizeof(double) * 2 * D.size(), cudaMemcpyHostToDevice, c.stream);
    return c.work_xi.as<double>();
}
long long xi_entries(int L) { return (long long)(L + 1) * (2 * L + 1) * (2 * L + 3) / 3; }
struct Grid {
    int na, nb, ng;
    explicit Grid(double step) {  // EulerGrid::with_step (optimize.cpp:30-36)
        const double pi = 3.14159265358979323846;
        na = ng = (int)std::ceil(2.0 * pi / step);
        nb = (int)std::ceil(pi / step) + 1;
    }
    double beta(int j) const { return nb > 1 ? 3.14159265358979323846 * j / (nb - 1) : 0.0; }
};
}  // namespace

int bm_xi_coefficients(bm_context* ctx, const double* f, int n, const double* t, double* out, void* stream) {
    return guarded("bm_xi_coefficients", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (n < 0 || (n > 0 && (!f || !t || !out))) throw std::invalid_argument("bad buffers");
        if (n == 0) return (int)BM_OK;
        auto& c = *ctx->impl;
        cudaSetDevice(c.device);
        StreamJoin join(ctx, stream);
        if (bmb::launch_xi_coefficients(f, c.geo.coeffs, t, 0, n, c.geo.block_off, c.geo.radial_count,
                                        c.basis.l_max, out, c.stream) != 0)
            throw std::runtime_error("xi kernel launch failed");
        return (int)BM_OK;
    });
}

int bm_xi_compose_right(bm_context* ctx, const double* xi, const double* quat, int l_limit, double* out,
                        void* stream) {
    return guarded("bm_xi_compose_right", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (!xi || !quat || !out) throw std::invalid_argument("bad buffers");
        auto& c = *ctx->impl;
        cudaSetDevice(c.device);
        StreamJoin join(ctx, stream);
        const int L = c.basis.l_max;
        const double* D = device_wigner(c, L, quat);
        if (bmb::launch_xi_compose_right(xi, D, L, l_limit < 0 ? L : l_limit, out, c.stream) != 0)
            throw std::runtime_error("compose kernel launch failed");
        cudaStreamSynchronize(c.stream);  // the D scratch is reused by the next call
        return (int)BM_OK;
    });
}

int bm_rotate_expansion(bm_context* ctx, const double* f, const double* quat, double* out, void* stream) {
    return guarded("bm_rotate_expansion", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (!f || !quat || !out) throw std::invalid_argument("bad buffers");
        auto& c = *ctx->impl;
        cudaSetDevice(c.device);
        StreamJoin join(ctx, stream);
        const int L = c.basis.l_max;
        const double* D = device_wigner(c, L, quat);
        if (bmb::launch_rotate_expansion(f, D, c.geo.block_off, c.geo.radial_count, L, c.geo.coeffs, out,
                                         c.stream) != 0)
            throw std::runtime_error("rotate kernel launch failed");
        cudaStreamSynchronize(c.stream);
        return (int)BM_OK;
    });
}

int bm_wigner_D(int L, const double* quat, double* out) {
    return guarded("bm_wigner_D", [&] {
        if (L < 0 || L > bmb::kMaxL || !quat || !out) throw std::invalid_argument("bad arguments");
        const bmb::Euler3 e = euler_of(quat);
        const std::vector<std::complex<double>> D = bmb::wigner_D_blocks(L, e.a, e.b, e.g);
        std::memcpy(out, D.data(), sizeof(double) * 2 * D.size());
        return (int)BM_OK;
    });
}

long long bm_baseline_evaluation_count(double angular_step) {
    if (!(angular_step > 0.0)) return -1;
    const Grid g(angular_step);
    return (long long)g.na * g.nb * g.ng;
}

int bm_exhaustive_baseline(bm_context* ctx, const double* xi, int l_cut, double angular_step, double* quat,
                           double* score, long long* evaluations, void* stream) {
    return guarded("bm_exhaustive_baseline", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (!xi || !quat || !score) throw std::invalid_argument("bad buffers");
        if (!(angular_step > 0.0)) throw std::invalid_argument("baseline: step must be positive");
        auto& c = *ctx->impl;
        if (l_cut < 0 || l_cut > c.basis.l_max) throw std::invalid_argument("baseline: band outside [0, l_max]");
        cudaSetDevice(c.device);
        StreamJoin join(ctx, stream);
        const Grid g(angular_step);
        std::vector<double> dgrid;
        dgrid.reserve((size_t)g.nb * xi_entries(l_cut));
        for (int j = 0; j < g.nb; ++j) {
            const std::vector<double> d = bmb::little_d_full(l_cut, g.beta(j));
            dgrid.insert(dgrid.end(), d.begin(), d.end());
        }
        bmb::upload(c.work_f, dgrid, c.stream);
        c.filtered.reserve(bmb::exhaustive_scratch_bytes(l_cut, g.nb, g.ng));
        double best = 0.0;
        long long flat = 0;
        if (bmb::launch_exhaustive(xi, c.work_f.as<double>(), c.basis.l_max, l_cut, g.na, g.nb, g.ng,
                                   c.filtered.as<double>(), &best, &flat, c.stream) != 0)
            throw std::runtime_error("baseline kernel launch failed");
        if (cudaStreamSynchronize(c.stream) != cudaSuccess) throw std::runtime_error("baseline kernel failed");
        const double pi = 3.14159265358979323846;
        const int k = (int)(flat % g.ng), i = (int)((flat / g.ng) % g.na), j = (int)(flat / ((long long)g.ng * g.na));
        const bmb::Quat q = bmb::q_from_euler(2.0 * pi * i / g.na, g.beta(j), 2.0 * pi * k / g.ng);
        quat[0] = q.w, quat[1] = q.x, quat[2] = q.y, quat[3] = q.z;
        *score = best;
        if (evaluations) *evaluations = (long long)g.na * g.nb * g.ng;
        return (int)BM_OK;
    });
}

int bm_eval_sweep_tc(bm_context* ctx, const double* f, int n_f, const double* t, const double* euler, int n_rot,
                     double* out, double* timing, void* stream) {
    return guarded("bm_eval_sweep_tc", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (n_f < 0 || n_rot < 0) throw std::invalid_argument("bad sizes");
        if (n_f == 0 || n_rot == 0) return (int)BM_OK;
        if (!f || !t || !euler || !out) throw std::invalid_argument("bad buffers");
        auto& c = *ctx->impl;
        cudaSetDevice(c.device);
        StreamJoin join(ctx, stream);
        const int L = c.basis.l_max;
        const long long nxi = xi_entries(L);
        c.work_xi.reserve(sizeof(double) * 2 * (size_t)nxi * n_f);
        if (bmb::launch_xi_coefficients(f, c.geo.coeffs, t, 0, n_f, c.geo.block_off, c.geo.radial_count, L,
                                        c.work_xi.as<double>(), c.stream) != 0)
            throw std::runtime_error("xi kernel launch failed");
        bmb::SweepTcTimes tm;
        c.filtered.reserve(bmb::sweep_tc_bytes(n_f, L, n_rot));  // grow-only scratch
        if (bmb::sweep_tc(c.work_xi.as<double>(), n_f, L, euler, n_rot, out, c.filtered.p, c.stream,
                          timing ? &tm : nullptr) != 0)
            throw std::runtime_error("tensor-core sweep failed");
        if (timing) {
            timing[0] = tm.tables_ms;
            timing[1] = tm.gemm_ms;
            timing[2] = tm.gather_ms;
            timing[3] = tm.gemm_flops;
        }
        return (int)BM_OK;
    });
}

int bm_apply_wedge_taper(bm_context* ctx, const float* in, float* out, int count, void* stream) {
    return guarded("bm_apply_wedge_taper", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        auto& c = *ctx->impl;
        if (!c.wedge) throw std::invalid_argument("no wedge configured (bm_set_template with theta in (0,90))");
        cudaSetDevice(c.device);
        StreamJoin join(ctx, stream);
        c.wedge->apply(in, out, count, c.stream);
        return (int)BM_OK;
    });
}


int bm_average_accumulate(bm_context* ctx, const float* particles, int count,
                          const bm_align_result* results, double* sum, void* stream) {
    return guarded("bm_average_accumulate", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (count < 0 || (count > 0 && (!particles || !results || !sum))) throw std::invalid_argument("bad buffers");
        if (count == 0) return (int)BM_OK;
        auto& c = *ctx->impl;
        cudaSetDevice(c.device);
        StreamJoin join(ctx, stream);
        const long long vstride = (long long)c.n * c.n * c.n;
        particles = c.device_particles(particles, count);  // host buffers: the staged copy
        const float* fw = particles;
        if (c.wedge) {
            c.filtered.reserve(sizeof(float) * vstride * count);
            c.wedge->apply(particles, c.filtered.as<float>(), count, c.stream);
            ++c.timer.launches;
            fw = c.filtered.as<float>();
        }
        std::vector<int> wv(count), ws(3 * count);
        std::vector<double> q(4 * (size_t)count);
        for (int i = 0; i < count; ++i) {
            wv[i] = i;
            for (int j = 0; j < 3; ++j) ws[3 * i + j] = results[i].shift[j];
            for (int j = 0; j < 4; ++j) q[4 * i + j] = results[i].quat[j];
        }
        c.expand_windows(fw, vstride, count, wv, ws);
        bmb::upload(c.work_xi, q, c.stream);
        bmb::launch_average(c.coef.as<float>(), c.geo.m_pad, c.work_xi.as<double>(), count, c.basis.l_max,
                            c.geo.block_off, c.geo.radial_count, sum, c.stream);
        ++c.timer.launches;
        return (int)BM_OK;
    });
}

int bm_synthesize(bm_context* ctx, const double* coeffs, int real_volume, int n, double* out, void* stream) {
    return guarded("bm_synthesize", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (!coeffs || !out) throw std::invalid_argument("bad buffers");
        auto& c = *ctx->impl;
        cudaSetDevice(c.device);
        StreamJoin join(ctx, stream);
        c.synthesize(coeffs, real_volume != 0, n, out);
        return (int)BM_OK;
    });
}

int bm_context_set_timing(bm_context* ctx, int on) {
    if (!ctx) return BM_ERR_STATE;
    ctx->impl->timer.on = on != 0;
    return BM_OK;
}

int bm_context_timings(bm_context* ctx, double* out_ms, long long* out_counts, int reset) {
    if (!ctx) return BM_ERR_STATE;
    auto& t = ctx->impl->timer;
    t.collect();
    if (out_ms)
        for (int i = 0; i < bmb::K_COUNT; ++i) out_ms[i] = t.ms[i];
    if (out_counts) {
        out_counts[0] = t.launches;
        out_counts[1] = t.windows_expanded;
        out_counts[2] = t.gemm_launches;
        out_counts[3] = t.refine_launches;
    }
    if (reset) t.reset();
    return BM_OK;
}

int bm_context_eval_counts(bm_context* ctx, int L, long long* out) {
    return guarded("bm_context_eval_counts", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (L < 0 || L > bmb::kMaxL) throw std::invalid_argument("band out of range");
        cudaSetDevice(ctx->impl->device);
        ctx->impl->eval_counts(L, out);
        return (int)BM_OK;
    });
}

int bm_context_band_timings(bm_context* ctx, double* ms) {
    return guarded("bm_context_band_timings", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        auto& c = *ctx->impl;
        c.timer.collect();
        for (int b = 0; b < 4; ++b)
            for (int k = 0; k < bmb::K_COUNT; ++k) ms[b * bmb::K_COUNT + k] = c.timer.band_ms[b][k];
        return (int)BM_OK;
    });
}

int bm_context_set_lanes(bm_context* ctx, int lanes, int min_per_lane) {
    return guarded("bm_context_set_lanes", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (lanes < 1 || lanes > 8 || min_per_lane < 1) throw std::invalid_argument("lanes must be 1..8, min_per_lane >= 1");
        ctx->impl->lanes = lanes;
        ctx->impl->lane_min_particles = min_per_lane;
        return (int)BM_OK;
    });
}

int bm_context_set_expand_mode(bm_context* ctx, int mode) {
    return guarded("bm_context_set_expand_mode", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (mode != 0 && mode != 1) throw std::invalid_argument("expand mode must be 0 (factored) or 1 (gemm)");
        auto& c = *ctx->impl;
        cudaSetDevice(c.device);
        c.expand_mode = mode;
        if (mode == 1) c.ensure_operator();
        return (int)BM_OK;
    });
}

int bm_context_set_expand_pairs(bm_context* ctx, int mode) {
    return guarded("bm_context_set_expand_pairs", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        if (mode < 0 || mode > 3) throw std::invalid_argument("expand pairs mode must be 0, 1, 2 or 3");
        ctx->impl->pairs_mode = mode;
        return (int)BM_OK;
    });
}

int bm_context_set_stage_reuse(bm_context* ctx, int on) {
    return guarded("bm_context_set_stage_reuse", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        ctx->impl->stage_reuse_ = on != 0;
        return (int)BM_OK;
    });
}

int bm_context_eval_stats(bm_context* ctx, long long* evals, double* flops, int reset) {
    return guarded("bm_context_eval_stats", [&] {
        if (!ctx) return (int)BM_ERR_STATE;
        cudaSetDevice(ctx->impl->device);
        ctx->impl->read_eval_stats(evals, flops, reset != 0);
        return (int)BM_OK;
    });
}

int bm_make_template(int device, int n, int blobs, unsigned long long seed, float* out, void* stream) {
    return guarded("bm_make_template", [&] {
        if (n < 8 || n % 2 || blobs < 1 || !out) throw std::invalid_argument("bad template arguments");
        if (cudaSetDevice(device) != cudaSuccess) throw std::runtime_error("no CUDA device");
        bmb::make_template(n, blobs, seed, out, static_cast<cudaStream_t>(stream));
        return (int)BM_OK;
    });
}

int bm_make_particles(int device, const float* tmpl, int n, int count, unsigned long long base_seed,
                      int shift_max, double snr, double wedge_deg, float* out, double* quats,
                      int* shifts, void* stream) {
    return guarded("bm_make_particles", [&] {
        if (n < 8 || n % 2 || count < 0 || !tmpl || (count > 0 && !out) || shift_max < 0)
            throw std::invalid_argument("bad particle arguments");
        if (cudaSetDevice(device) != cudaSuccess) throw std::runtime_error("no CUDA device");
        std::vector<double> q(4 * (size_t)count);
        std::vector<int> sh(3 * (size_t)count);
        bmb::make_particles(tmpl, n, count, base_seed, shift_max, snr, wedge_deg, out, q.data(), sh.data(),
                            static_cast<cudaStream_t>(stream));
        if (quats) std::memcpy(quats, q.data(), sizeof(double) * q.size());
        if (shifts) std::memcpy(shifts, sh.data(), sizeof(int) * sh.size());
        return (int)BM_OK;
    });
}

}  // extern "C"
