// extern "C" boundary of libballmatch_b200 (declared in include/ballmatch_b200.h).
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>

#include "../../include/ballmatch_b200.h"
#include "bmb_internal.hpp"
#include "context.hpp"

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

}  // extern "C"
