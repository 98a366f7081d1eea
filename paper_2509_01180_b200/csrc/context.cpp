// Context construction and the batched expansion driver.
#include <cstdlib>
#include <cstring>
#include "context.hpp"

#include <algorithm>
#include <stdexcept>

#include "synth.hpp"
#include "wedge.hpp"

namespace bmb {

#define BMB_CUDA(x)                                                                   \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess)                                                        \
            throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

Context::Context(int dev, int n_, int l_max, double lambda_cut) : device(dev), n(n_) {
    // n = 0: basis-only context (coefficient-space work, no expansion operator)
    if (n_ != 0 && (n_ < 8 || n_ % 2)) throw std::invalid_argument("context: grid size must be even and >= 8");
    if (l_max > kMaxL) throw std::invalid_argument("context: l_max exceeds the device tables (48)");
    BMB_CUDA(cudaSetDevice(device));
    BMB_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    {  // stream-ordered scratch (large-basis expansion, average): keep freed blocks in
       // the device pool instead of returning them to the driver at every sync
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            unsigned long long keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    basis = host::make_basis(l_max, lambda_cut);
    if (const char* e = std::getenv("BMB_EXPAND")) expand_mode = std::string(e) == "gemm" ? 1 : 0;
    geo.n = n;
    geo.l_max = l_max;
    geo.coeffs = basis.coeffs;
    geo.m_pad = (basis.coeffs + 127) / 128 * 128;
    geo.support = n_ > 0 ? host::support_count(basis, n) : 0;
    geo.k_pad = 0;
    if (n_ > 0) {
        build_factored_tables();
        if (expand_mode == 1) ensure_operator();
    }
    std::vector<int> rc(l_max + 1);
    for (int l = 0; l <= l_max; ++l) rc[l] = basis.radial_count(l);
    upload(block_off, basis.block_off, stream);
    upload(radial_count, rc, stream);
    std::vector<float> rw(geo.coeffs);
    std::vector<int4> lkm(geo.coeffs);
    for (int l = 0; l <= l_max; ++l)
        for (int k = 1; k <= basis.radial_count(l); ++k)
            for (int m = 0; m <= l; ++m)
                for (int part = 0; part < (m ? 2 : 1); ++part) {
                    const int r = basis.row(l, k, m, part);
                    rw[r] = m ? 2.0f : 1.0f;
                    lkm[r] = make_int4(l, k, m, part);
                }
    upload(row_weight, rw, stream);
    upload(row_lkm, lkm, stream);
    geo.block_off = block_off.as<int>();
    geo.radial_count = radial_count.as<int>();
    geo.row_weight = row_weight.as<float>();
    geo.row_lkm = row_lkm.as<int4>();
    BMB_CUDA(cudaStreamSynchronize(stream));
}

// dense pulled-back operator of the GEMM expansion path (built on first use)
void Context::ensure_operator() {
    if (operator_ready || n == 0) return;
    host::Operator op = host::build_operator(basis, n);
    if (op.m_pad != geo.m_pad || op.rows != geo.coeffs) throw std::logic_error("operator layout mismatch");
    voxels_host = op.voxels;
    geo.support = op.support;
    geo.k_pad = op.k_pad;
    upload(E_hi, op.hi, stream);
    upload(E_lo, op.lo, stream);
    upload(row_scale, op.row_scale, stream);
    upload(voxels, op.voxels, stream);
    BMB_CUDA(cudaStreamSynchronize(stream));
    operator_ready = true;
}

void Context::build_factored_tables() {
    const host::FactorTables ft = host::build_factor_tables(basis);
    const int L = basis.l_max, nr = basis.n_r, nt = basis.n_theta, np = basis.n_phi;
    const double h = 0.5 * n;
    std::vector<double> dirh((size_t)3 * nt * np);
    for (int t = 0; t < nt; ++t) {
        const double st = std::sqrt(std::max(0.0, 1.0 - basis.u[t] * basis.u[t]));
        for (int p = 0; p < np; ++p) {
            const double phi = 2.0 * host::kPi * p / np;  // the sample points of expand()
            double* d = dirh.data() + 3 * ((size_t)t * np + p);
            d[0] = h * st * std::cos(phi);
            d[1] = h * st * std::sin(phi);
            d[2] = h * basis.u[t];
        }
    }
    const int half = np / 2;
    std::vector<float2> tw((size_t)(half + 1) * (L + 1));
    for (int p = 0; p <= half; ++p)
        for (int m = 0; m <= L; ++m)
            tw[(size_t)p * (L + 1) + m] = make_float2((float)ft.cs[(size_t)m * np + p], (float)ft.sn[(size_t)m * np + p]);
    const int ntri = (int)host::tri_count(L);
    std::vector<float> ptab(ft.ptab.begin(), ft.ptab.end());
    std::vector<int2> tlm(ntri);
    for (int l = 0; l <= L; ++l)
        for (int m = 0; m <= l; ++m) tlm[host::tri(l, m)] = make_int2(l, m);
    std::vector<float> radial_t((size_t)nr * ft.pairs);
    for (int pr = 0; pr < ft.pairs; ++pr)
        for (int i = 0; i < nr; ++i) radial_t[(size_t)i * ft.pairs + pr] = (float)ft.radial[(size_t)pr * nr + i];
    if (ft.pairs >= 32768 || (L + 1) * (L + 1) >= 65536) throw std::invalid_argument("basis too large for the factored tables");
    std::vector<int> rowpack(geo.coeffs);
    for (int l = 0; l <= L; ++l)
        for (int k = 1; k <= basis.radial_count(l); ++k)
            for (int m = 0; m <= l; ++m)
                for (int part = 0; part < (m ? 2 : 1); ++part) {
                    const int j = m == 0 ? 0 : 2 * m - 1 + part;
                    rowpack[basis.row(l, k, m, part)] = ((ft.pair_off[l] + k - 1) << 16) | (l * l + j);
                }
    // trilinear footprint of every quadrature sample (sample_trilinear,
    // src/volume.cpp:19-48): g = r * (h d_tp) + h in FP64 exactly as the device
    // formerly computed it, base voxel packed 10 bits per axis, FP32 fractions;
    // indexed [ray][radius] (a warp's lanes walk along rays)
    if (n > 1023) throw std::invalid_argument("factored expansion: grid edge above 1023");
    std::vector<int4> samp((size_t)nt * np * nr);
    for (int s = 0; s < nt * np; ++s)
        for (int i = 0; i < nr; ++i) {
            const double r = basis.r[i];
            const double* d = dirh.data() + 3 * (size_t)s;
            const double gx = std::fma(r, d[0], h), gy = std::fma(r, d[1], h), gz = std::fma(r, d[2], h);
            const int x0 = (int)gx, y0 = (int)gy, z0 = (int)gz;
            const float fx = (float)(gx - (double)x0), fy = (float)(gy - (double)y0), fz = (float)(gz - (double)z0);
            int4 e;
            e.x = (x0 & 1023) | ((y0 & 1023) << 10) | ((z0 & 1023) << 20);
            // bit 30: the footprint leaves the window grid (0 <= g, so only on the high side)
            if (x0 + 1 >= n || y0 + 1 >= n || z0 + 1 >= n) e.x |= 1 << 30;
            std::memcpy(&e.y, &fx, 4);
            std::memcpy(&e.z, &fy, 4);
            std::memcpy(&e.w, &fz, 4);
            samp[(size_t)s * nr + i] = e;
        }
    upload(fx_r, basis.r, stream);
    upload(fx_samp, samp, stream);
    upload(fx_tw, tw, stream);
    upload(fx_ptab, ptab, stream);
    upload(fx_trilm, tlm, stream);
    upload(fx_radial, radial_t, stream);
    upload(fx_rowmap, rowpack, stream);
    fx.n = n;
    fx.L = L;
    fx.nr = nr;
    fx.nt = nt;
    fx.np = np;
    fx.coeffs = geo.coeffs;
    fx.ntri = ntri;
    fx.pairs = ft.pairs;
    fx.r = fx_r.as<double>();
    fx.samp = fx_samp.as<int4>();
    fx.tw = fx_tw.as<float2>();
    fx.ptab = fx_ptab.as<float>();
    fx.tri_lm = fx_trilm.as<int2>();
    fx.radial_t = fx_radial.as<float>();
    fx.rowpack = fx_rowmap.as<int>();
}

void Context::synthesize(const double* coef, bool real_volume, int n_out, double* out) {
    if (n_out < 8) throw std::invalid_argument("synthesize: grid size must be >= 8");
    const int L = basis.l_max;
    const int n_fine = 2048, row_len = n_fine + 3;
    std::vector<int> pair_off(L + 1);
    int pairs = 0;
    for (int l = 0; l <= L; ++l) {
        pair_off[l] = pairs;
        pairs += basis.radial_count(l);
    }
    if (!synth_table_.p) {
        std::vector<double> rows((size_t)pairs * row_len, 0.0);
        const double h = 1.0 / n_fine;
        for (int l = 0; l <= L; ++l)
            for (int k = 0; k < basis.radial_count(l); ++k) {
                double* row = rows.data() + (size_t)(pair_off[l] + k) * row_len;
                for (int j = 1; j < row_len; ++j) row[j] = basis.norms[l][k] * host::sph_jl(l, basis.roots[l][k] * (j - 1) * h);
                row[0] = (l % 2 ? -1.0 : 1.0) * row[2];  // ghost node at -h by parity
            }
        upload(synth_table_, rows, stream);
        upload(synth_pair_off_, pair_off, stream);
    }
    SynthArgs a;
    a.coef = reinterpret_cast<const double2*>(coef);
    a.real_volume = real_volume;
    a.n = n_out;
    a.L = L;
    a.block_off = geo.block_off;
    a.radial_count = geo.radial_count;
    a.pair_off = synth_pair_off_.as<int>();
    a.table = synth_table_.as<double>();
    a.n_fine = n_fine;
    a.row_len = row_len;
    a.out = out;
    if (launch_synthesize(a, stream) != 0) throw std::runtime_error("synthesize launch failed");
    ++timer.launches;
}

Context::~Context() {
    cudaSetDevice(device);
    wedge.reset();
    if (pinned_) cudaFreeHost(pinned_);
    if (stream) {
        cudaStreamSynchronize(stream);
        cudaStreamDestroy(stream);
    }
}

void Context::expand_windows(const float* vols, long long vol_stride, int n_vol,
                             const std::vector<int>& wvol, const std::vector<int>& wshift) {
    const int nw = (int)wvol.size();
    if (nw == 0) return;
    if (n == 0) throw std::invalid_argument("expand: context has no operator (n = 0)");
    if (expand_mode == 0) {
        upload(win_vol, wvol, stream);
        upload(win_shift, wshift, stream);
        coef.reserve(sizeof(float) * (size_t)nw * geo.m_pad);
        cudaEvent_t f0 = timer.begin(stream);
        // several windows per volume (the alignment's shift search): gather from an
        // x-paired copy, one 8-byte load per footprint row.  pairs_mode 0: off,
        // 1: when a volume has >= 4 windows, 2: always (tests).  Same FP32 values
        // and FMA order either way, so the coefficients are bit-identical.
        const float2* pairs = nullptr;
        const size_t pair_bytes = sizeof(float2) * (size_t)pair_volume_elems(n) * n_vol;
        const bool want = pairs_mode == 2 || (pairs_mode == 1 && nw >= 4 * (long long)n_vol);
        // pairs_mode 1 (when a volume has >= 4 windows) or 3 (always, tests): the
        // zero-padded quad copy and the pair-list kernel (K2q) when every shift fits
        // the padding and the basis has a specialised kernel
        if (pairs_mode == 3 || want) {
            static const bool quad_on = [] {
                const char* e = std::getenv("BMB_EXPAND_QUAD");
                return !(e && std::atoi(e) == 0);
            }();
            int smax = 0;
            for (int v : wshift) smax = std::max(smax, std::abs(v));
            const size_t quad_bytes = sizeof(float4) * (size_t)quad_volume_elems(n) * n_vol;
            if ((quad_on || pairs_mode == 3) && pairs_mode != 2 && smax <= kQuadPad && quad_bytes <= kMaxPairBytes &&
                expand_quads_supported(fx)) {
                // pair list: x-neighbours (same volume, y and z shift; x apart by 1 or 2) share their loads
                std::vector<int4> pl;
                std::vector<int> singles;
                for (int i = 0; i < nw;) {
                    const int dx = i + 1 < nw ? wshift[3 * i + 3] - wshift[3 * i] : 0;
                    if (i + 1 < nw && wvol[i] == wvol[i + 1] && wshift[3 * i + 1] == wshift[3 * i + 4] &&
                        wshift[3 * i + 2] == wshift[3 * i + 5] && (dx == 1 || dx == 2)) {
                        pl.push_back(make_int4(i, i + 1, dx, 0));
                        i += 2;
                    } else {
                        singles.push_back(i++);
                    }
                }
                for (size_t k = 0; k < singles.size(); k += 2)
                    pl.push_back(make_int4(singles[k], k + 1 < singles.size() ? singles[k + 1] : singles[k], 0, 0));
                const bool have = quads_hold_ && quads_src_ == vols && quads_nvol_ == n_vol && quads_stride_ == vol_stride;
                if (!have) {
                    vol_quads.reserve(quad_bytes);
                    launch_quad_volumes(vols, vol_stride, n_vol, n, vol_quads.as<float4>(), stream);
                    ++timer.launches;
                    quads_src_ = pairs_hold_ ? vols : nullptr;
                    quads_hold_ = pairs_hold_;
                    quads_nvol_ = n_vol;
                    quads_stride_ = vol_stride;
                }
                upload(win_pairs, pl, stream);
                const int rc = launch_expand_quads(fx, vol_quads.as<float4>(), win_vol.as<int>(), win_shift.as<int>(),
                                                   win_pairs.as<int4>(), (int)pl.size(), coef.as<float>(), geo.m_pad, stream);
                if (rc == 0) {
                    ++timer.launches;
                    ++timer.gemm_launches;
                    timer.windows_expanded += nw;
                    timer.end(K_GEMM, f0, stream);
                    return;
                }
                if (rc != 1) throw std::runtime_error("quad expansion launch failed");
            }
        }
        if (want && pair_bytes <= kMaxPairBytes) {
            // inside one align_group the coarse and fine passes share the copy
            const bool have = pairs_hold_ && pairs_src_ == vols && pairs_nvol_ == n_vol && pairs_stride_ == vol_stride;
            if (!have) {
                vol_pairs.reserve(pair_bytes);
                launch_pair_volumes(vols, vol_stride, n_vol, n, vol_pairs.as<float2>(), stream);
                ++timer.launches;
                pairs_src_ = pairs_hold_ ? vols : nullptr;
                pairs_nvol_ = n_vol;
                pairs_stride_ = vol_stride;
            }
            pairs = vol_pairs.as<float2>();
        }
        if (launch_expand_factored(fx, vols, vol_stride, win_vol.as<int>(), win_shift.as<int>(), nw, coef.as<float>(),
                                   geo.m_pad, stream, pairs, nw >= 2LL * n_vol) != 0)
            throw std::runtime_error("factored expansion launch failed");
        ++timer.launches;
        ++timer.gemm_launches;
        timer.windows_expanded += nw;
        timer.end(K_GEMM, f0, stream);
        return;
    }
    ensure_operator();
    const int bn = gemm_block_n;
    const long long chunk = std::min<long long>(nw, max_chunk_windows);
    const long long n_pad = (chunk + bn - 1) / bn * bn;
    vol_scale.reserve(sizeof(float) * n_vol);
    cudaEvent_t t0 = timer.begin(stream);
    launch_absmax_scale(vols, n_vol, vol_stride, vol_scale.as<float>(), stream);
    ++timer.launches;
    timer.end(K_MISC, t0, stream);
    upload(win_vol, wvol, stream);
    upload(win_shift, wshift, stream);
    B_hi.reserve(sizeof(__half) * n_pad * geo.k_pad);
    B_lo.reserve(sizeof(__half) * n_pad * geo.k_pad);
    col_scale.reserve(sizeof(float) * n_pad);
    coef.reserve(sizeof(float) * (size_t)nw * geo.m_pad);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    for (long long w0 = 0; w0 < nw; w0 += chunk) {
        const int cnt = (int)std::min<long long>(chunk, nw - w0);
        cudaEvent_t g0 = timer.begin(stream);
        launch_gather_windows(vols, vol_stride, win_vol.as<int>() + w0, win_shift.as<int>() + 3 * w0,
                              cnt, vol_scale.as<float>(), voxels.as<int>(), geo.support, geo.k_pad,
                              n, B_hi.as<__half>(), B_lo.as<__half>(), col_scale.as<float>(), stream);
        ++timer.launches;
        timer.end(K_GATHER, g0, stream);
        SplitGemmArgs a;
        a.fmt = 0;
        a.block_n = bn;
        a.kchunk = gemm_kchunk;
        a.a_hi = E_hi.p;
        a.a_lo = E_lo.p;
        a.b_hi = B_hi.p;
        a.b_lo = B_lo.p;
        a.out = coef.as<float>() + (size_t)w0 * geo.m_pad;
        a.ldo = geo.m_pad;
        a.m_pad = geo.m_pad;
        a.n_pad = (cnt + bn - 1) / bn * bn;
        a.k_pad = geo.k_pad;
        a.m_valid = geo.coeffs;
        a.n_valid = cnt;
        a.row_scale = row_scale.as<float>();
        a.col_scale = col_scale.as<float>();
        a.num_sms = sms;
        cudaEvent_t m0 = timer.begin(stream);
        if (launch_split3_gemm(a, stream) != BMB_OK) throw std::runtime_error("split3 gemm launch failed");
        ++timer.launches;
        ++timer.gemm_launches;
        timer.windows_expanded += cnt;
        timer.end(K_GEMM, m0, stream);
    }
}

}  // namespace bmb
