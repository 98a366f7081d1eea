// Missing-wedge handling (kernel K8 + the template power kernel).
//
// apply_wedge_taper (src/xcorr.cpp:210-232): r2c -> x smoothstep keep profile
// -> c2r -> / n^3, batched over particles with cuFFT (FP32) before any shift
// window is cut.  wedge_power_kernel (xcorr.cpp:234-357): |T|^2 of the 2n
// zero-padded template (cuFFT, FP64), ray integrals of the power over a
// Gauss-Legendre x uniform direction grid on the GPU, spherical-harmonic
// analysis of both fields on the host (FP64, a few thousand directions).
// Binary projector apply_wedge (xcorr.cpp:359-381) for the data generator.
#include <cufft.h>

#include <cmath>
#include <complex>
#include <stdexcept>
#include <vector>

#include "wedge.hpp"

namespace bmb {

namespace {

__global__ void scale_spectrum_kernel(float2* spec, const float* __restrict__ profile,
                                      long long per_vol, long long total) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const float p = profile[i % per_vol];
        spec[i].x *= p;
        spec[i].y *= p;
    }
}

__global__ void scale_spectrum_d_kernel(double2* spec, const double* __restrict__ profile,
                                        long long per_vol, long long total) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const double p = profile[i % per_vol];
        spec[i].x *= p;
        spec[i].y *= p;
    }
}

__global__ void pad_template_kernel(const float* __restrict__ t, int n, double* __restrict__ out) {
    const int np = 2 * n, off = n / 2;
    const long long tot = (long long)n * n * n;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % n), y = (int)((i / n) % n), z = (int)(i / ((long long)n * n));
        out[((long long)(z + off) * np + (y + off)) * np + (x + off)] = t[i];
    }
}

// full power grid from the half spectrum (Hermitian mirror), DC zeroed
__global__ void power_grid_kernel(const double2* __restrict__ half, int np, double* __restrict__ pw) {
    const int nph = np / 2 + 1;
    const long long tot = (long long)np * np * np;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % np), y = (int)((i / np) % np), z = (int)(i / ((long long)np * np));
        double2 h;
        if (x < nph) {
            h = half[((long long)z * np + y) * nph + x];
        } else {
            const int zz = (np - z) % np, yy = (np - y) % np;
            h = half[((long long)zz * np + yy) * nph + (np - x)];
        }
        pw[i] = i == 0 ? 0.0 : h.x * h.x + h.y * h.y;
    }
}

// q(dir) = sum_j r_j^2 P(r_j dir), r_j = (j + 1/2) r_max / n_rad, trilinear in
// the periodic power grid (xcorr.cpp:271-315)
__global__ void power_rays_kernel(const double* __restrict__ pw, int np, const double* __restrict__ dirs,
                                  int n_dir, int n_rad, double* __restrict__ q) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_dir) return;
    const double dx = dirs[3 * d], dy = dirs[3 * d + 1], dz = dirs[3 * d + 2];
    const double r_max = np / 2.0;
    auto wrap = [np](int i) { return (i % np + np) % np; };
    double acc = 0.0;
    for (int j = 0; j < n_rad; ++j) {
        const double r = (j + 0.5) * r_max / n_rad;
        const double fx = r * dx, fy = r * dy, fz = r * dz;
        const int ix = (int)floor(fx), iy = (int)floor(fy), iz = (int)floor(fz);
        const double ux = fx - ix, uy = fy - iy, uz = fz - iz;
        double v = 0.0;
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b)
                for (int c = 0; c < 2; ++c) {
                    const double w = (c ? ux : 1 - ux) * (b ? uy : 1 - uy) * (a ? uz : 1 - uz);
                    v += w * pw[((long long)wrap(iz + a) * np + wrap(iy + b)) * np + wrap(ix + c)];
                }
        acc += r * r * v;
    }
    q[d] = acc;
}

void check_cufft(cufftResult r, const char* what) {
    if (r != CUFFT_SUCCESS) throw std::runtime_error(std::string("cuFFT failure in ") + what);
}

}  // namespace

// smoothstep keep profile (wedge_keep_profile, xcorr.cpp:195-208), tilt axis y, beam z
double keep_profile(double theta_deg, double nx, double ny, double nz, double taper_deg) {
    (void)ny;
    if (theta_deg >= 90.0) return 1.0;
    const double along = std::fabs(nz), in_plane = std::fabs(nx);
    if (taper_deg <= 0.0) return along <= std::tan(theta_deg * kPiH / 180.0) * in_plane ? 1.0 : 0.0;
    if (along == 0.0 && in_plane == 0.0) return 1.0;
    const double a = std::atan2(along, in_plane) * 180.0 / kPiH;
    const double x = (theta_deg - a) / taper_deg;
    if (x >= 1.0) return 1.0;
    if (x <= 0.0) return 0.0;
    return x * x * (3.0 - 2.0 * x);
}

WedgeFilter::WedgeFilter(int n_, double theta, double taper) : n(n_), theta_deg(theta), taper_deg(taper) {
    const int nh = n / 2 + 1;
    std::vector<float> prof((size_t)n * n * nh);
    std::vector<double> prof_d(prof.size());
    const double inv = 1.0 / ((double)n * n * n);
    auto sf = [this](int i) { return i <= n / 2 ? i : i - n; };
    for (int z = 0; z < n; ++z)
        for (int y = 0; y < n; ++y)
            for (int x = 0; x < nh; ++x) {
                const size_t at = ((size_t)z * n + y) * nh + x;
                const double p = keep_profile(theta_deg, x, sf(y), sf(z), taper_deg);
                prof[at] = (float)(p * inv);
                prof_d[at] = p * inv;
            }
    profile.reserve(sizeof(float) * prof.size());
    cudaMemcpy(profile.p, prof.data(), sizeof(float) * prof.size(), cudaMemcpyHostToDevice);
    profile_d.reserve(sizeof(double) * prof_d.size());
    cudaMemcpy(profile_d.p, prof_d.data(), sizeof(double) * prof_d.size(), cudaMemcpyHostToDevice);
}

WedgeFilter::~WedgeFilter() {
    for (auto& kv : plans) {
        cufftDestroy(kv.second.first);
        cufftDestroy(kv.second.second);
    }
}

void WedgeFilter::apply(const float* in, float* out, int count, cudaStream_t s) {
    if (count <= 0) return;
    const int nh = n / 2 + 1;
    const long long per = (long long)n * n * nh;
    auto it = plans.find(count);
    if (it == plans.end()) {
        int dims[3] = {n, n, n};
        cufftHandle f, b;
        check_cufft(cufftPlanMany(&f, 3, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_R2C, count), "plan r2c");
        check_cufft(cufftPlanMany(&b, 3, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_C2R, count), "plan c2r");
        it = plans.emplace(count, std::make_pair(f, b)).first;
    }
    cufftSetStream(it->second.first, s);
    cufftSetStream(it->second.second, s);
    spec.reserve(sizeof(float2) * per * count);
    check_cufft(cufftExecR2C(it->second.first, const_cast<float*>(in), spec.as<cufftComplex>()), "r2c");
    scale_spectrum_kernel<<<1024, 256, 0, s>>>(spec.as<float2>(), profile.as<float>(), per, per * count);
    check_cufft(cufftExecC2R(it->second.second, spec.as<cufftComplex>(), out), "c2r");
}

// Binary or tapered filter in FP64 for one volume (data generator / tests).
void apply_wedge_d(const double* in, double* out, int n, const double* profile_d, cudaStream_t s) {
    const int nh = n / 2 + 1;
    const long long per = (long long)n * n * nh;
    int dims[3] = {n, n, n};
    cufftHandle f, b;
    check_cufft(cufftPlanMany(&f, 3, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, 1), "plan d2z");
    check_cufft(cufftPlanMany(&b, 3, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D, 1), "plan z2d");
    cufftSetStream(f, s);
    cufftSetStream(b, s);
    double2* spec = nullptr;
    cudaMallocAsync(&spec, sizeof(double2) * per, s);
    check_cufft(cufftExecD2Z(f, const_cast<double*>(in), reinterpret_cast<cufftDoubleComplex*>(spec)), "d2z");
    scale_spectrum_d_kernel<<<512, 256, 0, s>>>(spec, profile_d, per, per);
    check_cufft(cufftExecZ2D(b, reinterpret_cast<cufftDoubleComplex*>(spec), out), "z2d");
    cudaFreeAsync(spec, s);
    cudaStreamSynchronize(s);
    cufftDestroy(f);
    cufftDestroy(b);
}

WedgePowerFactors wedge_power_factors(const float* tmpl_dev, int n, int l_max, double theta_deg,
                                      double taper_deg, cudaStream_t s) {
    WedgePowerFactors wf;
    const size_t ntri = (size_t)(l_max + 1) * (l_max + 2) / 2;
    wf.chi_hat.assign(ntri, {0.0, 0.0});
    wf.q_hat.assign(ntri, {0.0, 0.0});
    wf.total = 0.0;
    if (theta_deg >= 90.0) return wf;
    const int np = 2 * n, nph = np / 2 + 1;
    const long long tot = (long long)np * np * np;
    double *pad = nullptr, *pw = nullptr, *dirs_d = nullptr, *q_d = nullptr;
    double2* half = nullptr;
    cudaMallocAsync(&pad, sizeof(double) * tot, s);
    cudaMemsetAsync(pad, 0, sizeof(double) * tot, s);
    pad_template_kernel<<<512, 256, 0, s>>>(tmpl_dev, n, pad);
    cudaMallocAsync(&half, sizeof(double2) * (long long)np * np * nph, s);
    cufftHandle f;
    int dims[3] = {np, np, np};
    check_cufft(cufftPlanMany(&f, 3, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, 1), "plan pad");
    cufftSetStream(f, s);
    check_cufft(cufftExecD2Z(f, pad, reinterpret_cast<cufftDoubleComplex*>(half)), "pad d2z");
    cudaMallocAsync(&pw, sizeof(double) * tot, s);
    power_grid_kernel<<<1024, 256, 0, s>>>(half, np, pw);
    // direction grid: 3(L+1) Gauss-Legendre polar x 3(L+1) uniform azimuth
    const int nt = 3 * (l_max + 1), npf = 3 * (l_max + 1), n_rad = 2 * n;
    std::vector<double> u, wu;
    host::gauss_legendre(nt, u, wu);
    std::vector<double> dirs((size_t)nt * npf * 3);
    for (int t = 0; t < nt; ++t) {
        const double st = std::sqrt(std::max(0.0, 1.0 - u[t] * u[t]));
        for (int p = 0; p < npf; ++p) {
            const double phi = 2.0 * kPiH * p / npf;
            double* d = &dirs[((size_t)t * npf + p) * 3];
            d[0] = st * std::cos(phi);
            d[1] = st * std::sin(phi);
            d[2] = u[t];
        }
    }
    cudaMallocAsync(&dirs_d, sizeof(double) * dirs.size(), s);
    cudaMemcpyAsync(dirs_d, dirs.data(), sizeof(double) * dirs.size(), cudaMemcpyHostToDevice, s);
    cudaMallocAsync(&q_d, sizeof(double) * nt * npf, s);
    power_rays_kernel<<<(nt * npf + 127) / 128, 128, 0, s>>>(pw, np, dirs_d, nt * npf, n_rad, q_d);
    std::vector<double> q((size_t)nt * npf);
    cudaMemcpyAsync(q.data(), q_d, sizeof(double) * q.size(), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cufftDestroy(f);
    cudaFree(pad);
    cudaFree(half);
    cudaFree(pw);
    cudaFree(dirs_d);
    cudaFree(q_d);
    // spherical-harmonic analysis (xcorr.cpp:317-341)
    std::vector<double> ptab(ntri);
    const double wphi = 2.0 * kPiH / npf;
    for (int t = 0; t < nt; ++t) {
        host::legendre(l_max, u[t], ptab.data());
        const double wt = wu[t];
        for (int m = 0; m <= l_max; ++m) {
            std::complex<double> gq{0, 0}, gc{0, 0};
            for (int p = 0; p < npf; ++p) {
                const std::complex<double> e = std::polar(1.0, -m * (2.0 * kPiH * p / npf));
                const double* d = &dirs[((size_t)t * npf + p) * 3];
                const double chi = 1.0 - keep_profile(theta_deg, d[0], d[1], d[2], taper_deg);
                gq += q[(size_t)t * npf + p] * e;
                gc += chi * e;
            }
            for (int l = m; l <= l_max; ++l) {
                const double pwt = ptab[host::tri(l, m)] * wt * wphi;
                wf.q_hat[host::tri(l, m)] += gq * pwt;
                wf.chi_hat[host::tri(l, m)] += gc * pwt;
            }
        }
        for (int p = 0; p < npf; ++p) wf.total += q[(size_t)t * npf + p] * wt * wphi;
    }
    return wf;
}

}  // namespace bmb
