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
__host__ __device__ double keep_profile_hd(double theta_deg, double nx, double nz, double taper_deg) {
    const double pi = 3.14159265358979323846;
    if (theta_deg >= 90.0) return 1.0;
    const double along = fabs(nz), in_plane = fabs(nx);
    if (taper_deg <= 0.0) return along <= tan(theta_deg * pi / 180.0) * in_plane ? 1.0 : 0.0;
    if (along == 0.0 && in_plane == 0.0) return 1.0;
    const double a = atan2(along, in_plane) * 180.0 / pi;
    const double x = (theta_deg - a) / taper_deg;
    if (x >= 1.0) return 1.0;
    if (x <= 0.0) return 0.0;
    return x * x * (3.0 - 2.0 * x);
}
double keep_profile(double theta_deg, double nx, double ny, double nz, double taper_deg) {
    (void)ny;
    return keep_profile_hd(theta_deg, nx, nz, taper_deg);
}

namespace {
// Spherical-harmonic analysis of the directional power q and of the removed
// fraction chi = 1 - keep on the (Gauss-Legendre u_t, uniform phi_p) sphere grid
// (the analysis step of wedge_power_kernel, xcorr.cpp:317-341), in FP64 on the
// device.  Stage 1, one CTA per ring t: the ring's phi-DFT of q and chi for every
// order m (and the ring's share of the total power).  Stage 2, one thread per
// packed (l, m): the Gauss-Legendre quadrature over the rings with the
// fully-normalised P_l^m(u_t), recomputed per thread by its column recurrence.
__global__ void ring_dft_kernel(const double* __restrict__ q, const double* __restrict__ u, int npf, int L,
                                double theta_deg, double taper_deg, double2* __restrict__ gq,
                                double2* __restrict__ gc, double* __restrict__ ring_q) {
    const int t = blockIdx.x;
    const double pi = 3.14159265358979323846;
    const double st = sqrt(fmax(0.0, 1.0 - u[t] * u[t]));
    const double* qr = q + (size_t)t * npf;
    for (int m = threadIdx.x; m <= L; m += blockDim.x) {
        double qr_re = 0.0, qr_im = 0.0, cr = 0.0, ci = 0.0;
        for (int p = 0; p < npf; ++p) {
            const double phi = 2.0 * pi * p / npf;
            double sn, cs;
            sincos(-m * phi, &sn, &cs);
            double sp, cp;
            sincos(phi, &sp, &cp);
            const double chi = 1.0 - keep_profile_hd(theta_deg, st * cp, u[t], taper_deg);
            qr_re += qr[p] * cs;
            qr_im += qr[p] * sn;
            cr += chi * cs;
            ci += chi * sn;
        }
        gq[(size_t)t * (L + 1) + m] = make_double2(qr_re, qr_im);
        gc[(size_t)t * (L + 1) + m] = make_double2(cr, ci);
    }
    if (threadIdx.x == 0) {
        double acc = 0.0;
        for (int p = 0; p < npf; ++p) acc += qr[p];
        ring_q[t] = acc;
    }
}

__global__ void sh_project_kernel(const double2* __restrict__ gq, const double2* __restrict__ gc,
                                  const double* __restrict__ ring_q, const double* __restrict__ u,
                                  const double* __restrict__ wu, int nt, int L, double wphi,
                                  double2* __restrict__ q_hat, double2* __restrict__ chi_hat, double* total) {
    const int ntri = (L + 1) * (L + 2) / 2;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == ntri) {  // the extra thread: total power sum_t w_t wphi sum_p q
        double acc = 0.0;
        for (int t = 0; t < nt; ++t) acc += ring_q[t] * wu[t] * wphi;
        *total = acc;
    }
    if (i >= ntri) return;
    int l = (int)((sqrt(8.0 * i + 1.0) - 1.0) / 2.0);
    while ((l + 1) * (l + 2) / 2 <= i) ++l;
    while (l * (l + 1) / 2 > i) --l;
    const int m = i - l * (l + 1) / 2;
    double aq_re = 0.0, aq_im = 0.0, ac_re = 0.0, ac_im = 0.0;
    for (int t = 0; t < nt; ++t) {
        // Pbar_l^m(u) by the column recurrence from Pbar_m^m (Condon-Shortley phase)
        const double x = u[t], s = sqrt(fmax(0.0, 1.0 - x * x));
        double pmm = 0.28209479177387814;  // 1/sqrt(4 pi)
        for (int k = 1; k <= m; ++k) pmm = -sqrt((2.0 * k + 1.0) / (2.0 * k)) * s * pmm;
        double pl = pmm;
        if (l > m) {
            double p0 = pmm, p1 = sqrt(2.0 * m + 3.0) * x * pmm;
            for (int k = m + 2; k <= l; ++k) {
                const double a = sqrt((4.0 * k * k - 1.0) / ((double)k * k - (double)m * m));
                const double b = sqrt(((double)(k - 1) * (k - 1) - (double)m * m) / (4.0 * (double)(k - 1) * (k - 1) - 1.0));
                const double p2 = a * (x * p1 - b * p0);
                p0 = p1;
                p1 = p2;
            }
            pl = p1;
        }
        const double w = pl * wu[t] * wphi;
        const double2 a = gq[(size_t)t * (L + 1) + m], c = gc[(size_t)t * (L + 1) + m];
        aq_re += a.x * w;
        aq_im += a.y * w;
        ac_re += c.x * w;
        ac_im += c.y * w;
    }
    q_hat[i] = make_double2(aq_re, aq_im);
    chi_hat[i] = make_double2(ac_re, ac_im);
}
}  // namespace

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
    // spherical-harmonic analysis on the device (ring_dft_kernel, sh_project_kernel)
    double *u_d = nullptr, *wu_d = nullptr, *ring_d = nullptr, *total_d = nullptr;
    double2 *gq_d = nullptr, *gc_d = nullptr, *qh_d = nullptr, *ch_d = nullptr;
    cudaMallocAsync(&u_d, sizeof(double) * nt, s);
    cudaMallocAsync(&wu_d, sizeof(double) * nt, s);
    cudaMallocAsync(&ring_d, sizeof(double) * nt, s);
    cudaMallocAsync(&total_d, sizeof(double), s);
    cudaMallocAsync(&gq_d, sizeof(double2) * nt * (l_max + 1), s);
    cudaMallocAsync(&gc_d, sizeof(double2) * nt * (l_max + 1), s);
    cudaMallocAsync(&qh_d, sizeof(double2) * ntri, s);
    cudaMallocAsync(&ch_d, sizeof(double2) * ntri, s);
    cudaMemcpyAsync(u_d, u.data(), sizeof(double) * nt, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(wu_d, wu.data(), sizeof(double) * nt, cudaMemcpyHostToDevice, s);
    ring_dft_kernel<<<nt, 64, 0, s>>>(q_d, u_d, npf, l_max, theta_deg, taper_deg, gq_d, gc_d, ring_d);
    sh_project_kernel<<<((int)ntri + 1 + 127) / 128, 128, 0, s>>>(gq_d, gc_d, ring_d, u_d, wu_d, nt, l_max,
                                                                 2.0 * kPiH / npf, qh_d, ch_d, total_d);
    std::vector<double2> qh(ntri), ch(ntri);
    cudaMemcpyAsync(qh.data(), qh_d, sizeof(double2) * ntri, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(ch.data(), ch_d, sizeof(double2) * ntri, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&wf.total, total_d, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) throw std::runtime_error("wedge power kernel failed");
    for (size_t i = 0; i < ntri; ++i) {
        wf.q_hat[i] = {qh[i].x, qh[i].y};
        wf.chi_hat[i] = {ch[i].x, ch[i].y};
    }
    cufftDestroy(f);
    for (void* p : {(void*)pad, (void*)half, (void*)pw, (void*)dirs_d, (void*)q_d, (void*)u_d, (void*)wu_d,
                    (void*)ring_d, (void*)total_d, (void*)gq_d, (void*)gc_d, (void*)qh_d, (void*)ch_d})
        cudaFree(p);
    return wf;
}

}  // namespace bmb
