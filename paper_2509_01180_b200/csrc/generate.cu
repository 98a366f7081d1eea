// Seeded synthetic inputs on the device (kernel K10): the BASELINE.json
// template model (isotropic Gaussian blobs, sigma ~ U[1.5,3] voxels, amplitude
// ~ U[0.5,1], centres uniform in the ball of radius 0.6, masked to the unit
// ball) and the particle pipeline of make_phantom (src/volio.cpp:285-314):
// trilinear rotation out(x) = in(R^T x) (volio.cpp:195-206), shift by -s,
// optional binary missing wedge (apply_wedge, xcorr.cpp:359-381), Gaussian
// noise at a target SNR measured inside the unit ball, float32 rounding.
// Philox4x32-10 (include/ballmatch/philox.hpp) is integer arithmetic and runs
// bit-exactly on the device; stream ids: 0 template geometry, 1 rotation,
// 2 shift, 3 noise.
#include <cuda_runtime.h>
#include <cufft.h>

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "generate.hpp"
#include "rotation.cuh"
#include "wedge.hpp"

namespace bmb {

namespace {

__host__ __device__ inline void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
    for (int i = 0; i < 10; ++i) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c[0] = n0, c[1] = n1, c[2] = n2, c[3] = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// sequential stream view (host), PhiloxStream semantics (philox.hpp:34-87)
struct HostStream {
    uint32_t k0, k1, stream, ctr = 0, blk[4];
    int lane = 4;
    bool have = false;
    double spare = 0;
    HostStream(uint64_t seed, uint32_t s) : k0((uint32_t)seed), k1((uint32_t)(seed >> 32)), stream(s) {}
    uint32_t u32() {
        if (lane == 4) {
            blk[0] = ctr, blk[1] = 0, blk[2] = stream, blk[3] = 0;
            philox10(blk, k0, k1);
            ++ctr;
            lane = 0;
        }
        return blk[lane++];
    }
    double unit() { return ((double)u32() + 1.0) * 0x1p-32; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * unit(); }
    double gauss() {
        if (have) {
            have = false;
            return spare;
        }
        const double u1 = unit(), u2 = unit();
        const double r = std::sqrt(-2.0 * std::log(u1)), a = 2.0 * kPiH * u2;
        spare = r * std::sin(a);
        have = true;
        return r * std::cos(a);
    }
    int next_int(int lo, int hi) {
        const uint64_t span = (uint64_t)(hi - lo + 1);
        return lo + (int)(((uint64_t)u32() * span) >> 32);
    }
};

struct Blob {
    double cx, cy, cz, s, a;
};

__global__ void template_kernel(int n, const Blob* __restrict__ blobs, int nb, float* __restrict__ out) {
    const long long tot = (long long)n * n * n;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % n), y = (int)((i / n) % n), z = (int)(i / ((long long)n * n));
        const double cx = (x - n / 2) * (2.0 / n), cy = (y - n / 2) * (2.0 / n), cz = (z - n / 2) * (2.0 / n);
        double v = 0.0;
        if (cx * cx + cy * cy + cz * cz < 1.0)
            for (int b = 0; b < nb; ++b) {
                const double d2 = (cx - blobs[b].cx) * (cx - blobs[b].cx) +
                                  (cy - blobs[b].cy) * (cy - blobs[b].cy) +
                                  (cz - blobs[b].cz) * (cz - blobs[b].cz);
                v += blobs[b].a * exp(-0.5 * d2 / (blobs[b].s * blobs[b].s));
            }
        out[i] = (float)v;
    }
}

// sample_trilinear (volume.cpp:19-48) of a float volume, FP64 weights
__device__ double trilinear(const float* v, int n, double x, double y, double z) {
    const double u = x * (n / 2.0) + n / 2.0, w = y * (n / 2.0) + n / 2.0, q = z * (n / 2.0) + n / 2.0;
    const int i0 = (int)floor(u), j0 = (int)floor(w), k0 = (int)floor(q);
    const double fx = u - i0, fy = w - j0, fz = q - k0;
    double acc = 0.0;
    for (int dz = 0; dz < 2; ++dz) {
        const int k = k0 + dz;
        if (k < 0 || k >= n) continue;
        const double wz = dz ? fz : 1.0 - fz;
        for (int dy = 0; dy < 2; ++dy) {
            const int j = j0 + dy;
            if (j < 0 || j >= n) continue;
            const double wy = dy ? fy : 1.0 - fy;
            for (int dx = 0; dx < 2; ++dx) {
                const int i = i0 + dx;
                if (i < 0 || i >= n) continue;
                acc += (dx ? fx : 1.0 - fx) * wy * wz * (double)v[((long long)k * n + j) * n + i];
            }
        }
    }
    return acc;
}

// rotate (out(x) = in(R^T x)) then shift by -s: sub[i] = rot[i - s]
__global__ void rotate_shift_kernel(const float* __restrict__ tmpl, int n, const double* __restrict__ rmat,
                                    const int* __restrict__ shifts, double* __restrict__ out) {
    const int p = blockIdx.y;
    const double* R = rmat + 9 * p;
    const int sx = shifts[3 * p], sy = shifts[3 * p + 1], sz = shifts[3 * p + 2];
    const long long tot = (long long)n * n * n;
    double* o = out + tot * p;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % n), y = (int)((i / n) % n), z = (int)(i / ((long long)n * n));
        // shift_volume(v, -s): out[x] = rot[x - s] (zero outside)
        const int xs = x - sx, ys = y - sy, zs = z - sz;
        double val = 0.0;
        if ((unsigned)xs < (unsigned)n && (unsigned)ys < (unsigned)n && (unsigned)zs < (unsigned)n) {
            const double cx = (xs - n / 2) * (2.0 / n), cy = (ys - n / 2) * (2.0 / n), cz = (zs - n / 2) * (2.0 / n);
            const double px = R[0] * cx + R[3] * cy + R[6] * cz;
            const double py = R[1] * cx + R[4] * cy + R[7] * cz;
            const double pz = R[2] * cx + R[5] * cy + R[8] * cz;
            val = trilinear(tmpl, n, px, py, pz);
        }
        o[i] = val;
    }
}

// in-ball mean/second moment per particle (volio.cpp:290-307)
__global__ void ball_moments_kernel(const double* __restrict__ v, int n, double* __restrict__ mom) {
    const long long tot = (long long)n * n * n;
    const double* o = v + tot * blockIdx.x;
    double s = 0.0, s2 = 0.0, c = 0.0;
    for (long long i = threadIdx.x; i < tot; i += blockDim.x) {
        const int x = (int)(i % n), y = (int)((i / n) % n), z = (int)(i / ((long long)n * n));
        const double cx = (x - n / 2) * (2.0 / n), cy = (y - n / 2) * (2.0 / n), cz = (z - n / 2) * (2.0 / n);
        if (cx * cx + cy * cy + cz * cz >= 1.0) continue;
        s += o[i];
        s2 += o[i] * o[i];
        c += 1.0;
    }
    __shared__ double red[3][32];
    for (int off = 16; off; off >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, off);
        s2 += __shfl_xor_sync(0xffffffffu, s2, off);
        c += __shfl_xor_sync(0xffffffffu, c, off);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = s;
        red[1][threadIdx.x >> 5] = s2;
        red[2][threadIdx.x >> 5] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0, d = 0;
        for (int w = 0; w < (int)(blockDim.x / 32); ++w) a += red[0][w], b += red[1][w], d += red[2][w];
        mom[3 * blockIdx.x] = a;
        mom[3 * blockIdx.x + 1] = b;
        mom[3 * blockIdx.x + 2] = d;
    }
}

// add sigma * N(0,1) (Philox stream 3, Box-Muller pairs in stream order) and round to float
__global__ void noise_round_kernel(const double* __restrict__ v, int n, const uint64_t* __restrict__ seeds,
                                   const double* __restrict__ sigma, float* __restrict__ out) {
    const int p = blockIdx.y;
    const long long tot = (long long)n * n * n;
    const uint64_t seed = seeds[p];
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    const double sg = sigma ? sigma[p] : 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
         i += (long long)gridDim.x * blockDim.x) {
        double val = v[tot * p + i];
        if (sigma) {
            // gaussian #i: pair j = i/2 uses u32 draws 2j, 2j+1 -> block j/2, lanes 2(j%2), +1
            const long long j = i >> 1;
            uint32_t c[4] = {(uint32_t)(j >> 1), 0u, 3u, 0u};
            philox10(c, k0, k1);
            const int l0 = (int)(j & 1) * 2;
            const double u1 = ((double)c[l0] + 1.0) * 0x1p-32, u2 = ((double)c[l0 + 1] + 1.0) * 0x1p-32;
            const double r = sqrt(-2.0 * log(u1)), a = 2.0 * 3.14159265358979323846 * u2;
            val += sg * ((i & 1) ? r * sin(a) : r * cos(a));
        }
        out[tot * p + i] = (float)val;
    }
}

}  // namespace

void make_template(int n, int blobs, uint64_t seed, float* out, cudaStream_t s) {
    HostStream g(seed, 0);
    std::vector<Blob> bl;
    for (int b = 0; b < blobs; ++b) {
        const double sig = g.uniform(1.5, 3.0) * (2.0 / n);
        const double amp = g.uniform(0.5, 1.0);
        double dx = g.gauss(), dy = g.gauss(), dz = g.gauss();
        double dn = std::sqrt(dx * dx + dy * dy + dz * dz);
        if (dn < 1e-12) dx = 1, dy = 0, dz = 0, dn = 1;
        const double rad = 0.6 * std::cbrt(g.unit());
        bl.push_back({rad * dx / dn, rad * dy / dn, rad * dz / dn, sig, amp});
    }
    Blob* d = nullptr;
    cudaMallocAsync(&d, sizeof(Blob) * bl.size(), s);
    cudaMemcpyAsync(d, bl.data(), sizeof(Blob) * bl.size(), cudaMemcpyHostToDevice, s);
    template_kernel<<<512, 256, 0, s>>>(n, d, blobs, out);
    cudaFreeAsync(d, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) throw std::runtime_error("template generation failed");
}

void make_particles(const float* tmpl, int n, int count, uint64_t base_seed, int shift_max, double snr,
                    double wedge_deg, float* out, double* quats, int* shifts, cudaStream_t s) {
    if (count <= 0) return;
    std::vector<double> rm(9 * (size_t)count);
    std::vector<int> sh(3 * (size_t)count);
    std::vector<uint64_t> seeds(count);
    for (int p = 0; p < count; ++p) {
        const uint64_t seed = base_seed + (uint64_t)p;
        seeds[p] = seed;
        HostStream rs(seed, 1);  // haar_rotation (volio.cpp:208-215)
        const double u1 = rs.unit(), u2 = rs.unit(), u3 = rs.unit();
        const double a = std::sqrt(1.0 - u1), b = std::sqrt(u1);
        const double t2 = 2.0 * kPiH * u2, t3 = 2.0 * kPiH * u3;
        const Quat q = q_normalized(b * std::cos(t3), a * std::sin(t2), a * std::cos(t2), b * std::sin(t3));
        quats[4 * p] = q.w, quats[4 * p + 1] = q.x, quats[4 * p + 2] = q.y, quats[4 * p + 3] = q.z;
        const double w = q.w, x = q.x, y = q.y, z = q.z;
        double* R = &rm[9 * (size_t)p];
        R[0] = 1 - 2 * (y * y + z * z), R[1] = 2 * (x * y - w * z), R[2] = 2 * (x * z + w * y);
        R[3] = 2 * (x * y + w * z), R[4] = 1 - 2 * (x * x + z * z), R[5] = 2 * (y * z - w * x);
        R[6] = 2 * (x * z - w * y), R[7] = 2 * (y * z + w * x), R[8] = 1 - 2 * (x * x + y * y);
        HostStream ss(seed, 2);
        for (int i = 0; i < 3; ++i) sh[3 * p + i] = shift_max > 0 ? ss.next_int(-shift_max, shift_max) : 0;
        for (int i = 0; i < 3; ++i) shifts[3 * p + i] = sh[3 * p + i];
    }
    const long long tot = (long long)n * n * n;
    double *rm_d, *vol_d, *mom_d, *sig_d;
    int* sh_d;
    uint64_t* seeds_d;
    cudaMallocAsync(&rm_d, sizeof(double) * rm.size(), s);
    cudaMallocAsync(&sh_d, sizeof(int) * sh.size(), s);
    cudaMallocAsync(&seeds_d, sizeof(uint64_t) * count, s);
    cudaMallocAsync(&vol_d, sizeof(double) * tot * count, s);
    cudaMallocAsync(&mom_d, sizeof(double) * 3 * count, s);
    cudaMallocAsync(&sig_d, sizeof(double) * count, s);
    cudaMemcpyAsync(rm_d, rm.data(), sizeof(double) * rm.size(), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(sh_d, sh.data(), sizeof(int) * sh.size(), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(seeds_d, seeds.data(), sizeof(uint64_t) * count, cudaMemcpyHostToDevice, s);
    dim3 grid((unsigned)((tot + 255) / 256 > 1024 ? 1024 : (tot + 255) / 256), count);
    rotate_shift_kernel<<<grid, 256, 0, s>>>(tmpl, n, rm_d, sh_d, vol_d);
    if (wedge_deg > 0.0 && wedge_deg < 90.0) {
        WedgeFilter wf(n, wedge_deg, 0.0);  // binary projector
        for (int p = 0; p < count; ++p)
            apply_wedge_d(vol_d + tot * p, vol_d + tot * p, n, wf.profile_d.as<double>(), s);
    }
    std::vector<double> sig(count, 0.0);
    if (snr > 0.0) {
        ball_moments_kernel<<<count, 512, 0, s>>>(vol_d, n, mom_d);
        std::vector<double> mom(3 * (size_t)count);
        cudaMemcpyAsync(mom.data(), mom_d, sizeof(double) * mom.size(), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        for (int p = 0; p < count; ++p) {
            const double mean = mom[3 * p] / mom[3 * p + 2];
            const double var = std::max(0.0, mom[3 * p + 1] / mom[3 * p + 2] - mean * mean);
            sig[p] = std::sqrt(var / snr);
        }
        cudaMemcpyAsync(sig_d, sig.data(), sizeof(double) * count, cudaMemcpyHostToDevice, s);
    }
    noise_round_kernel<<<grid, 256, 0, s>>>(vol_d, n, seeds_d, snr > 0.0 ? sig_d : nullptr, out);
    cudaFreeAsync(rm_d, s);
    cudaFreeAsync(sh_d, s);
    cudaFreeAsync(seeds_d, s);
    cudaFreeAsync(vol_d, s);
    cudaFreeAsync(mom_d, s);
    cudaFreeAsync(sig_d, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) throw std::runtime_error("particle generation failed");
}

}  // namespace bmb
