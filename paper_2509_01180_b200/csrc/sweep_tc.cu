// Rotate-score-gradient sweep (config 4) on the tensor cores.
//
// For n_f kernels xi_p = xi_coefficients(f_p, t) and n_rot rotations g,
//   C(p, g)        = Re sum_{l,m,m'} xi_p[l,m,m'] D^l_{m,m'}(g)
//   dC/dalpha      = Re sum (-i m)  xi D,   dC/dgamma = Re sum (-i m') xi D,
//   dC/dbeta       = Re sum xi D'   (D' = e^{-i m a} d'^l_{m,m'}(b) e^{-i m' g})
// (correlation_derivatives order 1, src/xcorr.cpp:52-105).  The real-volume
// symmetry xi_{-m,-m'} D_{-m,-m'} = conj(xi_{m,m'} D_{m,m'}) folds the plane to
// its half (weight 2, the (0,0) entry weight 1), and every sum becomes a dot
// product of a per-particle row with a per-rotation row over K = 2 x half-plane
// entries (real, imaginary parts interleaved):
//   GEMM 1: [value | alpha | gamma rows of every particle] x [D rows]^T
//   GEMM 2: [value rows]                                   x [D' rows]^T
// run on tcgen05 with the FP16 three-pass split (split_gemm.cuh, FP32-accurate
// with the chunked TMEM drain).  The D and D' rows of a rotation are built once
// (FP64 Wigner-d recursion per (m, m') chain, steer.cpp:101-141) and shared by
// every particle -- the recursion is amortised over the particles instead of
// repeated per (particle, rotation) pair.
#include <cuda_fp16.h>

#include <cmath>
#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <utility>
#include <vector>

#include "bmb_internal.hpp"
#include "sweep_tc.hpp"

namespace bmb {

namespace {

constexpr int kMaxSweepL = 48;

// half-plane entries of degree l: (0, m') for m' = 0..l, then (m, m') for m = 1..l, m' = -l..l
__host__ __device__ __forceinline__ long long hp_offset(int l) {
    const long long L = l;
    return (L - 1) * L * (2 * L - 1) / 3 + (L - 1) * L + L;  // sum_{j<l} (2 j^2 + 2 j + 1)
}
__device__ __forceinline__ long long hp_index(int l, int m, int mp) {
    return hp_offset(l) + (m == 0 ? mp : l + 1 + (long long)(m - 1) * (2 * l + 1) + (mp + l));
}

__device__ __forceinline__ void split_store(double v, float inv_scale, __half* hi, __half* lo, long long at) {
    const float x = (float)(v * inv_scale);
    const __half h = __float2half_rn(x);
    hi[at] = h;
    lo[at] = __float2half_rn(x - __half2float(h));
}

// Per-chain recursion data (rotation independent, FP64, built on the host):
// chain c = (m, m') with l0 = max(m, |m'|): border factor and exponents, and for
// every l in (l0, L] the coefficients t1 = P cos b + Q, t1' = -P sin b, t2 = R of
// the three-term recursion (steer.cpp:101-141); l = 1 of the (0, 0) chain is
// d = cos b (P = 1, Q = 0, R = 0).
struct ChainInfo {
    double fac;
    int pa, pp, m, mp;
};

// D and D' rows of rotation g (one CTA per rotation, one thread per chain):
// FMA-only recursion on the tabulated coefficients, phases e^{-i m a}, e^{-i m' g}
// from per-rotation tables in shared memory
// (STAGED: the four half rows are assembled in shared memory and written out as
// coalesced 16-byte stores; the chains of a warp sit in different degree blocks)
template <bool STAGED>
__global__ void rotation_rows_kernel(const double* __restrict__ euler, int L, long long k_pad,
                                     const ChainInfo* __restrict__ chain, const double3* __restrict__ pqr, int chains,
                                     __half* __restrict__ d_hi_g, __half* __restrict__ d_lo_g, __half* __restrict__ p_hi_g,
                                     __half* __restrict__ p_lo_g, float dp_inv_scale) {
    extern __shared__ __align__(16) __half rows_sm[];
    __shared__ double2 ua[kMaxSweepL + 1], ug[2 * kMaxSweepL + 1];
    __shared__ double cpow[2 * kMaxSweepL + 3], spow[2 * kMaxSweepL + 3];
    const int g = blockIdx.x;
    const double al = euler[3 * g], be = euler[3 * g + 1], ga = euler[3 * g + 2];
    double sb, cb, sh, ch;
    sincos(be, &sb, &cb);
    sincos(0.5 * be, &sh, &ch);
    for (int m = threadIdx.x; m <= L; m += blockDim.x) {
        double sn, cs;
        sincos(-m * al, &sn, &cs);
        ua[m] = make_double2(cs, sn);
    }
    for (int mp = (int)threadIdx.x - L; mp <= L; mp += blockDim.x) {
        double sn, cs;
        sincos(-mp * ga, &sn, &cs);
        ug[mp + L] = make_double2(cs, sn);
    }
    for (int e = threadIdx.x; e <= 2 * L + 2; e += blockDim.x) {
        double c = 1.0, s = 1.0;
        for (int i = 0; i < e; ++i) c *= ch, s *= sh;
        cpow[e] = c;
        spow[e] = s;
    }
    __syncthreads();
    const long long row = STAGED ? 0 : (long long)g * k_pad;
    __half* d_hi = STAGED ? rows_sm : d_hi_g;
    __half* d_lo = STAGED ? rows_sm + k_pad : d_lo_g;
    __half* p_hi = STAGED ? rows_sm + 2 * k_pad : p_hi_g;
    __half* p_lo = STAGED ? rows_sm + 3 * k_pad : p_lo_g;
    if (STAGED)  // K padding of the row
        for (long long k = 2 * hp_offset(L + 1) + threadIdx.x; k < k_pad; k += blockDim.x)
            d_hi[k] = d_lo[k] = p_hi[k] = p_lo[k] = __float2half_rn(0.0f);
    for (int c = threadIdx.x; c < chains; c += blockDim.x) {
        const ChainInfo ci = chain[c];
        const int m = ci.m, mp = ci.mp, l0 = max(m, abs(mp)), pa = ci.pa, pp = ci.pp;
        double d = ci.fac * cpow[pa] * spow[pp];
        double dp = 0.5 * ci.fac * ((pp ? pp * cpow[pa + 1] * spow[pp - 1] : 0.0) -
                                    (pa ? pa * cpow[pa - 1] * spow[pp + 1] : 0.0));
        double d1 = 0.0, dp1 = 0.0;
        const double2 a = ua[m], b = ug[mp + L];
        const double phr = a.x * b.x - a.y * b.y, phi = a.x * b.y + a.y * b.x;  // e^{-i m a} e^{-i m' g}
        long long k = 2 * hp_index(l0, m, mp);
        for (int l = l0; l <= L; ++l) {
            if (l > l0) {
                const double3 t = pqr[(size_t)(l - l0 - 1) * chains + c];
                const double t1 = fma(t.x, cb, t.y), t1p = -t.x * sb;
                const double nd = fma(t1, d, -t.z * d1);
                const double ndp = fma(t1p, d, fma(t1, dp, -t.z * dp1));
                d1 = d, dp1 = dp;
                d = nd, dp = ndp;
                k = 2 * hp_index(l, m, mp);
            }
            split_store(phr * d, 1.0f, d_hi, d_lo, row + k);
            split_store(phi * d, 1.0f, d_hi, d_lo, row + k + 1);
            split_store(phr * dp, dp_inv_scale, p_hi, p_lo, row + k);
            split_store(phi * dp, dp_inv_scale, p_hi, p_lo, row + k + 1);
        }
    }
    if (STAGED) {
        __syncthreads();
        const long long v = k_pad / 8;  // uint4 per half row (k_pad is a multiple of 64)
        const uint4* src = reinterpret_cast<const uint4*>(rows_sm);
        __half* dst[4] = {d_hi_g, d_lo_g, p_hi_g, p_lo_g};
        for (int a = 0; a < 4; ++a) {
            uint4* o = reinterpret_cast<uint4*>(dst[a] + (long long)g * k_pad);
            for (long long i = threadIdx.x; i < v; i += blockDim.x) o[i] = src[a * v + i];
        }
    }
}

__device__ __forceinline__ float block_max(float v, float* red) {
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
        for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const float r = red[0];
    __syncthreads();
    return r;
}

// value / alpha / gamma rows of particle p (rows p, P + p, 2P + p), from its
// full-plane XiBlocks kernel; per-row power-of-two scales
__global__ void particle_rows_kernel(const double2* __restrict__ xi, long long nxi, int L, int P, long long k_pad,
                                     __half* __restrict__ a_hi, __half* __restrict__ a_lo, float* __restrict__ scale) {
    __shared__ float red[32];
    const int p = blockIdx.x;
    const double2* x = xi + (size_t)p * nxi;
    const long long nh = hp_offset(L + 1);
    float mx[3] = {0.f, 0.f, 0.f};
    for (int pass = 0; pass < 2; ++pass) {
        float inv[3];
        if (pass == 1)
            for (int r = 0; r < 3; ++r) {
                const float s = mx[r] > 0.f ? exp2f(ceilf(log2f(mx[r]))) : 1.0f;
                inv[r] = 1.0f / s;
                if (threadIdx.x == 0) scale[r * P + p] = s;
            }
        for (long long e = threadIdx.x; e < nh; e += blockDim.x) {
            int l = 0;
            while (l < L && hp_offset(l + 1) <= e) ++l;
            const long long r = e - hp_offset(l);
            int m, mp;
            if (r <= l) {
                m = 0, mp = (int)r;
            } else {
                m = 1 + (int)((r - l - 1) / (2 * l + 1));
                mp = (int)((r - l - 1) % (2 * l + 1)) - l;
            }
            const double w = (m == 0 && mp == 0) ? 1.0 : 2.0;
            const double2 z = x[(long long)l * (2 * l - 1) * (2 * l + 1) / 3 + (long long)(m + l) * (2 * l + 1) + (mp + l)];
            // value: [w xr, -w xi]; alpha (-i m): [w m xi, w m xr]; gamma (-i m'): [w m' xi, w m' xr]
            const double v[3][2] = {{w * z.x, -w * z.y}, {w * m * z.y, w * m * z.x}, {w * mp * z.y, w * mp * z.x}};
            for (int q = 0; q < 3; ++q) {
                if (pass == 0) {
                    mx[q] = fmaxf(mx[q], fmaxf(fabsf((float)v[q][0]), fabsf((float)v[q][1])));
                } else {
                    const long long at = (long long)(q * P + p) * k_pad + 2 * e;
                    split_store(v[q][0], inv[q], a_hi, a_lo, at);
                    split_store(v[q][1], inv[q], a_hi, a_lo, at + 1);
                }
            }
        }
        if (pass == 0)
            for (int q = 0; q < 3; ++q) mx[q] = block_max(mx[q], red);
    }
}

__global__ void gather_sweep_kernel(const float* __restrict__ o1, long long ld1, const float* __restrict__ o2,
                                    long long ld2, int P, int G, double* __restrict__ out) {
    const long long n = (long long)P * G;
    for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n; u += (long long)gridDim.x * blockDim.x) {
        const int p = (int)(u / G), g = (int)(u % G);
        double* o = out + 4 * u;
        o[0] = o1[g * ld1 + p];
        o[1] = o1[g * ld1 + P + p];
        o[2] = o2[g * ld2 + p];
        o[3] = o1[g * ld1 + 2 * P + p];
    }
}

__global__ void fill_kernel(float* p, int n, float v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

long long round_up(long long x, long long a) { return (x + a - 1) / a * a; }

double sqrt_binom_h(int n, int k) {
    double r = 1.0;
    for (int i = 1; i <= k; ++i) r *= (double)(n - k + i) / i;
    return std::sqrt(r);
}

// chains (m, m') of the half plane and their recursion coefficients, step-major
void build_chain_tables(int L, std::vector<ChainInfo>& info, std::vector<double3>& pqr) {
    const int W = 2 * L + 1;
    info.clear();
    for (int mp = 0; mp <= L; ++mp) info.push_back({0.0, 0, 0, 0, mp});
    for (int m = 1; m <= L; ++m)
        for (int mp = -L; mp <= L; ++mp) info.push_back({0.0, 0, 0, m, mp});
    const int chains = (int)info.size();
    (void)W;
    pqr.assign((size_t)L * chains, double3{0.0, 0.0, 0.0});
    for (int c = 0; c < chains; ++c) {
        ChainInfo& ci = info[c];
        const int m = ci.m, mp = ci.mp, l0 = std::max(m, std::abs(mp));
        if (l0 == 0) {
            ci.fac = 1.0, ci.pa = ci.pp = 0;
        } else if (m == l0) {
            ci.fac = (((l0 - mp) & 1) ? -1.0 : 1.0) * sqrt_binom_h(2 * l0, l0 + mp), ci.pa = l0 + mp, ci.pp = l0 - mp;
        } else if (mp == l0) {
            ci.fac = sqrt_binom_h(2 * l0, l0 + m), ci.pa = l0 + m, ci.pp = l0 - m;
        } else {  // m' = -l0
            ci.fac = (((l0 + m) & 1) ? -1.0 : 1.0) * sqrt_binom_h(2 * l0, l0 + m), ci.pa = l0 - m, ci.pp = l0 + m;
        }
        for (int l = l0 + 1; l <= L; ++l) {
            double3 t{0.0, 0.0, 0.0};
            if (l == 1) {  // d^1_00 = cos b
                t = double3{1.0, 0.0, 0.0};
            } else {
                const double a = std::sqrt(((double)l * l - (double)m * m) * ((double)l * l - (double)mp * mp));
                t.x = (2.0 * l - 1.0) * l * (l - 1.0) / ((l - 1.0) * a);
                t.y = -(2.0 * l - 1.0) * (double)m * mp / ((l - 1.0) * a);
                const bool has2 = m <= l - 2 && std::abs(mp) <= l - 2;
                t.z = has2 ? l * std::sqrt(((double)(l - 1) * (l - 1) - (double)m * m) *
                                           ((double)(l - 1) * (l - 1) - (double)mp * mp)) /
                                 ((l - 1.0) * a)
                           : 0.0;
            }
            pqr[(size_t)(l - l0 - 1) * chains + c] = t;
        }
    }
}

struct ChainTablesDev {
    ChainInfo* info = nullptr;
    double3* pqr = nullptr;
    int chains = 0;
};
// per (device, L), built once and kept for the process
const ChainTablesDev& chain_tables(int L) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, ChainTablesDev> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    ChainTablesDev& t = cache[{dev, L}];
    if (t.info) return t;
    std::vector<ChainInfo> info;
    std::vector<double3> pqr;
    build_chain_tables(L, info, pqr);
    if (cudaMalloc(&t.info, sizeof(ChainInfo) * info.size()) != cudaSuccess ||
        cudaMalloc(&t.pqr, sizeof(double3) * (pqr.empty() ? 1 : pqr.size())) != cudaSuccess) {
        t.info = nullptr;
        return t;
    }
    cudaMemcpy(t.info, info.data(), sizeof(ChainInfo) * info.size(), cudaMemcpyHostToDevice);
    if (!pqr.empty()) cudaMemcpy(t.pqr, pqr.data(), sizeof(double3) * pqr.size(), cudaMemcpyHostToDevice);
    t.chains = (int)info.size();
    return t;
}

}  // namespace

long long sweep_tc_k(int L) { return 2 * hp_offset(L + 1); }

size_t sweep_tc_bytes(int P, int L, int G) {
    const long long k_pad = round_up(sweep_tc_k(L), 64);
    const long long m1 = round_up(3LL * P, 128), m2 = round_up(P, 128), n_pad = round_up(G, 128);
    const size_t b_rows = sizeof(__half) * (size_t)n_pad * k_pad;
    const size_t a_rows = sizeof(__half) * (size_t)m1 * k_pad;
    return 4 * b_rows + 2 * a_rows + sizeof(float) * (m1 + n_pad * 2) + sizeof(float) * (size_t)n_pad * (m1 + m2);
}

int sweep_tc(const double* xi, int P, int L, const double* euler, int G, double* out, void* scratch, cudaStream_t s,
             SweepTcTimes* times) {
    if (P <= 0 || G <= 0) return 0;
    if (L < 0 || L > kMaxSweepL || !scratch) return 1;
    const long long nxi = (long long)(L + 1) * (2 * L + 1) * (2 * L + 3) / 3;
    const long long k_pad = round_up(sweep_tc_k(L), 64);
    const long long m1 = round_up(3LL * P, 128), m2 = round_up(P, 128), n_pad = round_up(G, 128);
    const float dp_scale = exp2f(ceilf(log2f((float)(L > 0 ? L : 1))));
    char* buf = static_cast<char*>(scratch);
    const size_t b_rows = sizeof(__half) * (size_t)n_pad * k_pad;  // one of hi / lo
    const size_t a_rows = sizeof(__half) * (size_t)m1 * k_pad;
    cudaMemsetAsync(buf, 0, 4 * b_rows + 2 * a_rows, s);  // K and row padding must be zero
    __half* d_hi = reinterpret_cast<__half*>(buf);
    __half* d_lo = d_hi + (size_t)n_pad * k_pad;
    __half* p_hi = d_lo + (size_t)n_pad * k_pad;
    __half* p_lo = p_hi + (size_t)n_pad * k_pad;
    __half* a_hi = p_lo + (size_t)n_pad * k_pad;
    __half* a_lo = a_hi + (size_t)m1 * k_pad;
    float* a_scale = reinterpret_cast<float*>(a_lo + (size_t)m1 * k_pad);
    float* col_dp = a_scale + m1;
    float* o1 = col_dp + n_pad;
    float* o2 = o1 + (size_t)n_pad * m1;
    cudaEvent_t ev[4];
    if (times)
        for (auto& e : ev) cudaEventCreate(&e);
    if (times) cudaEventRecord(ev[0], s);
    const ChainTablesDev& ct = chain_tables(L);
    if (!ct.info) return 2;
    const size_t rows_smem = sizeof(__half) * 4 * (size_t)k_pad;
    if (rows_smem <= 200 * 1024) {
        if (cudaFuncSetAttribute(rotation_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)rows_smem) != cudaSuccess)
            return 2;
        rotation_rows_kernel<true><<<G, 256, rows_smem, s>>>(euler, L, k_pad, ct.info, ct.pqr, ct.chains, d_hi, d_lo,
                                                             p_hi, p_lo, 1.0f / dp_scale);
    } else {
        rotation_rows_kernel<false><<<G, 256, 0, s>>>(euler, L, k_pad, ct.info, ct.pqr, ct.chains, d_hi, d_lo, p_hi,
                                                      p_lo, 1.0f / dp_scale);
    }
    particle_rows_kernel<<<P, 256, 0, s>>>(reinterpret_cast<const double2*>(xi), nxi, L, P, k_pad, a_hi, a_lo,
                                           a_scale);
    fill_kernel<<<(int)((n_pad + 255) / 256), 256, 0, s>>>(col_dp, (int)n_pad, dp_scale);  // D' column scale
    if (times) cudaEventRecord(ev[1], s);
    SplitGemmArgs g;
    g.fmt = 0;
    g.block_n = 128;
    g.a_hi = a_hi;
    g.a_lo = a_lo;
    g.b_hi = d_hi;
    g.b_lo = d_lo;
    g.out = o1;
    g.ldo = m1;
    g.m_pad = m1;
    g.n_pad = n_pad;
    g.k_pad = k_pad;
    g.m_valid = 3 * P;
    g.n_valid = G;
    g.row_scale = a_scale;
    g.col_scale = nullptr;
    int rc = launch_split3_gemm(g, s);
    g.b_hi = p_hi;
    g.b_lo = p_lo;
    g.out = o2;
    g.ldo = m2;
    g.m_pad = m2;
    g.m_valid = P;
    g.col_scale = col_dp;
    rc |= launch_split3_gemm(g, s);
    if (times) cudaEventRecord(ev[2], s);
    gather_sweep_kernel<<<1184, 256, 0, s>>>(o1, m1, o2, m2, P, G, out);
    if (times) {
        cudaEventRecord(ev[3], s);
        cudaEventSynchronize(ev[3]);
        float t0, t1, t2;
        cudaEventElapsedTime(&t0, ev[0], ev[1]);
        cudaEventElapsedTime(&t1, ev[1], ev[2]);
        cudaEventElapsedTime(&t2, ev[2], ev[3]);
        times->tables_ms = t0;
        times->gemm_ms = t1;
        times->gather_ms = t2;
        times->gemm_flops = 2.0 * (double)k_pad * n_pad * (m1 + m2) * 3.0;  // three FP16 passes
        for (auto& e : ev) cudaEventDestroy(e);
    }
    if (rc != 0 || cudaGetLastError() != cudaSuccess) return 2;
    return 0;
}

}  // namespace bmb
