// Fine-grained operators of the reference API on the device, FP64, on the
// reference's own layouts (complex128 coefficient sets: degree blocks, row k,
// column m + l; XiBlocks: degree blocks of (2l+1)^2 entries [m][m']):
//   xi_coefficients      (src/xcorr.cpp:21-50)
//   xi_compose_right     (src/xcorr.cpp:149-155)
//   rotate_expansion     (src/steer.cpp:208-223)
//   exhaustive_baseline  (src/optimize.cpp:523-539, grid_scores 48-97)
// These serve the reference-facing entry points and the evaluation-ratio
// report; the alignment itself runs the FP32 band-layout kernels of refine.cu.
#include <cfloat>

#include "ops.hpp"

namespace bmb {

namespace {

__host__ __device__ __forceinline__ int xi_block(int l) { return l * (2 * l - 1) * (2 * l + 1) / 3; }

__device__ __forceinline__ void degree_of(int e, int L, int& l, int& r) {
    // XiBlocks entry e -> degree l and offset r inside the block
    l = 0;
    while (l < L && xi_block(l + 1) <= e) ++l;
    r = e - xi_block(l);
}

// xi_l[m,m'] = sum_k conj(f_klm) t_klm'
__global__ void xi_coefficients_kernel(const double2* __restrict__ f, long long ldf, const double2* __restrict__ t,
                                       long long ldt, const int* __restrict__ coef_off,
                                       const int* __restrict__ radial_count, int L, double2* __restrict__ out) {
    const int nxi = xi_block(L + 1);
    const int set = blockIdx.y;
    const double2* fs = f + set * ldf;
    const double2* ts = t + set * ldt;
    double2* o = out + (size_t)set * nxi;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nxi; e += gridDim.x * blockDim.x) {
        int l, r;
        degree_of(e, L, l, r);
        const int w = 2 * l + 1, m = r / w, mp = r % w;  // (m + l, m' + l)
        double re = 0.0, im = 0.0;
        const int base = coef_off[l];
        for (int k = 0; k < radial_count[l]; ++k) {
            const double2 a = fs[base + k * w + m], b = ts[base + k * w + mp];
            re += a.x * b.x + a.y * b.y;  // conj(a) b
            im += a.x * b.y - a.y * b.x;
        }
        o[e] = make_double2(re, im);
    }
}

// out_l[m,m'] = sum_n xi_l[m,n] D^l_{m',n}(a), degrees l <= l_limit (zero above)
__global__ void xi_compose_right_kernel(const double2* __restrict__ xi, const double2* __restrict__ D, int L,
                                        int l_limit, double2* __restrict__ out) {
    const int nxi = xi_block(L + 1);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nxi; e += gridDim.x * blockDim.x) {
        int l, r;
        degree_of(e, L, l, r);
        if (l > l_limit) {
            out[e] = make_double2(0.0, 0.0);
            continue;
        }
        const int w = 2 * l + 1, m = r / w, mp = r % w;
        const double2* xr = xi + xi_block(l) + m * w;
        const double2* dr = D + xi_block(l) + mp * w;
        double re = 0.0, im = 0.0;
        for (int n = 0; n < w; ++n) {
            const double2 x = xr[n], d = dr[n];
            re += x.x * d.x - x.y * d.y;
            im += x.x * d.y + x.y * d.x;
        }
        out[e] = make_double2(re, im);
    }
}

// f'_{k,l,n} = sum_m D^l_{n,m} f_{k,l,m}
__global__ void rotate_expansion_kernel(const double2* __restrict__ f, const double2* __restrict__ D,
                                        const int* __restrict__ coef_off, const int* __restrict__ radial_count,
                                        int L, int coeffs, double2* __restrict__ out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < coeffs; e += gridDim.x * blockDim.x) {
        int l = 0;
        while (l < L && coef_off[l + 1] <= e) ++l;
        const int w = 2 * l + 1, r = e - coef_off[l], k = r / w, n = r % w;
        const double2* fr = f + coef_off[l] + k * w;
        const double2* dr = D + xi_block(l) + n * w;
        double re = 0.0, im = 0.0;
        for (int m = 0; m < w; ++m) {
            const double2 x = fr[m], d = dr[m];
            re += d.x * x.x - d.y * x.y;
            im += d.x * x.y + d.y * x.x;
        }
        out[e] = make_double2(re, im);
    }
}

// ---------------------------------------------------------------- exhaustive grid
// Per beta row j: A_j[m][m'] = sum_l xi_l[m,m'] d^l_{m,m'}(beta_j) (degree collapse).
__global__ void grid_collapse_kernel(const double2* __restrict__ xi, const double* __restrict__ dgrid, int L,
                                     int l_cut, double2* __restrict__ A) {
    const int j = blockIdx.y, w = 2 * l_cut + 1;
    const int nxc = xi_block(l_cut + 1);
    const double* d = dgrid + (size_t)j * nxc;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < w * w; e += gridDim.x * blockDim.x) {
        const int m = e / w - l_cut, mp = e % w - l_cut;
        const int l0 = max(abs(m), abs(mp));
        double re = 0.0, im = 0.0;
        for (int l = l0; l <= l_cut; ++l) {
            const int wl = 2 * l + 1, at = xi_block(l) + (m + l) * wl + (mp + l);
            const double dv = d[at];
            re += xi[at].x * dv;
            im += xi[at].y * dv;
        }
        A[(size_t)j * w * w + e] = make_double2(re, im);
    }
    (void)L;
}

struct Best {
    double score;
    long long flat;
};
__device__ __forceinline__ bool better(const Best& a, const Best& b) {
    return a.score > b.score || (a.score == b.score && a.flat < b.flat);
}

// One CTA per (beta row j, gamma k): b[m] = sum_m' A_j[m][m'] e^{-i m' gamma_k}, then
// score(i) = Re sum_m e^{-i m alpha_i} b[m] for every alpha_i; the CTA's best
// (first maximum in flat order) to block_best.
__global__ void grid_sweep_kernel(const double2* __restrict__ A, int l_cut, int na, int ng, Best* block_best) {
    extern __shared__ double2 sb[];
    const int j = blockIdx.y, k = blockIdx.x, w = 2 * l_cut + 1;
    const double pi = 3.14159265358979323846;
    const double gam = 2.0 * pi * k / ng;
    const double2* Aj = A + (size_t)j * w * w;
    for (int m = threadIdx.x; m < w; m += blockDim.x) {
        double re = 0.0, im = 0.0;
        for (int mp = 0; mp < w; ++mp) {
            double s, c;
            sincos(-(mp - l_cut) * gam, &s, &c);
            const double2 a = Aj[m * w + mp];
            re += a.x * c - a.y * s;
            im += a.x * s + a.y * c;
        }
        sb[m] = make_double2(re, im);
    }
    __syncthreads();
    Best mine{-DBL_MAX, LLONG_MAX};
    for (int i = threadIdx.x; i < na; i += blockDim.x) {
        const double alp = 2.0 * pi * i / na;
        double acc = 0.0;
        for (int m = 0; m < w; ++m) {
            double s, c;
            sincos(-(m - l_cut) * alp, &s, &c);
            acc += c * sb[m].x - s * sb[m].y;
        }
        const Best cand{acc, ((long long)j * na + i) * ng + k};
        if (better(cand, mine)) mine = cand;
    }
    // block reduction
    __shared__ Best red[32];
    for (int o = 16; o; o >>= 1) {
        Best other{__shfl_xor_sync(0xffffffffu, mine.score, o), __shfl_xor_sync(0xffffffffu, mine.flat, o)};
        if (better(other, mine)) mine = other;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mine;
    __syncthreads();
    if (threadIdx.x < 32) {
        const int nw = blockDim.x >> 5;
        mine = threadIdx.x < nw ? red[threadIdx.x] : Best{-DBL_MAX, LLONG_MAX};
        for (int o = 16; o; o >>= 1) {
            Best other{__shfl_xor_sync(0xffffffffu, mine.score, o), __shfl_xor_sync(0xffffffffu, mine.flat, o)};
            if (better(other, mine)) mine = other;
        }
        if (threadIdx.x == 0) block_best[(size_t)j * gridDim.x + k] = mine;
    }
}

__global__ void best_reduce_kernel(const Best* in, long long n, Best* out) {
    Best mine{-DBL_MAX, LLONG_MAX};
    for (long long i = threadIdx.x; i < n; i += blockDim.x)
        if (better(in[i], mine)) mine = in[i];
    __shared__ Best red[32];
    for (int o = 16; o; o >>= 1) {
        Best other{__shfl_xor_sync(0xffffffffu, mine.score, o), __shfl_xor_sync(0xffffffffu, mine.flat, o)};
        if (better(other, mine)) mine = other;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int wv = 1; wv < (int)(blockDim.x >> 5); ++wv)
            if (better(red[wv], mine)) mine = red[wv];
        *out = mine;
    }
}

}  // namespace

int launch_xi_coefficients(const double* f, long long ldf, const double* t, long long ldt, int n,
                           const int* coef_off, const int* radial_count, int L, double* out, cudaStream_t s) {
    if (n <= 0) return 0;
    const int nxi = xi_block(L + 1);
    dim3 grid((nxi + 255) / 256, n);
    xi_coefficients_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const double2*>(f), ldf,
                                               reinterpret_cast<const double2*>(t), ldt, coef_off, radial_count, L,
                                               reinterpret_cast<double2*>(out));
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int launch_xi_compose_right(const double* xi, const double* D, int L, int l_limit, double* out, cudaStream_t s) {
    const int nxi = xi_block(L + 1);
    xi_compose_right_kernel<<<(nxi + 255) / 256, 256, 0, s>>>(reinterpret_cast<const double2*>(xi),
                                                              reinterpret_cast<const double2*>(D), L, l_limit,
                                                              reinterpret_cast<double2*>(out));
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int launch_rotate_expansion(const double* f, const double* D, const int* coef_off, const int* radial_count, int L,
                            int coeffs, double* out, cudaStream_t s) {
    rotate_expansion_kernel<<<(coeffs + 255) / 256, 256, 0, s>>>(reinterpret_cast<const double2*>(f),
                                                                 reinterpret_cast<const double2*>(D), coef_off,
                                                                 radial_count, L, coeffs,
                                                                 reinterpret_cast<double2*>(out));
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int launch_exhaustive(const double* xi, const double* dgrid, int L, int l_cut, int na, int nb, int ng,
                      double* scratch, double* best_score, long long* best_flat, cudaStream_t s) {
    const int w = 2 * l_cut + 1;
    double2* A = reinterpret_cast<double2*>(scratch);
    Best* blocks = reinterpret_cast<Best*>(A + (size_t)nb * w * w);
    Best* fin = blocks + (size_t)nb * ng;
    grid_collapse_kernel<<<dim3((w * w + 255) / 256, nb), 256, 0, s>>>(reinterpret_cast<const double2*>(xi), dgrid,
                                                                      L, l_cut, A);
    grid_sweep_kernel<<<dim3(ng, nb), 128, sizeof(double2) * w, s>>>(A, l_cut, na, ng, blocks);
    best_reduce_kernel<<<1, 1024, 0, s>>>(blocks, (long long)nb * ng, fin);
    cudaMemcpyAsync(best_score, &fin->score, sizeof(double), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(best_flat, &fin->flat, sizeof(long long), cudaMemcpyDeviceToHost, s);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

size_t exhaustive_scratch_bytes(int l_cut, int nb, int ng) {
    const size_t w = 2 * l_cut + 1;
    return sizeof(double2) * nb * w * w + sizeof(Best) * ((size_t)nb * ng + 1);
}

}  // namespace bmb
