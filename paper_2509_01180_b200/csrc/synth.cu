// Voxel synthesis of a coefficient set (the averaged map), kernel K11 — the
// device form of synthesize() (src/basis.cpp:332-419) with its Catmull-Rom
// radial table (basis.cpp:221-245): FP64 throughout, one thread per voxel.
#include "synth.hpp"

namespace bmb {

namespace {

__host__ __device__ inline int tri_i(int l, int m) { return l * (l + 1) / 2 + m; }

// fully normalized Condon-Shortley Pbar_l^m(u), packed (l, m >= 0) triangle
// (legendre_table, src/detail/quadrature.hpp:62-85)
template <int LB>
__device__ void legendre_d(int L, double u, double* out) {
    const double s = sqrt(fmax(0.0, 1.0 - u * u));
    out[0] = 0.28209479177387814;  // 1/sqrt(4 pi)
    for (int m = 1; m <= L; ++m) out[tri_i(m, m)] = -sqrt((2.0 * m + 1.0) / (2.0 * m)) * s * out[tri_i(m - 1, m - 1)];
    for (int m = 0; m < L; ++m) out[tri_i(m + 1, m)] = sqrt(2.0 * m + 3.0) * u * out[tri_i(m, m)];
    for (int m = 0; m <= L; ++m)
        for (int l = m + 2; l <= L; ++l) {
            const double a = sqrt((4.0 * l * l - 1.0) / ((double)l * l - (double)m * m));
            const double b = sqrt(((double)(l - 1) * (l - 1) - (double)m * m) / (4.0 * (double)(l - 1) * (l - 1) - 1.0));
            out[tri_i(l, m)] = a * (u * out[tri_i(l - 1, m)] - b * out[tri_i(l - 2, m)]);
        }
}

template <int LB>
__global__ void __launch_bounds__(128) synthesize_kernel(SynthArgs a) {
    const long long nvox = (long long)a.n * a.n * a.n;
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= nvox) return;
    const int n = a.n, L = a.L;
    const int xi = (int)(idx % n), yi = (int)((idx / n) % n), zi = (int)(idx / ((long long)n * n));
    const double x = (xi - n / 2) * (2.0 / n), y = (yi - n / 2) * (2.0 / n), z = (zi - n / 2) * (2.0 / n);
    const double r2 = x * x + y * y + z * z;
    if (r2 >= 1.0) {  // outside the unit ball
        a.out[idx] = 0.0;
        return;
    }
    const double r = sqrt(r2);
    const double u = r > 1e-14 ? z / r : 1.0;
    const double phi = atan2(y, x);
    double ptab[(LB + 1) * (LB + 2) / 2];
    legendre_d<LB>(L, u, ptab);
    double2 phase[LB + 1];
    phase[0] = make_double2(1.0, 0.0);
    double sphi, cphi;
    sincos(phi, &sphi, &cphi);
    for (int m = 1; m <= L; ++m)
        phase[m] = make_double2(phase[m - 1].x * cphi - phase[m - 1].y * sphi,
                                phase[m - 1].x * sphi + phase[m - 1].y * cphi);
    // Catmull-Rom weights on the fine radial grid
    const double tpos = r * a.n_fine;
    const int i0 = min((int)tpos, a.n_fine - 1);
    const double f = tpos - i0;
    const double wm1 = ((-0.5 * f + 1.0) * f - 0.5) * f;
    const double w0 = (1.5 * f - 2.5) * f * f + 1.0;
    const double w1 = ((-1.5 * f + 2.0) * f + 0.5) * f;
    const double w2 = (0.5 * f - 0.5) * f * f;
    double acc = 0.0;
    double2 bm[LB + 1], bneg[LB + 1];
    for (int l = 0; l <= L; ++l) {
        const int nk = a.radial_count[l];
        if (nk == 0) continue;
        for (int m = 0; m <= l; ++m) bm[m] = bneg[m] = make_double2(0.0, 0.0);
        const double2* block = a.coef + a.block_off[l];
        for (int k = 0; k < nk; ++k) {
            const double* row = a.table + (size_t)(a.pair_off[l] + k) * a.row_len + i0;
            const double rv = wm1 * row[0] + w0 * row[1] + w1 * row[2] + w2 * row[3];
            const double2* c = block + (size_t)k * (2 * l + 1) + l;
            for (int m = 0; m <= l; ++m) {
                bm[m].x += rv * c[m].x;
                bm[m].y += rv * c[m].y;
            }
            if (!a.real_volume)
                for (int m = 1; m <= l; ++m) {
                    bneg[m].x += rv * c[-m].x;
                    bneg[m].y += rv * c[-m].y;
                }
        }
        if (a.real_volume) {
            // f(k,l,-m) = (-1)^m conj f(k,l,m) pairs with Y_{l,-m}: twice the real part
            acc += ptab[tri_i(l, 0)] * bm[0].x;
            for (int m = 1; m <= l; ++m) {
                const double pp = ptab[tri_i(l, m)];
                acc += 2.0 * pp * (bm[m].x * phase[m].x - bm[m].y * phase[m].y);
            }
        } else {  // Re of sum_m b_m Y_lm + sum_{m>0} b_{-m} Y_{l,-m}
            for (int m = 0; m <= l; ++m) {
                const double pp = ptab[tri_i(l, m)];
                acc += pp * (bm[m].x * phase[m].x - bm[m].y * phase[m].y);
            }
            for (int m = 1; m <= l; ++m) {
                const double pp = ((m & 1) ? -1.0 : 1.0) * ptab[tri_i(l, m)];
                // conj(pp * phase) = pp * (phase.x, -phase.y)
                acc += pp * (bneg[m].x * phase[m].x + bneg[m].y * phase[m].y);
            }
        }
    }
    a.out[idx] = acc;
}

}  // namespace

int launch_synthesize(const SynthArgs& a, cudaStream_t s) {
    const long long nvox = (long long)a.n * a.n * a.n;
    const int grid = (int)((nvox + 127) / 128);
    if (a.L <= 8) synthesize_kernel<8><<<grid, 128, 0, s>>>(a);
    else if (a.L <= 16) synthesize_kernel<16><<<grid, 128, 0, s>>>(a);
    else if (a.L <= 24) synthesize_kernel<24><<<grid, 128, 0, s>>>(a);
    else if (a.L <= 48) synthesize_kernel<48><<<grid, 128, 0, s>>>(a);
    else return 1;
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace bmb
