// Seeding (kernel K6): band-L_low correlation on the uniform ZYZ Euler grid,
// strict 26-neighbour local maxima, best-first top-N, initial candidate states.
// Restates grid_scores + seed_candidates (src/optimize.cpp:48-97, 197-253) with
// one CTA per shift window; FP64 throughout (the grid is small), the A(beta)
// collapse and phase sweeps in the reference's summation order.
#include <cfloat>

#include "smem_attr.hpp"
#include "kernels.cuh"
#include "rotation.cuh"
#include "seed.cuh"

namespace bmb {

// shared-memory plan: [f | t] (later reused for one beta slice A_j), xi (or
// the global scratch when it does not fit), scores, maxima
// shared-memory budget of a CTA (sets the beta slices per batch) and resident CTAs per SM
#ifndef BMB_SEED_SMEM_KB
#define BMB_SEED_SMEM_KB 52
#endif
#ifndef BMB_SEED_MINB
#define BMB_SEED_MINB 4
#endif
struct SeedSmem {
    size_t region0, xi, sc, maxima, bk, cands, total;
    bool xi_in_smem;
    int sb;  // beta slices collapsed per batch (A_j and b[k][m] of sb slices live at once)
};
__host__ __device__ inline SeedSmem seed_smem_plan(int rows_low, int L, int nxi, int npt, int nb, int ng) {
    const int wd = 2 * L + 1;
    SeedSmem p;
    const size_t ft = sizeof(double) * 2 * (size_t)rows_low;
    const size_t aj = sizeof(double2) * (size_t)wd * wd;
    const size_t xib = sizeof(double2) * (size_t)nxi;
    const size_t fixed = sizeof(double) * npt + 2 * sizeof(int) * (size_t)npt + 64;
    // as many slices per batch as keep the CTA near 52 KB (four CTAs per SM, measured best): the
    // three phases of a batch then run on sb times the threads between barriers
    p.sb = 1;
    for (int sb = nb; sb > 1; --sb) {
        const size_t r0 = ft > aj * sb ? ft : aj * sb;
        if (r0 + xib + fixed + sizeof(double2) * (size_t)wd * ng * sb <= BMB_SEED_SMEM_KB * 1024) {
            p.sb = sb;
            break;
        }
    }
    p.region0 = ft > aj * p.sb ? ft : aj * p.sb;
    p.region0 = (p.region0 + 15) / 16 * 16;
    const size_t bkb = sizeof(double2) * (size_t)wd * ng * p.sb;  // b[j][k][m] of one batch
    const bool cands_extra = sizeof(int) * (size_t)npt > bkb;
    const size_t rest = sizeof(double) * npt + sizeof(int) * npt + bkb + (cands_extra ? sizeof(int) * npt : 0);
    p.xi_in_smem = p.region0 + xib + rest <= 200 * 1024;
    p.xi = p.region0;
    p.sc = p.xi + (p.xi_in_smem ? xib : 0);
    p.maxima = p.sc + sizeof(double) * npt;
    p.bk = (p.maxima + sizeof(int) * npt + 15) / 16 * 16;
    p.total = p.bk + bkb;
    // axis-neighbour survivors: in the b[k][m] staging once the scores are done
    if (!cands_extra) {
        p.cands = p.bk;
    } else {
        p.cands = p.total;
        p.total += sizeof(int) * (size_t)npt;
    }
    return p;
}

// floor(x / d) for x < 2^32 / d by one multiply-high (the index arithmetic of the
// grid phases divides by run-time extents)
struct FastDiv {
    unsigned d, magic;
    __device__ __forceinline__ explicit FastDiv(int dd) : d((unsigned)dd), magic(0xFFFFFFFFu / (unsigned)dd + 1u) {}
    __device__ __forceinline__ int div(int x) const { return d == 1 ? x : (int)__umulhi((unsigned)x, magic); }
};

__global__ void __launch_bounds__(256, BMB_SEED_MINB) seed_kernel(SeedArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int w = blockIdx.x;
    const int L = a.L_low, wd = 2 * L + 1;
    const int npt = a.na * a.nb * a.ng;
    const int nrow = a.rows_low;  // real-packed rows of degrees <= L
    const SeedSmem plan = seed_smem_plan(nrow, L, a.nxi, npt, a.nb, a.ng);
    double* f = reinterpret_cast<double*>(sm);
    double* t = f + nrow;
    double2* Aj = reinterpret_cast<double2*>(sm);  // overlays f, t once xi is built
    double2* xi = plan.xi_in_smem ? reinterpret_cast<double2*>(sm + plan.xi)
                                  : a.xi_scratch + (size_t)w * a.nxi;
    double* sc = reinterpret_cast<double*>(sm + plan.sc);
    double2* Bk = reinterpret_cast<double2*>(sm + plan.bk);
    int* maxima = reinterpret_cast<int*>(sm + plan.maxima);
    __shared__ int n_max, n_cand;

    const float* cw = a.coef + (long long)w * a.ldc;
    for (int r = threadIdx.x; r < nrow; r += blockDim.x) {
        f[r] = cw[r];
        t[r] = a.t_hat[r];
    }
    if (threadIdx.x == 0) n_max = n_cand = 0;
    __syncthreads();

    // xi_l[m,m'] = sum_k conj(f_klm) t_klm'  (xi_coefficients(f_hat, t_hat), xcorr.cpp:34-50)
    for (int e = threadIdx.x; e < a.nxi; e += blockDim.x) {
        int l = 0;
        while ((l + 1) * (2 * l + 1) * (2 * l + 3) / 3 <= e) ++l;
        const int o = e - l * (2 * l - 1) * (2 * l + 1) / 3;
        const int m = o / (2 * l + 1) - l, mp = o % (2 * l + 1) - l;
        const int nk = a.radial_count[l], base = a.block_off[l];
        double re = 0.0, im = 0.0;
        for (int k = 0; k < nk; ++k) {
            const double* fr = f + base + k * (2 * l + 1);
            const double* tr = t + base + k * (2 * l + 1);
            const int am = abs(m), amp = abs(mp);
            double fre = fr[am == 0 ? 0 : 2 * am - 1], fim = am == 0 ? 0.0 : fr[2 * am];
            if (m < 0) {
                const double s = (am & 1) ? -1.0 : 1.0;
                fre *= s;
                fim *= -s;
            }
            double tre = tr[amp == 0 ? 0 : 2 * amp - 1], tim = amp == 0 ? 0.0 : tr[2 * amp];
            if (mp < 0) {
                const double s = (amp & 1) ? -1.0 : 1.0;
                tre *= s;
                tim *= -s;
            }
            re += fre * tre + fim * tim;  // conj(f) * t
            im += fre * tim - fim * tre;
        }
        xi[e] = make_double2(re, im);
    }
    __syncthreads();

    // per beta slice j: A_j[m][m'] = sum_l xi_l[m,m'] d^l_{m,m'}(beta_j), then
    // score(i,j,k) = Re sum_m ua_i[m] sum_m' A_j[m][m'] ug_k[m'].  plan.sb slices go
    // through each phase together (three barriers per batch instead of per slice);
    // every output keeps its own summation order.
    const int wd2 = wd * wd, gw = a.ng * wd, ag = a.na * a.ng;
    const FastDiv d_wd(wd), d_wd2(wd2), d_gw(gw), d_ag(ag), d_ng(a.ng), d_plane(ag);
    for (int j0 = 0; j0 < a.nb; j0 += plan.sb) {
        const int nj = min(plan.sb, a.nb - j0);
        for (int q = threadIdx.x; q < nj * wd2; q += blockDim.x) {
            const int dj = d_wd2.div(q), e = q - dj * wd2;
            const int mr = d_wd.div(e);
            const int m = mr - L, mp = e - mr * wd - L;
            double re = 0.0, im = 0.0;
            for (int l = max(abs(m), abs(mp)); l <= L; ++l) {
                const int o = l * (2 * l - 1) * (2 * l + 1) / 3 + (m + l) * (2 * l + 1) + (mp + l);
                const double d = a.dgrid[(size_t)(j0 + dj) * a.nxi + o];
                re += xi[o].x * d;
                im += xi[o].y * d;
            }
            Aj[q] = make_double2(re, im);
        }
        __syncthreads();
        // b[k][m] = sum_m' A_j[m][m'] ug_k[m'], then score = Re sum_m ua_i[m] b[k][m]
        // (the reference's collapse and sweep order, optimize.cpp:79-93)
        for (int q = threadIdx.x; q < nj * gw; q += blockDim.x) {
            const int dj = d_gw.div(q), r = q - dj * gw;
            const int k = d_wd.div(r), m = r - k * wd;
            const double2* pg = a.ug + (size_t)k * wd;
            const double2* Ar = Aj + dj * wd2 + m * wd;
            double bre = 0.0, bim = 0.0;
            for (int mp = 0; mp < wd; ++mp) {
                const double2 x = Ar[mp], y = pg[mp];
                bre += x.x * y.x - x.y * y.y;
                bim += x.x * y.y + x.y * y.x;
            }
            Bk[q] = make_double2(bre, bim);
        }
        __syncthreads();
        for (int q = threadIdx.x; q < nj * ag; q += blockDim.x) {
            const int dj = d_ag.div(q), r = q - dj * ag;
            const int i = d_ng.div(r), k = r - i * a.ng;
            const int idx = ((j0 + dj) * a.na + i) * a.ng + k;
            const double2* pa = a.ua + (size_t)i * wd;
            const double2* bk = Bk + (size_t)dj * gw + (size_t)k * wd;
            double acc = 0.0;
            for (int m = 0; m < wd; ++m) acc += pa[m].x * bk[m].x - pa[m].y * bk[m].y;
            if (a.wedge_sqrt) acc /= a.wedge_sqrt[idx];
            sc[idx] = acc;
        }
        __syncthreads();
    }

    // strict local maxima over the 26-neighbourhood (alpha/gamma wrap, beta clamps);
    // a plateau keeps its lowest flat index.  Two passes: the six axis neighbours
    // reject most points with cheap index arithmetic, and only the survivors,
    // compacted, run the full test (a warp no longer waits on its one survivor).
    int* cands = reinterpret_cast<int*>(sm + plan.cands);
    const int plane = a.na * a.ng;
    for (int idx = threadIdx.x; idx < npt; idx += blockDim.x) {
        const int j = d_plane.div(idx), ik = idx - j * plane, i = d_ng.div(ik), k = ik - i * a.ng;
        const double s = sc[idx];
        const int km = k == 0 ? idx + a.ng - 1 : idx - 1;
        const int kp = k == a.ng - 1 ? idx - (a.ng - 1) : idx + 1;
        const int im = i == 0 ? idx + (a.na - 1) * a.ng : idx - a.ng;
        const int ip = i == a.na - 1 ? idx - (a.na - 1) * a.ng : idx + a.ng;
        const int jm = j == 0 ? idx : idx - plane;
        const int jp = j == a.nb - 1 ? idx : idx + plane;
        const int nb6[6] = {km, kp, im, ip, jm, jp};
        bool keep_pt = true;
#pragma unroll
        for (int u = 0; u < 6; ++u) {
            const int other = nb6[u];
            const double o = sc[other];
            keep_pt = keep_pt && (other == idx || !(o > s || (o == s && other < idx)));
        }
        if (keep_pt) cands[atomicAdd(&n_cand, 1)] = idx;
    }
    __syncthreads();
    const int nc = n_cand;
    for (int q = threadIdx.x; q < nc; q += blockDim.x) {
        const int idx = cands[q];
        const int j = d_plane.div(idx), ik = idx - j * plane, i = d_ng.div(ik), k = ik - i * a.ng;
        const double s = sc[idx];
        bool is_max = true;
        for (int dj = -1; dj <= 1 && is_max; ++dj) {
            const int jj = j + dj;
            if (jj < 0 || jj >= a.nb) continue;
            for (int di = -1; di <= 1 && is_max; ++di) {
                int ii = i + di;  // alpha wraps (no integer modulo on the hot path)
                ii += ii < 0 ? a.na : (ii >= a.na ? -a.na : 0);
                const int row = (jj * a.na + ii) * a.ng;
                for (int dk = -1; dk <= 1; ++dk) {
                    int kk = k + dk;  // gamma wraps
                    kk += kk < 0 ? a.ng : (kk >= a.ng ? -a.ng : 0);
                    const int other = row + kk;
                    if (other == idx) continue;
                    const double o = sc[other];
                    if (o > s || (o == s && other < idx)) {
                        is_max = false;
                        break;
                    }
                }
            }
        }
        if (is_max) maxima[atomicAdd(&n_max, 1)] = idx;
    }
    __syncthreads();

    // rank by (score desc, flat index asc); keep the best max_cand
    const int nm = n_max;
    const int keep = min(nm, a.max_cand);
    for (int q = threadIdx.x; q < nm; q += blockDim.x) {
        const int idx = maxima[q];
        const double s = sc[idx];
        int rank = 0;
        for (int o = 0; o < nm; ++o) {
            const int jdx = maxima[o];
            const double t2 = sc[jdx];
            rank += (t2 > s || (t2 == s && jdx < idx)) ? 1 : 0;
        }
        if (rank < keep) {
            const int j = d_plane.div(idx), ik = idx - j * plane, i = d_ng.div(ik), k = ik - i * a.ng;
            const double alpha = 2.0 * 3.14159265358979323846 * i / a.na;
            const double beta = a.nb > 1 ? 3.14159265358979323846 * j / (a.nb - 1) : 0.0;
            const double gamma = 2.0 * 3.14159265358979323846 * k / a.ng;
            const Quat q0 = q_from_euler(alpha, beta, gamma);
            CandState& c = a.cand[(size_t)w * a.max_cand + rank];
            c.g[0] = c.best_g[0] = q0.w;
            c.g[1] = c.best_g[1] = q0.x;
            c.g[2] = c.best_g[2] = q0.y;
            c.g[3] = c.best_g[3] = q0.z;
            c.anchor[0] = 1.0;
            c.anchor[1] = c.anchor[2] = c.anchor[3] = 0.0;
            c.best_score = -DBL_MAX * 2.0;  // -inf
            c.score = 0.0;
            c.anchored = 0;
            c.anchor_limit = -1;
            c.diverged = 0;
            c.band_converged = 0;
            c.evals = 0;
            c.active = 1;
            if (a.seed_score) a.seed_score[(size_t)w * a.max_cand + rank] = s;
        }
    }
    if (threadIdx.x == 0) a.cand_count[w] = keep;
}

size_t seed_smem_bytes(const SeedArgs& a) {
    return seed_smem_plan(a.rows_low, a.L_low, a.nxi, a.na * a.nb * a.ng, a.nb, a.ng).total;
}
bool seed_needs_scratch(const SeedArgs& a) {
    return !seed_smem_plan(a.rows_low, a.L_low, a.nxi, a.na * a.nb * a.ng, a.nb, a.ng).xi_in_smem;
}

int launch_seed(const SeedArgs& a, int n_win, cudaStream_t s) {
    if (n_win <= 0) return 0;
    const size_t smem = seed_smem_bytes(a);
    if (smem > 200 * 1024) return 1;
    if (ensure_dynamic_smem(seed_kernel, (int)smem) != cudaSuccess) return 2;
    if (!seed_needs_scratch(a)) {
        seed_kernel<<<n_win, 256, smem, s>>>(a);
    } else {  // xi in global scratch: a.scratch_windows windows per launch
        if (!a.xi_scratch || a.scratch_windows < 1) return 1;
        for (int w0 = 0; w0 < n_win; w0 += a.scratch_windows) {
            SeedArgs c = a;
            c.coef = a.coef + (long long)w0 * a.ldc;
            c.cand = a.cand + (size_t)w0 * a.max_cand;
            c.cand_count = a.cand_count + w0;
            if (a.seed_score) c.seed_score = a.seed_score + (size_t)w0 * a.max_cand;
            seed_kernel<<<min(a.scratch_windows, n_win - w0), 256, smem, s>>>(c);
        }
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace bmb
