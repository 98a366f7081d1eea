// Host FP64 basis setup (once per context).  See basis_host.hpp.
#include "basis_host.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace bmb {
namespace host {

namespace {

// Miller downward recurrence normalized by j_0 (stable for l >= x);
// same start index as the reference (src/detail/bessel.cpp:21-38).
double jl_miller(int l, double x) {
    const int start = l + 20 + (int)std::sqrt(40.0 * l + 100.0);
    double hi = 0.0, cur = 1e-290, at_l = 0.0;
    for (int k = start; k >= 1; --k) {
        const double lo = (2.0 * k + 1.0) / x * cur - hi;
        hi = cur;
        cur = lo;
        if (k - 1 == l) at_l = cur;
        if (std::fabs(cur) > 1e270) {
            cur *= 1e-290;
            hi *= 1e-290;
            at_l *= 1e-290;
        }
    }
    return at_l * (std::sin(x) / x) / cur;
}

double djl(int l, double x) {
    if (l == 0) return -sph_jl(1, x);
    if (x < 1e-12) return l == 1 ? 1.0 / 3.0 : 0.0;
    return sph_jl(l - 1, x) - (l + 1.0) / x * sph_jl(l, x);
}

// k-th zero estimate of J_{l+1/2} (McMahon)
double zero_guess(int l, int k) {
    const double mu = 4.0 * (l + 0.5) * (l + 0.5);
    const double b = (k + 0.5 * (l + 0.5) - 0.25) * kPi;
    const double b8 = 8.0 * b;
    return b - (mu - 1.0) / b8 - 4.0 * (mu - 1.0) * (7.0 * mu - 31.0) / (3.0 * b8 * b8 * b8);
}

// root of j_l inside the sign-change bracket (lo, hi): safeguarded Newton
double bracketed_root(int l, double lo, double hi, double guess) {
    double f_lo = sph_jl(l, lo);
    double x = (guess > lo && guess < hi) ? guess : 0.5 * (lo + hi);
    for (int it = 0; it < 200; ++it) {
        const double f = sph_jl(l, x);
        if ((f > 0) == (f_lo > 0)) {
            lo = x;
            f_lo = f;
        } else {
            hi = x;
        }
        if (std::fabs(f) < 1e-14 && (hi - lo) < 1e-12 * x) return x;
        const double d = djl(l, x);
        double nx = d != 0.0 ? x - f / d : 0.5 * (lo + hi);
        if (!(nx > lo && nx < hi)) nx = 0.5 * (lo + hi);
        if (nx == x) return x;
        x = nx;
    }
    return x;
}

}  // namespace

double sph_jl(int l, double x) {
    if (x < 0.0) return ((l & 1) ? -1.0 : 1.0) * sph_jl(l, -x);
    if (x < 1e-6) {
        if (l == 0) return 1.0 - x * x / 6.0;
        double v = 1.0;
        for (int i = 1; i <= l; ++i) v *= x / (2 * i + 1);
        return v * (1.0 - x * x / (2.0 * (2 * l + 3)));
    }
    const double j0 = std::sin(x) / x;
    if (l == 0) return j0;
    const double j1 = j0 / x - std::cos(x) / x;
    if (l == 1) return j1;
    if (x > l + 0.5) {
        double a = j0, b = j1;
        for (int k = 1; k < l; ++k) {
            const double c = (2.0 * k + 1.0) / x * b - a;
            a = b;
            b = c;
        }
        return b;
    }
    return jl_miller(l, x);
}

// Roots of j_l interlace those of j_{l-1}; each row keeps a shrinking margin of
// roots beyond the cutoff so the next row stays bracketed (the reference's
// table rule, src/detail/bessel.cpp:150-178).
std::vector<std::vector<double>> bessel_roots(int l_max, double cut) {
    std::vector<std::vector<double>> rows(l_max + 1);
    std::vector<double> prev;
    for (int k = 1, beyond = 0; beyond < l_max + 2; ++k) {
        prev.push_back(k * kPi);
        if (prev.back() > cut) ++beyond;
    }
    rows[0] = prev;
    for (int l = 1; l <= l_max; ++l) {
        std::vector<double> cur;
        for (size_t i = 0, beyond = 0; i + 1 < prev.size() && (int)beyond < l_max + 2 - l; ++i) {
            cur.push_back(bracketed_root(l, prev[i], prev[i + 1], zero_guess(l, (int)i + 1)));
            if (cur.back() > cut) ++beyond;
        }
        rows[l] = cur;
        prev.swap(cur);
    }
    for (auto& r : rows)
        while (!r.empty() && r.back() > cut) r.pop_back();
    return rows;
}

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    for (int i = 0; i < (n + 1) / 2; ++i) {
        double z = std::cos(kPi * (i + 0.75) / (n + 0.5)), dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = z;
            for (int j = 2; j <= n; ++j) {
                const double p2 = ((2 * j - 1) * z * p1 - (j - 1) * p0) / j;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (z * p1 - p0) / (z * z - 1.0);
            const double dz = p1 / dp;
            z -= dz;
            if (std::fabs(dz) < 1e-15) break;
        }
        const double wt = 2.0 / ((1.0 - z * z) * dp * dp);
        x[i] = -z;
        x[n - 1 - i] = z;
        w[i] = w[n - 1 - i] = wt;
    }
}

void legendre(int l_max, double u, double* out) {
    const double s = std::sqrt(std::max(0.0, 1.0 - u * u));
    out[0] = 0.28209479177387814;  // 1/sqrt(4 pi)
    for (int m = 1; m <= l_max; ++m)
        out[tri(m, m)] = -std::sqrt((2.0 * m + 1.0) / (2.0 * m)) * s * out[tri(m - 1, m - 1)];
    for (int m = 0; m < l_max; ++m) out[tri(m + 1, m)] = std::sqrt(2.0 * m + 3.0) * u * out[tri(m, m)];
    for (int m = 0; m <= l_max; ++m)
        for (int l = m + 2; l <= l_max; ++l) {
            const double a = std::sqrt((4.0 * l * l - 1.0) / ((double)l * l - (double)m * m));
            const double b = std::sqrt(((double)(l - 1) * (l - 1) - (double)m * m) /
                                       (4.0 * (double)(l - 1) * (l - 1) - 1.0));
            out[tri(l, m)] = a * (u * out[tri(l - 1, m)] - b * out[tri(l - 2, m)]);
        }
}

double default_lambda_cut(int n, int l_max) {
    const double nyq = kPi * n / 2.0;
    const auto rows = bessel_roots(l_max, nyq);
    const size_t cap = (size_t)n * n * n / 4;
    std::vector<std::pair<double, size_t>> all;
    size_t count = 0;
    for (int l = 0; l < (int)rows.size(); ++l)
        for (double r : rows[l]) {
            all.emplace_back(r, 2 * l + 1);
            count += 2 * l + 1;
        }
    if (count <= cap) return nyq;
    std::sort(all.begin(), all.end());
    size_t acc = 0;
    double cut = kPi;
    for (const auto& [r, w] : all) {
        if (acc + w > cap) break;
        acc += w;
        cut = r;
    }
    return cut;
}

Basis make_basis(int l_max, double lambda_cut) {
    if (l_max < 0) throw std::invalid_argument("build_spec: l_max must be >= 0");
    if (!(lambda_cut >= kPi))
        throw std::invalid_argument("build_spec: lambda_cut must retain the (l=0,k=1) root pi");
    Basis b;
    b.l_max = l_max;
    b.lambda_cut = lambda_cut;
    b.roots = bessel_roots(l_max, lambda_cut);
    b.norms.resize(l_max + 1);
    b.block_off.resize(l_max + 1);
    int c = 0;
    for (int l = 0; l <= l_max; ++l) {
        b.block_off[l] = c;
        for (double r : b.roots[l]) b.norms[l].push_back(std::sqrt(2.0) / std::fabs(sph_jl(l + 1, r)));
        c += (int)b.roots[l].size() * (2 * l + 1);
    }
    b.coeffs = c;
    // quadrature plan (src/basis.cpp:177-189)
    b.n_theta = b.n_phi = 2 * l_max + 2;
    b.n_r = std::max(l_max + 1, (int)std::ceil(0.55 * lambda_cut) + 8);
    gauss_legendre(b.n_r, b.r, b.wr);
    for (int i = 0; i < b.n_r; ++i) {
        b.r[i] = 0.5 * (b.r[i] + 1.0);
        b.wr[i] *= 0.5;
    }
    gauss_legendre(b.n_theta, b.u, b.wu);
    return b;
}

// E[row][v] = sum over quadrature samples s touching voxel v of
//   w_tri(s, v) * radial(l,k,i_s) * Pbar_l^m(u_t) w_t * trig_part(m phi_p)
// with radial(l,k,i) = c_lk j_l(lambda_lk r_i) r_i^2 w_i 2pi/n_phi, trig = cos
// (Re) or -sin (Im): the composition of the four stages of expand()
// (src/basis.cpp:254-328), evaluated exactly in FP64.
Operator build_operator(const Basis& b, int n) {
    Operator op;
    op.n = n;
    op.rows = b.coeffs;
    const int L = b.l_max, nr = b.n_r, nt = b.n_theta, np = b.n_phi;
    const int nsamp = nr * nt * np;
    // 1. trilinear taps of every sample (volume.cpp:19-48 convention)
    struct Tap {
        int32_t voxel;
        int32_t sample;
        double w;
    };
    std::vector<Tap> taps;
    taps.reserve((size_t)nsamp * 8);
    for (int i = 0; i < nr; ++i)
        for (int t = 0; t < nt; ++t) {
            const double st = std::sqrt(std::max(0.0, 1.0 - b.u[t] * b.u[t]));
            const double rs = b.r[i] * st, z = b.r[i] * b.u[t];
            for (int p = 0; p < np; ++p) {
                const double phi = 2.0 * kPi * p / np;
                const double x = rs * std::cos(phi), y = rs * std::sin(phi);
                const double gx = x * (n / 2.0) + n / 2.0, gy = y * (n / 2.0) + n / 2.0,
                             gz = z * (n / 2.0) + n / 2.0;
                const int x0 = (int)std::floor(gx), y0 = (int)std::floor(gy), z0 = (int)std::floor(gz);
                const double fx = gx - x0, fy = gy - y0, fz = gz - z0;
                const int s = (i * nt + t) * np + p;
                for (int dz = 0; dz < 2; ++dz) {
                    const int zz = z0 + dz;
                    if (zz < 0 || zz >= n) continue;
                    const double wz = dz ? fz : 1.0 - fz;
                    for (int dy = 0; dy < 2; ++dy) {
                        const int yy = y0 + dy;
                        if (yy < 0 || yy >= n) continue;
                        const double wy = dy ? fy : 1.0 - fy;
                        for (int dx = 0; dx < 2; ++dx) {
                            const int xx = x0 + dx;
                            if (xx < 0 || xx >= n) continue;
                            const double w = (dx ? fx : 1.0 - fx) * wy * wz;
                            if (w == 0.0) continue;
                            taps.push_back({(int32_t)((zz * n + yy) * n + xx), s, w});
                        }
                    }
                }
            }
        }
    std::sort(taps.begin(), taps.end(), [](const Tap& a, const Tap& c) {
        return a.voxel != c.voxel ? a.voxel < c.voxel : a.sample < c.sample;
    });
    std::vector<int> start;
    for (size_t j = 0; j < taps.size(); ++j)
        if (j == 0 || taps[j].voxel != taps[j - 1].voxel) {
            op.voxels.push_back(taps[j].voxel);
            start.push_back((int)j);
        }
    start.push_back((int)taps.size());
    op.support = (int)op.voxels.size();

    // 2. separable factor tables
    const FactorTables ft = build_factor_tables(b);
    const std::vector<double>& ptab = ft.ptab;
    const std::vector<double>& cs = ft.cs;
    const std::vector<double>& sn = ft.sn;

    // 3. columns of E, 32 voxels per task; pass 0 finds the row maxima (power-of-two
    //    row scales), pass 1 recomputes and writes the FP16 hi/lo split
    op.m_pad = (op.rows + 127) / 128 * 128;
    op.k_pad = (op.support + 63) / 64 * 64;
    op.row_scale.assign(op.m_pad, 1.0f);
    op.hi.assign((size_t)op.m_pad * op.k_pad, 0);
    op.lo.assign((size_t)op.m_pad * op.k_pad, 0);
    std::vector<double> rmax(op.rows, 0.0);
    constexpr int VB = 32;
    const int nblk = (op.support + VB - 1) / VB;
    auto column = [&](int v, double* col) {
        std::fill(col, col + op.rows, 0.0);
        for (int j = start[v]; j < start[v + 1]; ++j) {
            const int s = taps[j].sample;
            const int i = s / (nt * np), t = (s / np) % nt, p = s % np;
            const double w = taps[j].w;
            for (int l = 0; l <= L; ++l) {
                const int nk = b.radial_count(l);
                if (!nk) continue;
                for (int m = 0; m <= l; ++m) {
                    const double pt = w * ptab[tri(l, m) * nt + t];
                    const double re = pt * cs[(size_t)m * np + p];
                    const double im = pt * sn[(size_t)m * np + p];
                    for (int k = 1; k <= nk; ++k) {
                        const double rad = ft.radial[(size_t)(ft.pair_off[l] + k - 1) * nr + i];
                        col[b.row(l, k, m, 0)] += rad * re;
                        if (m > 0) col[b.row(l, k, m, 1)] += rad * im;
                    }
                }
            }
        }
    };
    for (int pass = 0; pass < 2; ++pass) {
#pragma omp parallel
        {
            std::vector<double> tile((size_t)VB * op.rows);
            std::vector<double> lmax(pass == 0 ? op.rows : 0, 0.0);
#pragma omp for schedule(dynamic, 4)
            for (int blk = 0; blk < nblk; ++blk) {
                const int v0 = blk * VB, v1 = std::min(op.support, v0 + VB);
                for (int v = v0; v < v1; ++v) column(v, tile.data() + (size_t)(v - v0) * op.rows);
                if (pass == 0) {
                    for (int v = v0; v < v1; ++v)
                        for (int r = 0; r < op.rows; ++r)
                            lmax[r] = std::max(lmax[r], std::fabs(tile[(size_t)(v - v0) * op.rows + r]));
                } else {
                    for (int r = 0; r < op.rows; ++r) {
                        const double inv = 1.0 / op.row_scale[r];
                        for (int v = v0; v < v1; ++v) {
                            const double x = tile[(size_t)(v - v0) * op.rows + r] * inv;
                            const uint16_t h = half_bits(x);
                            op.hi[(size_t)r * op.k_pad + v] = h;
                            op.lo[(size_t)r * op.k_pad + v] = half_bits(x - half_value(h));
                        }
                    }
                }
            }
            if (pass == 0) {
#pragma omp critical
                for (int r = 0; r < op.rows; ++r) rmax[r] = std::max(rmax[r], lmax[r]);
            }
        }
        if (pass == 0)
            for (int r = 0; r < op.rows; ++r)
                op.row_scale[r] = rmax[r] > 0.0 ? (float)std::ldexp(1.0, (int)std::ceil(std::log2(rmax[r]))) : 1.0f;
    }
    return op;
}

FactorTables build_factor_tables(const Basis& b) {
    const int L = b.l_max, nr = b.n_r, nt = b.n_theta, np = b.n_phi;
    FactorTables f;
    f.pair_off.resize(L + 1);
    for (int l = 0; l <= L; ++l) {
        f.pair_off[l] = f.pairs;
        f.pairs += b.radial_count(l);
    }
    const double wphi = 2.0 * kPi / np;
    f.radial.resize((size_t)f.pairs * nr);
    for (int l = 0; l <= L; ++l)
        for (int k = 0; k < b.radial_count(l); ++k)
            for (int i = 0; i < nr; ++i)
                f.radial[(size_t)(f.pair_off[l] + k) * nr + i] =
                    b.norms[l][k] * sph_jl(l, b.roots[l][k] * b.r[i]) * b.r[i] * b.r[i] * b.wr[i] * wphi;
    f.ptab.resize(tri_count(L) * nt);
    std::vector<double> tab(tri_count(L));
    for (int t = 0; t < nt; ++t) {
        legendre(L, b.u[t], tab.data());
        for (size_t q = 0; q < tab.size(); ++q) f.ptab[q * nt + t] = tab[q] * b.wu[t];
    }
    f.cs.resize((size_t)(L + 1) * np);
    f.sn.resize((size_t)(L + 1) * np);
    for (int m = 0; m <= L; ++m)
        for (int p = 0; p < np; ++p) {
            const long long a = ((long long)m * p) % np;  // exact argument reduction
            f.cs[(size_t)m * np + p] = std::cos(2.0 * kPi * a / np);
            f.sn[(size_t)m * np + p] = -std::sin(2.0 * kPi * a / np);
        }
    return f;
}

int support_count(const Basis& b, int n) {
    std::vector<char> hit((size_t)n * n * n, 0);
    for (int i = 0; i < b.n_r; ++i)
        for (int t = 0; t < b.n_theta; ++t) {
            const double st = std::sqrt(std::max(0.0, 1.0 - b.u[t] * b.u[t]));
            const double rs = b.r[i] * st, z = b.r[i] * b.u[t];
            for (int p = 0; p < b.n_phi; ++p) {
                const double phi = 2.0 * kPi * p / b.n_phi;
                const double g[3] = {rs * std::cos(phi) * (n / 2.0) + n / 2.0, rs * std::sin(phi) * (n / 2.0) + n / 2.0,
                                     z * (n / 2.0) + n / 2.0};
                int c0[3];
                double fr[3];
                for (int a = 0; a < 3; ++a) {
                    c0[a] = (int)std::floor(g[a]);
                    fr[a] = g[a] - c0[a];
                }
                for (int dz = 0; dz < 2; ++dz)
                    for (int dy = 0; dy < 2; ++dy)
                        for (int dx = 0; dx < 2; ++dx) {
                            const int xx = c0[0] + dx, yy = c0[1] + dy, zz = c0[2] + dz;
                            if (xx < 0 || xx >= n || yy < 0 || yy >= n || zz < 0 || zz >= n) continue;
                            const double w = (dx ? fr[0] : 1.0 - fr[0]) * (dy ? fr[1] : 1.0 - fr[1]) *
                                             (dz ? fr[2] : 1.0 - fr[2]);
                            if (w != 0.0) hit[((size_t)zz * n + yy) * n + xx] = 1;
                        }
            }
        }
    int c = 0;
    for (char h : hit) c += h;
    return c;
}

uint16_t half_bits(double x) {
    uint16_t sign = 0;
    if (std::signbit(x)) {
        sign = 0x8000;
        x = -x;
    }
    if (x == 0.0) return sign;
    if (x >= 65520.0) return sign | 0x7C00;  // overflow -> inf
    int e;
    std::frexp(x, &e);                        // x = f * 2^e, f in [0.5, 1)
    int exp = e - 1;                          // x = 1.xxx * 2^exp
    if (exp < -14) {                          // subnormal: multiples of 2^-24
        const double q = std::nearbyint(x * 16777216.0);  // RNE (default rounding mode)
        return sign | (uint16_t)q;           // q == 1024 rolls into the smallest normal
    }
    double mant = std::nearbyint((x / std::ldexp(1.0, exp) - 1.0) * 1024.0);
    if (mant >= 1024.0) {
        mant = 0.0;
        ++exp;
        if (exp > 15) return sign | 0x7C00;
    }
    return sign | (uint16_t)((exp + 15) << 10) | (uint16_t)mant;
}

double half_value(uint16_t h) {
    const double s = (h & 0x8000) ? -1.0 : 1.0;
    const int e = (h >> 10) & 0x1F, m = h & 0x3FF;
    if (e == 0) return s * std::ldexp((double)m, -24);
    if (e == 31) return s * INFINITY;
    return s * std::ldexp(1.0 + m / 1024.0, e - 15);
}

}  // namespace host
}  // namespace bmb
