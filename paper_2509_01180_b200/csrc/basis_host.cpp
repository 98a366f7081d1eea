// Host FP64 basis setup (once per context).  See basis_host.hpp.
#include "basis_host.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace bmb {
namespace host {

// ---------------------------------------------------------------- Bessel
// Spherical Bessel functions and their zeros, written from the definitions:
//   j_0(x) = sin x / x,  j_1(x) = sin x / x^2 - cos x / x,
//   j_{l+1}(x) = (2l+1)/x j_l(x) - j_{l-1}(x)          (forward-stable for x > l;
//                                                        run in long double),
//   j_l(x) = x^l / (2l+1)!! sum_k (-x^2/2)^k / (k! prod_{i=1..k} (2l+2i+1))
//                                                        (power series, x <= l).
// The zeros lambda_lk are found by a sign-change scan (consecutive zeros of j_l
// are more than pi apart) and polished with Newton steps on
// j_l'(x) = j_{l-1}(x) - (l+1)/x j_l(x).  Zeros of j_0 are k pi exactly.

namespace {

// power series in long double (x <= l: the terms first grow, then alternate
// and decay; the 64-bit mantissa absorbs the cancellation)
double jl_series(int l, double xd) {
    const long double x = xd, h = -0.5L * x * x;
    long double lead = 1.0L;
    for (int i = 1; i <= l; ++i) lead *= x / (long double)(2 * i + 1);
    long double term = 1.0L, sum = 1.0L;
    for (int k = 1; k < 400; ++k) {
        term *= h / ((long double)k * (long double)(2 * l + 2 * k + 1));
        sum += term;
        if (std::fabs((double)term) <= 1e-21 * std::fabs((double)sum)) break;
    }
    return (double)(lead * sum);
}

// j_l'(x)
double djl_dx(int l, double x) {
    if (l == 0) return -sph_jl(1, x);
    return sph_jl(l - 1, x) - (l + 1.0) / x * sph_jl(l, x);
}

// the zero of j_l in (a, b), where j_l changes sign exactly once
double polish_zero(int l, double a, double b) {
    double fa = sph_jl(l, a);
    for (int it = 0; it < 60 && b - a > 1e-6 * b; ++it) {  // bisect to a Newton-safe bracket
        const double c = 0.5 * (a + b), fc = sph_jl(l, c);
        if ((fc < 0.0) == (fa < 0.0)) {
            a = c;
            fa = fc;
        } else {
            b = c;
        }
    }
    double x = 0.5 * (a + b);
    for (int it = 0; it < 50; ++it) {
        const double dx = sph_jl(l, x) / djl_dx(l, x);
        const double nx = std::min(std::max(x - dx, a), b);
        if (std::fabs(nx - x) <= 4e-16 * x) return nx;
        x = nx;
    }
    return x;
}

}  // namespace

double sph_jl(int l, double x) {
    if (x < 0.0) return ((l & 1) ? -1.0 : 1.0) * sph_jl(l, -x);  // parity of j_l
    if (x <= (double)l || x < 0.5) return jl_series(l, x);
    // forward recurrence in long double: just above the turning point x ~ l it
    // amplifies rounding by ~10^3, which the 64-bit mantissa keeps below 1e-16
    const long double xl = x;
    long double prev = std::sin(xl) / xl;  // j_0
    if (l == 0) return (double)prev;
    long double cur = prev / xl - std::cos(xl) / xl;  // j_1
    for (int n = 1; n < l; ++n) {
        const long double next = (2.0L * n + 1.0L) / xl * cur - prev;
        prev = cur;
        cur = next;
    }
    return (double)cur;
}

std::vector<std::vector<double>> bessel_roots(int l_max, double cut) {
    std::vector<std::vector<double>> rows(l_max + 1);
    for (double z = kPi, k = 1.0; z <= cut; k += 1.0, z = k * kPi) rows[0].push_back(z);
    const double h = 0.25;  // scan step (< pi, the least zero spacing)
    for (int l = 1; l <= l_max; ++l) {
        // no zero of j_l lies below l (j_l > 0 there)
        double a = std::max(0.5, (double)l), fa = sph_jl(l, a);
        while (a < cut) {
            const double b = std::min(a + h, cut), fb = sph_jl(l, b);
            if (fb == 0.0) {
                rows[l].push_back(b);
                a = b + 1e-9 * b;
                fa = sph_jl(l, a);
                continue;
            }
            if ((fa < 0.0) != (fb < 0.0)) rows[l].push_back(polish_zero(l, a, b));
            a = b;
            fa = fb;
        }
        while (!rows[l].empty() && rows[l].back() > cut) rows[l].pop_back();
    }
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

// Nyquist cut pi n / 2, lowered (to a root of the table) when the basis would
// exceed n^3 / 4 coefficients: the largest cut whose coefficient count -- every
// root lambda_lk <= cut weighs 2l + 1 -- stays within n^3 / 4, pi if none does
// (default_lambda_cut semantics, src/basis.cpp:117-138).
double default_lambda_cut(int n, int l_max) {
    const double nyquist = kPi * n / 2.0;
    const long long budget = (long long)n * n * n / 4;
    std::vector<std::pair<double, int>> zeros;  // (lambda, weight 2l + 1)
    const auto table = bessel_roots(l_max, nyquist);
    for (int l = 0; l <= l_max; ++l)
        for (double z : table[l]) zeros.push_back({z, 2 * l + 1});
    std::sort(zeros.begin(), zeros.end());
    long long used = 0;
    for (const auto& z : zeros) used += z.second;
    if (used <= budget) return nyquist;
    double cut = kPi;
    used = 0;
    for (size_t i = 0; i < zeros.size() && used + zeros[i].second <= budget; ++i) {
        used += zeros[i].second;
        cut = zeros[i].first;
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
