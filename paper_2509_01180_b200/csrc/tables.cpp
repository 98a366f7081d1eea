// Host builders for the per-band device tables (see kernels.cuh BandTables).
#include "tables.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace bmb {

namespace {

double sqrt_binom(int n, int k) {  // sqrt(C(n, k)) (src/steer.cpp:34-39)
    double r = 1.0;
    for (int i = 1; i <= k; ++i) r *= (double)(n - k + i) / i;
    return std::sqrt(r);
}

// closed-form border of the recursion at degree l0 = max(|m|,|m'|):
// d^{l0}_{m,m'} = fac * cos(b/2)^a sin(b/2)^p  (src/steer.cpp:109-128)
void border(int m, int mp, double& fac, int& a, int& p) {
    const int l = std::max(std::abs(m), std::abs(mp));
    if (l == 0) {
        fac = 1.0;
        a = p = 0;
        return;
    }
    if (m == l) {  // top row
        fac = (((l - mp) % 2) ? -1.0 : 1.0) * sqrt_binom(2 * l, l + mp);
        a = l + mp;
        p = l - mp;
    } else if (m == -l) {  // bottom row
        fac = sqrt_binom(2 * l, l + mp);
        a = l - mp;
        p = l + mp;
    } else if (mp == l) {  // right column
        fac = sqrt_binom(2 * l, l + m);
        a = l + m;
        p = l - m;
    } else {  // left column, mp == -l
        fac = (((l + m) % 2) ? -1.0 : 1.0) * sqrt_binom(2 * l, l + m);
        a = l - m;
        p = l + m;
    }
}

}  // namespace

BandTablesHost build_band_tables(int L) {
    if (L < 0 || L > kMaxL) throw std::invalid_argument("band limit out of range");
    BandTablesHost t;
    t.L = L;
    struct It {
        int m, mp;
    };
    std::vector<It> items;  // sorted by l0 = m, then m'
    for (int m = 0; m <= L; ++m)
        for (int mp = -m; mp <= m; ++mp) items.push_back({m, mp});
    t.n_items = (int)items.size();
    t.n_groups = (t.n_items + 31) / 32;
    const int slots = t.n_groups * 32;
    t.item_mm.assign(slots, char2{0, 0});
    t.item_pm.assign(slots, char2{0, 0});
    t.item_w.assign(slots, float2{0.0f, 0.0f});
    t.item_len.assign(slots, 0);
    t.bfac.assign(slots, 0.0f);
    t.bexp.assign(slots, 0);
    t.row_off.assign(t.n_groups + 1, 0);
    for (int g = 0; g < t.n_groups; ++g) {
        int glen = 0;
        for (int j = 0; j < 32 && g * 32 + j < t.n_items; ++j) glen = std::max(glen, L - items[g * 32 + j].m + 1);
        t.row_off[g + 1] = t.row_off[g] + glen;
    }
    t.rows = t.row_off[t.n_groups];
    t.P.assign((size_t)t.rows * 32, 0.0f);
    t.Q.assign((size_t)t.rows * 32, 0.0f);
    t.R.assign((size_t)t.rows * 32, 0.0f);
    t.item_of.assign((size_t)(2 * L + 1) * (2 * L + 1), -1);
    t.out_pos.assign((size_t)(2 * L + 1) * (2 * L + 1), 0);
    t.at_desc.assign((size_t)t.rows * 32, int2{0, 0});
    for (int i = 0; i < t.n_items; ++i) {
        const It& it = items[i];
        const int g = i / 32, j = i % 32;
        const int m = it.m, mp = it.mp;
        // partner in the half plane: swap (m', m) with sign (-1)^(m-m') for m' >= 0,
        // anti-swap (-m', -m) with sign +1 for m' < 0 (d^l_{m'm} = (-1)^(m-m') d^l_{mm'},
        // d^l_{-m',-m} = d^l_{mm'}, src/steer.cpp:43-144)
        const int pa = mp >= 0 ? mp : -mp, pb = mp >= 0 ? m : -m;
        const double sg = mp >= 0 ? (((m - mp) & 1) ? -1.0 : 1.0) : 1.0;
        const bool self = pa == m && pb == mp;
        t.item_mm[i] = char2{(signed char)m, (signed char)mp};
        t.item_pm[i] = char2{(signed char)pa, (signed char)pb};
        t.item_w[i] = float2{(m == 0 && mp == 0) ? 1.0f : 2.0f, self ? 0.0f : (float)(2.0 * sg)};
        t.item_len[i] = L - m + 1;
        double fac;
        int a, p;
        border(m, mp, fac, a, p);
        t.bfac[i] = (float)fac;
        t.bexp[i] = a | (p << 8);
        t.item_of[(size_t)(m + L) * (2 * L + 1) + (mp + L)] = 2 * i;
        if (!self) t.item_of[(size_t)(pa + L) * (2 * L + 1) + (pb + L)] = 2 * i + 1;
        for (int st = 0; st <= L - m; ++st) {
            const int l = m + st;
            int2 dsc;
            dsc.x = 1 | (self ? 0 : 2) | (l << 2) | ((m + 64) << 8) | ((mp + 64) << 16);
            dsc.y = (pa + 64) | ((pb + 64) << 8);
            t.at_desc[(size_t)(t.row_off[g] + st) * 32 + j] = dsc;
        }
        {
            const int p0 = 2 * ((t.row_off[g] - m) * 32 + j);
            t.out_pos[(size_t)(m + L) * (2 * L + 1) + (mp + L)] = p0;
            if (!self) t.out_pos[(size_t)(pa + L) * (2 * L + 1) + (pb + L)] = p0 + 1;
        }
        for (int s = 1; s <= L - m; ++s) {
            const int l = m + s;
            const size_t at = (size_t)(t.row_off[g] + s) * 32 + j;
            if (m == 0 && l == 1) {  // d^1_00 = cos b (steer.cpp:130-133)
                t.P[at] = 1.0f;
                continue;
            }
            // steer.cpp:101-141: t1 = P cos b + Q, t2 = R (symmetric in m <-> m' and under m,m' -> -m',-m)
            const double dm = m, dmp = mp;
            const double a2 = std::sqrt(((double)l * l - dm * dm) * ((double)l * l - dmp * dmp));
            const bool has2 = std::abs(m) <= l - 2 && std::abs(mp) <= l - 2;
            const double b2 = has2 ? std::sqrt(((double)(l - 1) * (l - 1) - dm * dm) *
                                               ((double)(l - 1) * (l - 1) - dmp * dmp))
                                   : 0.0;
            t.P[at] = (float)((2.0 * l - 1.0) * l / a2);
            t.Q[at] = (float)(-(2.0 * l - 1.0) * dm * dmp / ((l - 1.0) * a2));
            t.R[at] = (float)(l * b2 / ((l - 1.0) * a2));
        }
    }
    return t;
}

std::vector<float4> wedge_band_entries(const BandTablesHost& t,
                                       const std::vector<std::complex<double>>& chi,
                                       const std::vector<std::complex<double>>& q, double total) {
    std::vector<float4> w((size_t)t.rows * 32, float4{0.0f, 0.0f, 0.0f, 0.0f});
    auto coef = [](const std::vector<std::complex<double>>& hat, int l, int m) {
        if (m >= 0) return hat[host::tri(l, m)];
        const std::complex<double> c = std::conj(hat[host::tri(l, -m)]);
        return ((-m) % 2) ? -c : c;
    };
    for (int i = 0; i < t.n_items; ++i) {
        const int m = t.item_mm[i].x, mp = t.item_mm[i].y;
        const int pa = t.item_pm[i].x, pb = t.item_pm[i].y;
        const bool self = t.item_w[i].y == 0.0f;
        const int g = i / 32, j = i % 32;
        for (int l = m; l <= t.L; ++l) {
            const std::complex<double> va = std::conj(coef(chi, l, m)) * coef(q, l, mp) / total;
            const std::complex<double> vb =
                self ? std::complex<double>(0.0, 0.0) : std::conj(coef(chi, l, pa)) * coef(q, l, pb) / total;
            w[(size_t)(t.row_off[g] + l - m) * 32 + j] =
                float4{(float)va.real(), (float)va.imag(), (float)vb.real(), (float)vb.imag()};
        }
    }
    return w;
}

std::vector<double> little_d_full(int L, double beta) {
    std::vector<size_t> off(L + 2, 0);
    for (int l = 0; l <= L; ++l) off[l + 1] = off[l] + (size_t)(2 * l + 1) * (2 * l + 1);
    std::vector<double> d(off[L + 1], 0.0);
    const double cb = std::cos(beta), ch = std::cos(0.5 * beta), sh = std::sin(0.5 * beta);
    auto at = [&](int l, int m, int mp) -> double& {
        return d[off[l] + (size_t)(m + l) * (2 * l + 1) + (mp + l)];
    };
    auto ipow = [](double x, int e) {
        double r = 1.0;
        for (int i = 0; i < e; ++i) r *= x;
        return r;
    };
    at(0, 0, 0) = 1.0;
    for (int l = 1; l <= L; ++l) {
        for (int m = -l; m <= l; ++m)
            for (int mp = -l; mp <= l; ++mp) {
                if (std::abs(m) != l && std::abs(mp) != l) continue;
                double fac;
                int a, p;
                border(m, mp, fac, a, p);
                at(l, m, mp) = fac * (ipow(ch, a) * ipow(sh, p));
            }
        if (l == 1) {
            at(1, 0, 0) = cb;
            continue;
        }
        for (int m = -(l - 1); m <= l - 1; ++m)
            for (int mp = -(l - 1); mp <= l - 1; ++mp) {
                const double a2 = std::sqrt(((double)l * l - (double)m * m) * ((double)l * l - (double)mp * mp));
                const double den = (l - 1.0) * a2;
                const double t1 = (2.0 * l - 1.0) * (l * (l - 1.0) * cb - (double)m * mp) / den;
                const bool has2 = std::abs(m) <= l - 2 && std::abs(mp) <= l - 2;
                const double b2 = has2 ? std::sqrt(((double)(l - 1) * (l - 1) - (double)m * m) *
                                                   ((double)(l - 1) * (l - 1) - (double)mp * mp))
                                       : 0.0;
                const double t2 = l * b2 / den;
                at(l, m, mp) = t1 * at(l - 1, m, mp) - (has2 ? t2 * at(l - 2, m, mp) : 0.0);
            }
    }
    return d;
}

std::vector<std::complex<double>> wigner_D_blocks(int L, double alpha, double beta, double gamma) {
    const std::vector<double> d = little_d_full(L, beta);
    std::vector<std::complex<double>> D(d.size());
    size_t off = 0;
    for (int l = 0; l <= L; ++l) {
        const int w = 2 * l + 1;
        for (int m = -l; m <= l; ++m)
            for (int mp = -l; mp <= l; ++mp) {
                const size_t i = off + (size_t)(m + l) * w + (mp + l);
                D[i] = std::polar(1.0, -(m * alpha + mp * gamma)) * d[i];
            }
        off += (size_t)w * w;
    }
    return D;
}

namespace {
std::complex<double> packed_value(const float* row, int m) {
    const int am = m < 0 ? -m : m;
    std::complex<double> z = am == 0 ? std::complex<double>(row[0], 0.0)
                                     : std::complex<double>(row[2 * am - 1], row[2 * am]);
    if (m < 0) z = ((am & 1) ? -1.0 : 1.0) * std::conj(z);  // f_{-m} = (-1)^m conj f_m
    return z;
}
}  // namespace

std::vector<float> rotate_real_packed(const std::vector<float>& f, const host::Basis& b,
                                      const std::vector<std::complex<double>>& D) {
    std::vector<float> out(f.size(), 0.0f);
    size_t off = 0;
    for (int l = 0; l <= b.l_max; ++l) {
        const int w = 2 * l + 1;
        for (int k = 0; k < b.radial_count(l); ++k) {
            const float* row = f.data() + b.block_off[l] + (size_t)k * w;
            float* o = out.data() + b.block_off[l] + (size_t)k * w;
            for (int n = 0; n <= l; ++n) {
                std::complex<double> acc = 0.0;
                for (int m = -l; m <= l; ++m) acc += D[off + (size_t)(n + l) * w + (m + l)] * packed_value(row, m);
                if (n == 0) {
                    o[0] = (float)acc.real();
                } else {
                    o[2 * n - 1] = (float)acc.real();
                    o[2 * n] = (float)acc.imag();
                }
            }
        }
        off += (size_t)w * w;
    }
    return out;
}

std::vector<std::complex<double>> rotate_tri(const std::vector<std::complex<double>>& q, int L,
                                             const std::vector<std::complex<double>>& D) {
    std::vector<std::complex<double>> out(q.size(), 0.0);
    auto coef = [&](int l, int m) {
        if (m >= 0) return q[host::tri(l, m)];
        const std::complex<double> c = std::conj(q[host::tri(l, -m)]);
        return ((-m) % 2) ? -c : c;
    };
    size_t off = 0;
    for (int l = 0; l <= L; ++l) {
        const int w = 2 * l + 1;
        for (int n = 0; n <= l; ++n) {
            std::complex<double> acc = 0.0;
            for (int m = -l; m <= l; ++m) acc += D[off + (size_t)(n + l) * w + (m + l)] * coef(l, m);
            out[host::tri(l, n)] = acc;
        }
        off += (size_t)w * w;
    }
    return out;
}

}  // namespace bmb
