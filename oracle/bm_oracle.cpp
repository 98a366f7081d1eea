// bm_oracle — CPU restatement of the reference hot path (see bm_oracle.hpp).
// TEST INFRASTRUCTURE ONLY (checker + CPU baseline); never linked by the product.
#include "bm_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace bmo {

// ======================================================================= philox
// include/ballmatch/philox.hpp:17-29
std::array<uint32_t, 4> Philox::round10(std::array<uint32_t, 4> ctr, std::array<uint32_t, 2> key) {
    for (int i = 0; i < 10; ++i) {
        const uint64_t p0 = uint64_t{0xD2511F53u} * ctr[0];
        const uint64_t p1 = uint64_t{0xCD9E8D57u} * ctr[2];
        ctr = {static_cast<uint32_t>(p1 >> 32) ^ ctr[1] ^ key[0], static_cast<uint32_t>(p1),
               static_cast<uint32_t>(p0 >> 32) ^ ctr[3] ^ key[1], static_cast<uint32_t>(p0)};
        key[0] += 0x9E3779B9u;
        key[1] += 0xBB67AE85u;
    }
    return ctr;
}

// philox.hpp:34-87
PhiloxStream::PhiloxStream(uint64_t seed, uint32_t stream)
    : key_{static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)}, stream_(stream) {}

uint32_t PhiloxStream::next_u32() {
    if (lane_ == 4) {
        block_ = Philox::round10({ctr_, 0, stream_, 0}, key_);
        ++ctr_;
        lane_ = 0;
    }
    return block_[lane_++];
}
double PhiloxStream::next_unit() { return (static_cast<double>(next_u32()) + 1.0) * 0x1p-32; }
double PhiloxStream::next_uniform(double lo, double hi) { return lo + (hi - lo) * next_unit(); }
double PhiloxStream::next_gaussian() {  // philox.hpp:60-72 (Box-Muller)
    if (have_spare_) {
        have_spare_ = false;
        return spare_;
    }
    const double u1 = next_unit();
    const double u2 = next_unit();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * kPi * u2;
    spare_ = r * std::sin(a);
    have_spare_ = true;
    return r * std::cos(a);
}
int PhiloxStream::next_int(int lo, int hi) {  // philox.hpp:74-77
    const auto span = static_cast<uint64_t>(hi - lo + 1);
    return lo + static_cast<int>((static_cast<uint64_t>(next_u32()) * span) >> 32);
}

// ======================================================================= rotation
// src/rotation.cpp:13-21 (normalizing constructor)
Rot Rot::make(double w, double x, double y, double z) {
    const double n = std::sqrt(w * w + x * x + y * y + z * z);
    if (!(n > 0.0) || !std::isfinite(n))
        throw std::invalid_argument("Rotation: quaternion must be nonzero and finite");
    return Rot{w / n, x / n, y / n, z / n};
}
// rotation.cpp:23-29
Rot Rot::from_axis_angle(Vec3 axis, double angle) {
    const double n = std::sqrt(axis[0] * axis[0] + axis[1] * axis[1] + axis[2] * axis[2]);
    if (!(n > 0.0)) throw std::invalid_argument("Rotation: axis must be nonzero");
    const double h = 0.5 * angle;
    const double s = std::sin(h) / n;
    return make(std::cos(h), axis[0] * s, axis[1] * s, axis[2] * s);
}
// rotation.cpp:31-34
Rot Rot::from_euler_zyz(double a, double b, double g) {
    return from_axis_angle({0, 0, 1}, a) * from_axis_angle({0, 1, 0}, b) *
           from_axis_angle({0, 0, 1}, g);
}
// rotation.cpp:68-75
Mat3 Rot::matrix() const {
    return {1 - 2 * (y * y + z * z), 2 * (x * y - w * z),     2 * (x * z + w * y),
            2 * (x * y + w * z),     1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
            2 * (x * z - w * y),     2 * (y * z + w * x),     1 - 2 * (x * x + y * y)};
}
// rotation.cpp:77-93
Euler Rot::euler_zyz() const {
    const Mat3 m = matrix();
    Euler e;
    const double sb = std::hypot(m[2], m[5]);
    e.beta = std::atan2(sb, m[8]);
    if (sb > 1e-12) {
        e.alpha = std::atan2(m[5], m[2]);
        e.gamma = std::atan2(m[7], -m[6]);
    } else if (m[8] > 0.0) {
        e.alpha = std::atan2(m[3], m[0]);
        e.gamma = 0.0;
    } else {
        e.alpha = std::atan2(-m[3], -m[0]);
        e.gamma = 0.0;
    }
    return e;
}
// rotation.cpp:95-100 (unchecked product)
Rot Rot::operator*(const Rot& r) const {
    return Rot{w * r.w - x * r.x - y * r.y - z * r.z, w * r.x + x * r.w + y * r.z - z * r.y,
               w * r.y - x * r.z + y * r.w + z * r.x, w * r.z + x * r.y - y * r.x + z * r.w};
}
// rotation.cpp:102-107
double Rot::angle_to(const Rot& o) const {
    const Rot r = inverse() * o;
    const double v = std::sqrt(r.x * r.x + r.y * r.y + r.z * r.z);
    return 2.0 * std::atan2(v, std::abs(r.w));
}
double geodesic_degrees(const Rot& a, const Rot& b) { return a.angle_to(b) * 180.0 / kPi; }

// ======================================================================= volume
double volume_l2_norm(const Volume& v) {  // volume.cpp:7-11
    double s = 0.0;
    for (double x : v.d) s += x * x;
    return std::sqrt(s);
}
// volume.cpp:19-48
double sample_trilinear(const Volume& v, double x, double y, double z) {
    const int n = v.n;
    const double u = x * (n / 2.0) + n / 2.0;
    const double w = y * (n / 2.0) + n / 2.0;
    const double q = z * (n / 2.0) + n / 2.0;
    const int i0 = static_cast<int>(std::floor(u));
    const int j0 = static_cast<int>(std::floor(w));
    const int k0 = static_cast<int>(std::floor(q));
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
                const double wx = dx ? fx : 1.0 - fx;
                acc += wx * wy * wz * v.at(i, j, k);
            }
        }
    }
    return acc;
}
// volume.cpp:50-67
Volume shift_volume(const Volume& v, const std::array<int, 3>& s) {
    Volume out(v.n);
    const int n = v.n;
    for (int z = 0; z < n; ++z) {
        const int sz = z + s[2];
        if (sz < 0 || sz >= n) continue;
        for (int y = 0; y < n; ++y) {
            const int sy = y + s[1];
            if (sy < 0 || sy >= n) continue;
            for (int x = 0; x < n; ++x) {
                const int sx = x + s[0];
                if (sx < 0 || sx >= n) continue;
                out.at(x, y, z) = v.at(sx, sy, sz);
            }
        }
    }
    return out;
}

// ======================================================================= bessel
// src/detail/bessel.cpp
namespace {
double jl_small_x(int l, double x) {  // bessel.cpp:13-18
    double v = 1.0;
    for (int i = 1; i <= l; ++i) v *= x / (2 * i + 1);
    return v * (1.0 - x * x / (2.0 * (2 * l + 3)));
}
double jl_downward(int l, double x) {  // bessel.cpp:21-38 (Miller)
    const int start = l + 20 + static_cast<int>(std::sqrt(40.0 * l + 100.0));
    double jp = 0.0, jn = 1e-290, jl_val = 0.0;
    for (int n = start; n >= 1; --n) {
        const double jm = (2.0 * n + 1.0) / x * jn - jp;
        jp = jn;
        jn = jm;
        if (n - 1 == l) jl_val = jn;
        if (std::abs(jn) > 1e270) {
            jn *= 1e-290;
            jp *= 1e-290;
            jl_val *= 1e-290;
        }
    }
    return jl_val * ((std::sin(x) / x) / jn);
}
double mcmahon_zero(int l, int k) {  // bessel.cpp:41-47
    const double nu = l + 0.5;
    const double mu = 4.0 * nu * nu;
    const double b = (k + 0.5 * nu - 0.25) * kPi;
    const double b8 = 8.0 * b;
    return b - (mu - 1.0) / b8 - 4.0 * (mu - 1.0) * (7.0 * mu - 31.0) / (3.0 * b8 * b8 * b8);
}
double refine_root(int l, double lo, double hi, double seed) {  // bessel.cpp:51-70
    double flo = sph_jl(l, lo);
    double x = (seed > lo && seed < hi) ? seed : 0.5 * (lo + hi);
    for (int it = 0; it < 200; ++it) {
        const double f = sph_jl(l, x);
        if ((f > 0) == (flo > 0)) {
            lo = x;
            flo = f;
        } else {
            hi = x;
        }
        if (std::abs(f) < 1e-14 && (hi - lo) < 1e-12 * x) return x;
        const double fp = sph_jl_prime(l, x);
        double next = (fp != 0.0) ? x - f / fp : 0.5 * (lo + hi);
        if (!(next > lo) || !(next < hi)) next = 0.5 * (lo + hi);
        if (next == x) return x;
        x = next;
    }
    return x;
}
}  // namespace

double sph_jl(int l, double x) {  // bessel.cpp:74-91
    if (x < 0.0) return (l % 2 ? -1.0 : 1.0) * sph_jl(l, -x);
    if (x < 1e-6) return l == 0 ? 1.0 - x * x / 6.0 : jl_small_x(l, x);
    if (l == 0) return std::sin(x) / x;
    const double j0 = std::sin(x) / x;
    const double j1 = j0 / x - std::cos(x) / x;
    if (l == 1) return j1;
    if (x > l + 0.5) {
        double jm = j0, jn = j1;
        for (int n = 1; n < l; ++n) {
            const double jp = (2.0 * n + 1.0) / x * jn - jm;
            jm = jn;
            jn = jp;
        }
        return jn;
    }
    return jl_downward(l, x);
}
double sph_jl_prime(int l, double x) {  // bessel.cpp:126-130
    if (l == 0) return -sph_jl(1, x);
    if (x < 1e-12) return l == 1 ? 1.0 / 3.0 : 0.0;
    return sph_jl(l - 1, x) - (l + 1.0) / x * sph_jl(l, x);
}
double bessel_root(int l, int k) {  // bessel.cpp:132-148
    if (l < 0) throw std::invalid_argument("bessel_root: degree l must be >= 0");
    if (k < 1) throw std::invalid_argument("bessel_root: root index k must be >= 1");
    if (l == 0) return k * kPi;
    std::vector<double> prev((size_t)(k + l));
    for (int i = 1; i <= k + l; ++i) prev[i - 1] = i * kPi;
    for (int ll = 1; ll <= l; ++ll) {
        const int count = k + (l - ll);
        std::vector<double> cur(count);
        for (int i = 0; i < count; ++i)
            cur[i] = refine_root(ll, prev[i], prev[i + 1], mcmahon_zero(ll, i + 1));
        prev = std::move(cur);
    }
    return prev[k - 1];
}
std::vector<std::vector<double>> bessel_root_table(int l_max, double lambda_cut) {  // :150-178
    std::vector<std::vector<double>> rows(l_max + 1);
    std::vector<double> prev;
    {
        int beyond = 0;
        for (int k = 1; beyond < l_max + 2; ++k) {
            prev.push_back(k * kPi);
            if (prev.back() > lambda_cut) ++beyond;
        }
    }
    rows[0] = prev;
    for (int l = 1; l <= l_max; ++l) {
        std::vector<double> cur;
        int beyond = 0;
        for (size_t i = 0; i + 1 < prev.size() && beyond < l_max + 2 - l; ++i) {
            cur.push_back(refine_root(l, prev[i], prev[i + 1], mcmahon_zero(l, (int)i + 1)));
            if (cur.back() > lambda_cut) ++beyond;
        }
        rows[l] = cur;
        prev = std::move(cur);
    }
    for (auto& row : rows)
        while (!row.empty() && row.back() > lambda_cut) row.pop_back();
    return rows;
}

// ======================================================================= quadrature
// src/detail/quadrature.hpp:16-42
GL gauss_legendre(int n) {
    GL gl;
    gl.nodes.resize(n);
    gl.weights.resize(n);
    for (int i = 0; i < (n + 1) / 2; ++i) {
        double x = std::cos(kPi * (i + 0.75) / (n + 0.5));
        double pp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = x;
            for (int j = 2; j <= n; ++j) {
                const double p2 = ((2 * j - 1) * x * p1 - (j - 1) * p0) / j;
                p0 = p1;
                p1 = p2;
            }
            pp = n * (x * p1 - p0) / (x * x - 1.0);
            const double dx = p1 / pp;
            x -= dx;
            if (std::abs(dx) < 1e-15) break;
        }
        const double w = 2.0 / ((1.0 - x * x) * pp * pp);
        gl.nodes[i] = -x;
        gl.nodes[n - 1 - i] = x;
        gl.weights[i] = w;
        gl.weights[n - 1 - i] = w;
    }
    return gl;
}
GL gauss_legendre01(int n) {  // quadrature.hpp:45-52
    GL gl = gauss_legendre(n);
    for (int i = 0; i < n; ++i) {
        gl.nodes[i] = 0.5 * (gl.nodes[i] + 1.0);
        gl.weights[i] *= 0.5;
    }
    return gl;
}
// quadrature.hpp:65-85
void legendre_table(int l_max, double u, double* out) {
    const double s = std::sqrt(std::max(0.0, 1.0 - u * u));
    constexpr double inv_sqrt4pi = 0.28209479177387814;
    out[tri_index(0, 0)] = inv_sqrt4pi;
    for (int m = 1; m <= l_max; ++m)
        out[tri_index(m, m)] = -std::sqrt((2.0 * m + 1.0) / (2.0 * m)) * s * out[tri_index(m - 1, m - 1)];
    for (int m = 0; m < l_max; ++m)
        out[tri_index(m + 1, m)] = std::sqrt(2.0 * m + 3.0) * u * out[tri_index(m, m)];
    for (int m = 0; m <= l_max; ++m) {
        for (int l = m + 2; l <= l_max; ++l) {
            const double a = std::sqrt((4.0 * l * l - 1.0) /
                                       (static_cast<double>(l) * l - static_cast<double>(m) * m));
            const double b = std::sqrt(
                (static_cast<double>(l - 1) * (l - 1) - static_cast<double>(m) * m) /
                (4.0 * static_cast<double>(l - 1) * (l - 1) - 1.0));
            out[tri_index(l, m)] = a * (u * out[tri_index(l - 1, m)] - b * out[tri_index(l - 2, m)]);
        }
    }
}

// ======================================================================= FFT
// Replaces FFTW (src/detail/fftw_util.cpp:58-73): unnormalized DFTs with the
// FFTW sign/index conventions.  Mixed-radix (2,3,5) recursive complex FFT with
// exact-argument twiddles; other factors fall back to a direct DFT.
namespace {
cd unit_root(long long num, long long den, int sign) {
    // exp(sign * 2 pi i num/den) with the argument reduced modulo den
    long long r = ((num % den) + den) % den;
    const double a = 2.0 * kPi * (double)r / (double)den;
    return {std::cos(a), sign * std::sin(a)};
}
void fft_rec(const cd* in, cd* out, int n, int stride, const std::vector<cd>& tw, int tw_n) {
    // decimation in time: x_q[j] = in[(j p + q) stride]; X[k' + r m] = sum_q W_n^{q (k' + r m)} Y_q[k']
    if (n == 1) {
        out[0] = in[0];
        return;
    }
    const size_t tstep = (size_t)(tw_n / n);
    int p = 0;
    for (int f : {2, 3, 5})
        if (n % f == 0) {
            p = f;
            break;
        }
    if (p == 0) {  // direct DFT for other prime factors
        for (int k = 0; k < n; ++k) {
            cd acc = 0;
            for (int j = 0; j < n; ++j) acc += in[(size_t)j * stride] * tw[(size_t)(((long long)j * k) % n) * tstep];
            out[k] = acc;
        }
        return;
    }
    const int m = n / p;
    for (int q = 0; q < p; ++q) fft_rec(in + (size_t)q * stride, out + (size_t)q * m, m, stride * p, tw, tw_n);
    cd v[5], s[5];
    for (int k = 0; k < m; ++k) {
        for (int q = 0; q < p; ++q) v[q] = out[(size_t)q * m + k];
        for (int r = 0; r < p; ++r) {
            cd acc = v[0];
            for (int q = 1; q < p; ++q) acc += v[q] * tw[(size_t)(((long long)q * (k + r * m)) % n) * tstep];
            s[r] = acc;
        }
        for (int r = 0; r < p; ++r) out[(size_t)r * m + k] = s[r];
    }
}
void fft1d(cd* data, int n, int sign) {
    static thread_local std::map<std::pair<int, int>, std::vector<cd>> cache;
    auto& tw = cache[{n, sign}];
    if (tw.empty()) {
        tw.resize(n);
        for (int j = 0; j < n; ++j) tw[j] = unit_root(j, n, sign);
    }
    std::vector<cd> in(data, data + n), out(n);
    fft_rec(in.data(), out.data(), n, 1, tw, n);
    std::copy(out.begin(), out.end(), data);
}
// complex 3-D transform in place, dims (n,n,n) row-major
void fft3d_inplace(std::vector<cd>& a, int n, int sign) {
    std::vector<cd> line(n);
    for (int axis = 0; axis < 3; ++axis) {
        const size_t stride = axis == 0 ? 1 : (axis == 1 ? (size_t)n : (size_t)n * n);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                size_t base;
                if (axis == 0) base = ((size_t)i * n + j) * n;
                else if (axis == 1) base = (size_t)i * n * n + j;
                else base = (size_t)i * n + j;
                for (int t = 0; t < n; ++t) line[t] = a[base + t * stride];
                fft1d(line.data(), n, sign);
                for (int t = 0; t < n; ++t) a[base + t * stride] = line[t];
            }
    }
}
}  // namespace

void fft_r2c_3d(int n, const double* in, cd* out) {
    std::vector<cd> a((size_t)n * n * n);
    for (size_t i = 0; i < a.size(); ++i) a[i] = in[i];
    fft3d_inplace(a, n, -1);
    const int nh = n / 2 + 1;
    for (int z = 0; z < n; ++z)
        for (int y = 0; y < n; ++y)
            for (int x = 0; x < nh; ++x)
                out[((size_t)z * n + y) * nh + x] = a[((size_t)z * n + y) * n + x];
}
void fft_c2r_3d(int n, const cd* in, double* out) {
    const int nh = n / 2 + 1;
    std::vector<cd> a((size_t)n * n * n);
    for (int z = 0; z < n; ++z)
        for (int y = 0; y < n; ++y)
            for (int x = 0; x < n; ++x) {
                cd v;
                if (x < nh) {
                    v = in[((size_t)z * n + y) * nh + x];
                } else {
                    const int zz = (n - z) % n, yy = (n - y) % n;
                    v = std::conj(in[((size_t)zz * n + yy) * nh + (n - x)]);
                }
                a[((size_t)z * n + y) * n + x] = v;
            }
    fft3d_inplace(a, n, +1);
    for (size_t i = 0; i < a.size(); ++i) out[i] = a[i].real();
}
// fftw_util.cpp:16-28,58-61: batched rows, bin m = sum_p f_p e^{-2 pi i m p / n}
void dft_r2c_rows(int n, int count, const double* in, cd* out) {
    const int nb = n / 2 + 1;
    std::vector<cd> tw(n);
    for (int j = 0; j < n; ++j) tw[j] = unit_root(j, n, -1);
    for (int r = 0; r < count; ++r) {
        const double* row = in + (size_t)r * n;
        for (int m = 0; m < nb; ++m) {
            cd acc = 0;
            for (int p = 0; p < n; ++p) acc += row[p] * tw[(size_t)(m * p) % n];
            out[(size_t)r * nb + m] = acc;
        }
    }
}

// ======================================================================= basis
// src/basis.cpp:42-46
static size_t ml_row(int l_max, int m, int l) {
    return (size_t)m * (l_max + 1) - (size_t)m * (m - 1) / 2 + (l - m);
}
// basis.cpp:76-86
cd spherical_harmonic(int l, int m, double theta, double phi) {
    if (l < 0 || std::abs(m) > l) throw std::invalid_argument("spherical_harmonic: require |m| <= l");
    const int ma = std::abs(m);
    std::vector<double> tab(tri_count(l));
    legendre_table(l, std::cos(theta), tab.data());
    const double p = tab[tri_index(l, ma)];
    const cd y = p * std::polar(1.0, ma * phi);
    if (m >= 0) return y;
    return (ma % 2 ? -1.0 : 1.0) * std::conj(y);
}
// basis.cpp:88-115
Spec build_spec(int l_max, double lambda_cut) {
    if (l_max < 0) throw std::invalid_argument("build_spec: l_max must be >= 0");
    if (!(lambda_cut >= kPi))
        throw std::invalid_argument("build_spec: lambda_cut must retain the (l=0,k=1) root pi");
    Spec s;
    s.l_max = l_max;
    s.lambda_cut = lambda_cut;
    s.roots = bessel_root_table(l_max, lambda_cut);
    s.norms.resize(l_max + 1);
    s.block_off.resize(l_max + 1);
    s.pair_off.resize(l_max + 1);
    size_t coeffs = 0, pairs = 0;
    for (int l = 0; l <= l_max; ++l) {
        s.block_off[l] = coeffs;
        s.pair_off[l] = pairs;
        auto& nr = s.norms[l];
        nr.resize(s.roots[l].size());
        for (size_t i = 0; i < nr.size(); ++i)
            nr[i] = std::sqrt(2.0) / std::abs(sph_jl(l + 1, s.roots[l][i]));
        coeffs += s.roots[l].size() * (2 * l + 1);
        pairs += s.roots[l].size();
    }
    s.coeff_total = coeffs;
    s.pair_total = pairs;
    s.build_plan();
    return s;
}
// basis.cpp:117-138
double default_lambda_cut(int n, int l_max) {
    const double nyquist = kPi * n / 2.0;
    auto rows = bessel_root_table(l_max, nyquist);
    const size_t cap = (size_t)n * n * n / 4;
    size_t count = 0;
    std::vector<std::pair<double, size_t>> weighted;
    for (int l = 0; l < (int)rows.size(); ++l)
        for (double r : rows[l]) {
            weighted.emplace_back(r, 2 * l + 1);
            count += 2 * l + 1;
        }
    if (count <= cap) return nyquist;
    std::sort(weighted.begin(), weighted.end());
    size_t acc = 0;
    double cut = kPi;
    for (const auto& [root, w] : weighted) {
        if (acc + w > cap) break;
        acc += w;
        cut = root;
    }
    return cut;
}
// basis.cpp:174-219
void Spec::build_plan() {
    n_theta = 2 * l_max + 2;
    n_phi = 2 * l_max + 2;
    n_r = std::max(l_max + 1, static_cast<int>(std::ceil(0.55 * lambda_cut)) + 8);
    const GL gr = gauss_legendre01(n_r);
    const GL gu = gauss_legendre(n_theta);
    r = gr.nodes;
    cos_theta = gu.nodes;
    sin_theta.resize(n_theta);
    for (int t = 0; t < n_theta; ++t)
        sin_theta[t] = std::sqrt(std::max(0.0, 1.0 - gu.nodes[t] * gu.nodes[t]));
    const size_t n_rows = tri_count(l_max);
    ptab.assign(n_rows * n_theta, 0.0);
    std::vector<double> tab(tri_count(l_max));
    for (int t = 0; t < n_theta; ++t) {
        legendre_table(l_max, gu.nodes[t], tab.data());
        for (int m = 0; m <= l_max; ++m)
            for (int l = m; l <= l_max; ++l)
                ptab[ml_row(l_max, m, l) * n_theta + t] = tab[tri_index(l, m)] * gu.weights[t];
    }
    radial.assign(pair_total * n_r, 0.0);
    const double wphi = 2.0 * kPi / n_phi;
    for (int l = 0; l <= l_max; ++l)
        for (size_t ki = 0; ki < roots[l].size(); ++ki) {
            double* row = radial.data() + (pair_off[l] + ki) * n_r;
            for (int i = 0; i < n_r; ++i) {
                const double rr = gr.nodes[i];
                row[i] = norms[l][ki] * sph_jl(l, roots[l][ki] * rr) * rr * rr * gr.weights[i] * wphi;
            }
        }
}
double Expansion::energy() const {
    double e = 0.0;
    for (const auto& x : c) e += std::norm(x);
    return e;
}
double Expansion::norm() const { return std::sqrt(energy()); }

// basis.cpp:247-330
Expansion expand(const Volume& v, const Spec& spec) {
    const int l_max = spec.l_max;
    const int n_r = spec.n_r, n_theta = spec.n_theta, n_phi = spec.n_phi;
    std::vector<double> samples((size_t)n_r * n_theta * n_phi);
    for (int i = 0; i < n_r; ++i)
        for (int t = 0; t < n_theta; ++t) {
            const double rs = spec.r[i] * spec.sin_theta[t];
            const double z = spec.r[i] * spec.cos_theta[t];
            double* dst = samples.data() + ((size_t)i * n_theta + t) * n_phi;
            for (int p = 0; p < n_phi; ++p) {
                const double phi = 2.0 * kPi * p / n_phi;
                dst[p] = sample_trilinear(v, rs * std::cos(phi), rs * std::sin(phi), z);
            }
        }
    const int n_bins = n_phi / 2 + 1;
    std::vector<cd> g((size_t)n_r * n_theta * n_bins);
    dft_r2c_rows(n_phi, n_r * n_theta, samples.data(), g.data());
    std::vector<cd> gt((size_t)(l_max + 1) * n_r * n_theta);
    for (int m = 0; m <= l_max; ++m)
        for (int i = 0; i < n_r; ++i)
            for (int t = 0; t < n_theta; ++t)
                gt[((size_t)m * n_r + i) * n_theta + t] = g[((size_t)i * n_theta + t) * n_bins + m];
    const size_t n_rows = tri_count(l_max);
    std::vector<cd> h(n_rows * n_r);
    for (int m = 0; m <= l_max; ++m)
        for (int l = m; l <= l_max; ++l) {
            const size_t row = ml_row(l_max, m, l);
            const double* p = spec.ptab.data() + row * n_theta;
            for (int i = 0; i < n_r; ++i) {
                const cd* src = gt.data() + ((size_t)m * n_r + i) * n_theta;
                cd acc{0.0, 0.0};
                for (int t = 0; t < n_theta; ++t) acc += src[t] * p[t];
                h[row * n_r + i] = acc;
            }
        }
    Expansion out;
    out.spec = &spec;
    out.real = true;
    out.c.assign(spec.coeff_total, cd{0.0, 0.0});
    for (int l = 0; l <= l_max; ++l) {
        const int n_k = (int)spec.roots[l].size();
        cd* block = out.c.data() + spec.block_off[l];
        for (int k = 1; k <= n_k; ++k) {
            const double* rw = spec.radial.data() + (spec.pair_off[l] + k - 1) * n_r;
            cd* row = block + (size_t)(k - 1) * (2 * l + 1) + l;
            for (int m = 0; m <= l; ++m) {
                const cd* hs = h.data() + ml_row(l_max, m, l) * n_r;
                cd acc{0.0, 0.0};
                for (int i = 0; i < n_r; ++i) acc += hs[i] * rw[i];
                row[m] = acc;
                if (m > 0) row[-m] = (m % 2 ? -1.0 : 1.0) * std::conj(acc);
            }
        }
    }
    return out;
}

// basis.cpp:221-245, 332-419 (real-volume branch; Catmull-Rom radial table)
Volume synthesize(const Expansion& e, int n) {
    if (n < 8) throw std::invalid_argument("synthesize: grid size must be >= 8");
    const Spec& spec = *e.spec;
    const int l_max = spec.l_max;
    const int n_fine = 2048;
    const size_t row_len = n_fine + 3;
    std::vector<double> rows(spec.pair_total * row_len, 0.0);
    const double hh = 1.0 / n_fine;
    for (int l = 0; l <= l_max; ++l)
        for (size_t ki = 0; ki < spec.roots[l].size(); ++ki) {
            double* row = rows.data() + (spec.pair_off[l] + ki) * row_len;
            const double lc = spec.roots[l][ki], c = spec.norms[l][ki];
            for (int j = 1; j < (int)row_len; ++j) row[j] = c * sph_jl(l, lc * (j - 1) * hh);
            row[0] = (l % 2 ? -1.0 : 1.0) * row[2];
        }
    Volume out(n);
#pragma omp parallel
    {
        std::vector<double> ptab(tri_count(l_max));
        std::vector<cd> phase(l_max + 1), bm(l_max + 1), bneg(l_max + 1);
#pragma omp for schedule(dynamic)
        for (int zi = 0; zi < n; ++zi) {
            const double z = out.coord(zi);
            for (int yi = 0; yi < n; ++yi) {
                const double y = out.coord(yi);
                for (int xi = 0; xi < n; ++xi) {
                    const double x = out.coord(xi);
                    const double r2 = x * x + y * y + z * z;
                    if (r2 >= 1.0) continue;
                    const double r = std::sqrt(r2);
                    const double u = r > 1e-14 ? z / r : 1.0;
                    const double phi = std::atan2(y, x);
                    legendre_table(l_max, u, ptab.data());
                    phase[0] = {1.0, 0.0};
                    const cd e1 = std::polar(1.0, phi);
                    for (int m = 1; m <= l_max; ++m) phase[m] = phase[m - 1] * e1;
                    const double tpos = r * n_fine;
                    const int i0 = std::min(static_cast<int>(tpos), n_fine - 1);
                    const double f = tpos - i0;
                    const double wm1 = ((-0.5 * f + 1.0) * f - 0.5) * f;
                    const double w0 = (1.5 * f - 2.5) * f * f + 1.0;
                    const double w1 = ((-1.5 * f + 2.0) * f + 0.5) * f;
                    const double w2 = (0.5 * f - 0.5) * f * f;
                    double acc = 0.0;
                    cd acc_c{0.0, 0.0};
                    for (int l = 0; l <= l_max; ++l) {
                        const int n_k = (int)spec.roots[l].size();
                        if (n_k == 0) continue;
                        std::fill(bm.begin(), bm.begin() + l + 1, cd{0.0, 0.0});
                        if (!e.real) std::fill(bneg.begin(), bneg.begin() + l + 1, cd{0.0, 0.0});
                        const cd* block = e.c.data() + spec.block_off[l];
                        for (int k = 0; k < n_k; ++k) {
                            const double* row = rows.data() + (spec.pair_off[l] + k) * row_len + i0;
                            const double rv = wm1 * row[0] + w0 * row[1] + w1 * row[2] + w2 * row[3];
                            const cd* c = block + (size_t)k * (2 * l + 1) + l;
                            for (int m = 0; m <= l; ++m) bm[m] += rv * c[m];
                            if (!e.real)
                                for (int m = 1; m <= l; ++m) bneg[m] += rv * c[-m];
                        }
                        if (e.real) {
                            acc += ptab[tri_index(l, 0)] * bm[0].real();
                            for (int m = 1; m <= l; ++m) {
                                const double pp = ptab[tri_index(l, m)];
                                acc += 2.0 * pp * (bm[m].real() * phase[m].real() - bm[m].imag() * phase[m].imag());
                            }
                        } else {
                            for (int m = 0; m <= l; ++m) acc_c += bm[m] * ptab[tri_index(l, m)] * phase[m];
                            for (int m = 1; m <= l; ++m)
                                acc_c += bneg[m] * (m % 2 ? -1.0 : 1.0) * std::conj(ptab[tri_index(l, m)] * phase[m]);
                        }
                    }
                    out.at(xi, yi, zi) = e.real ? acc : acc_c.real();
                }
            }
        }
    }
    return out;
}

// ======================================================================= steer
// src/steer.cpp:13-39
namespace {
struct Tri {
    double v = 0, d1 = 0, d2 = 0;
};
double ipow(double x, int e) {
    double r = 1.0;
    for (int i = 0; i < e; ++i) r *= x;
    return r;
}
Tri cs_power(int a, int p, double c, double s) {
    Tri t;
    t.v = ipow(c, a) * ipow(s, p);
    const double tb = p ? p * ipow(c, a + 1) * ipow(s, p - 1) : 0.0;
    const double ta = a ? a * ipow(c, a - 1) * ipow(s, p + 1) : 0.0;
    t.d1 = 0.5 * (tb - ta);
    const double t2b = p > 1 ? p * (p - 1.0) * ipow(c, a + 2) * ipow(s, p - 2) : 0.0;
    const double t2a = a > 1 ? a * (a - 1.0) * ipow(c, a - 2) * ipow(s, p + 2) : 0.0;
    t.d2 = 0.25 * (t2b + t2a - (2.0 * a * p + a + p) * t.v);
    return t;
}
double sqrt_binom(int n, int k) {
    double r = 1.0;
    for (int i = 1; i <= k; ++i) r *= static_cast<double>(n - k + i) / i;
    return std::sqrt(r);
}
}  // namespace

// steer.cpp:43-144
LittleD little_d_stack(int l_max, double beta, int order) {
    LittleD st;
    st.l_max = l_max;
    st.order = order;
    st.value.resize(l_max + 1);
    if (order >= 1) st.d1.resize(l_max + 1);
    if (order >= 2) st.d2.resize(l_max + 1);
    const double cb = std::cos(beta), sb = std::sin(beta);
    const double ch = std::cos(0.5 * beta), sh = std::sin(0.5 * beta);
    for (int l = 0; l <= l_max; ++l) {
        const size_t w = 2 * l + 1;
        st.value[l].assign(w * w, 0.0);
        if (order >= 1) st.d1[l].assign(w * w, 0.0);
        if (order >= 2) st.d2[l].assign(w * w, 0.0);
    }
    st.value[0][0] = 1.0;
    if (l_max == 0) return st;
    auto put = [&](int l, int m, int mp, const Tri& t) {
        const int w = 2 * l + 1;
        const size_t at = (size_t)(m + l) * w + (mp + l);
        st.value[l][at] = t.v;
        if (order >= 1) st.d1[l][at] = t.d1;
        if (order >= 2) st.d2[l][at] = t.d2;
    };
    for (int l = 1; l <= l_max; ++l) {
        const int w = 2 * l + 1;
        for (int mp = -l; mp <= l; ++mp) {
            const double k = sqrt_binom(2 * l, l + mp);
            const double sign = ((l - mp) % 2) ? -1.0 : 1.0;
            Tri top = cs_power(l + mp, l - mp, ch, sh);
            top.v *= sign * k, top.d1 *= sign * k, top.d2 *= sign * k;
            put(l, l, mp, top);
            Tri bot = cs_power(l - mp, l + mp, ch, sh);
            bot.v *= k, bot.d1 *= k, bot.d2 *= k;
            put(l, -l, mp, bot);
        }
        for (int m = -l + 1; m <= l - 1; ++m) {
            const double k = sqrt_binom(2 * l, l + m);
            Tri right = cs_power(l + m, l - m, ch, sh);
            right.v *= k, right.d1 *= k, right.d2 *= k;
            put(l, m, l, right);
            const double sign = ((l + m) % 2) ? -1.0 : 1.0;
            Tri left = cs_power(l - m, l + m, ch, sh);
            left.v *= sign * k, left.d1 *= sign * k, left.d2 *= sign * k;
            put(l, m, -l, left);
        }
        if (l == 1) {
            put(1, 0, 0, Tri{cb, -sb, -cb});
            continue;
        }
        const int w1 = 2 * l - 1, w2 = 2 * l - 3;
        const double* p1v = st.value[l - 1].data();
        const double* p2v = st.value[l - 2].data();
        const double* p1d = order >= 1 ? st.d1[l - 1].data() : nullptr;
        const double* p2d = order >= 1 ? st.d1[l - 2].data() : nullptr;
        const double* p1h = order >= 2 ? st.d2[l - 1].data() : nullptr;
        const double* p2h = order >= 2 ? st.d2[l - 2].data() : nullptr;
        for (int m = -(l - 1); m <= l - 1; ++m)
            for (int mp = -(l - 1); mp <= l - 1; ++mp) {
                const double a = std::sqrt((static_cast<double>(l) * l - static_cast<double>(m) * m) *
                                           (static_cast<double>(l) * l - static_cast<double>(mp) * mp));
                const double denom = (l - 1.0) * a;
                const double t1 = (2.0 * l - 1.0) * (l * (l - 1.0) * cb - static_cast<double>(m) * mp) / denom;
                const double t1p = -(2.0 * l - 1.0) * l * sb / a;
                const double t1pp = -(2.0 * l - 1.0) * l * cb / a;
                const bool has2 = std::abs(m) <= l - 2 && std::abs(mp) <= l - 2;
                const double b = has2 ? std::sqrt((static_cast<double>(l - 1) * (l - 1) - static_cast<double>(m) * m) *
                                                  (static_cast<double>(l - 1) * (l - 1) - static_cast<double>(mp) * mp))
                                      : 0.0;
                const double t2 = l * b / denom;
                const size_t i1 = (size_t)(m + l - 1) * w1 + (mp + l - 1);
                const size_t i2 = has2 ? (size_t)(m + l - 2) * w2 + (mp + l - 2) : 0;
                const size_t at = (size_t)(m + l) * w + (mp + l);
                const double v1 = p1v[i1];
                const double v2 = has2 ? p2v[i2] : 0.0;
                st.value[l][at] = t1 * v1 - t2 * v2;
                if (order >= 1) {
                    const double g1 = p1d[i1];
                    const double g2 = has2 ? p2d[i2] : 0.0;
                    st.d1[l][at] = t1p * v1 + t1 * g1 - t2 * g2;
                    if (order >= 2) {
                        const double h1 = p1h[i1];
                        const double h2 = has2 ? p2h[i2] : 0.0;
                        st.d2[l][at] = t1pp * v1 + 2.0 * t1p * g1 + t1 * h1 - t2 * h2;
                    }
                }
            }
    }
    return st;
}
// steer.cpp:158-178
std::vector<std::vector<cd>> wigner_D(int l_max, const Rot& g) {
    const Euler e = g.euler_zyz();
    auto st = little_d_stack(l_max, e.beta, 0);
    std::vector<std::vector<cd>> out(l_max + 1);
    for (int l = 0; l <= l_max; ++l) {
        const int w = 2 * l + 1;
        out[l].resize((size_t)w * w);
        for (int m = -l; m <= l; ++m) {
            const cd pa = std::polar(1.0, -m * e.alpha);
            for (int mp = -l; mp <= l; ++mp) {
                const cd pg = std::polar(1.0, -mp * e.gamma);
                out[l][(size_t)(m + l) * w + (mp + l)] = pa * st.value[l][(size_t)(m + l) * w + (mp + l)] * pg;
            }
        }
    }
    return out;
}
// steer.cpp:208-223: f'_m = sum_m' D_{m,m'} f_m' per (k,l) row
Expansion rotate_expansion(const Expansion& e, const Rot& g) {
    const Spec& spec = *e.spec;
    const auto D = wigner_D(spec.l_max, g);
    Expansion out;
    out.spec = e.spec;
    out.real = e.real;
    out.c.assign(spec.coeff_total, cd{0, 0});
    for (int l = 0; l <= spec.l_max; ++l) {
        const int n_k = spec.radial_count(l);
        const int w = 2 * l + 1;
        for (int k = 0; k < n_k; ++k) {
            const cd* src = e.c.data() + spec.block_off[l] + (size_t)k * w;
            cd* dst = out.c.data() + spec.block_off[l] + (size_t)k * w;
            for (int m = 0; m < w; ++m) {
                cd acc{0, 0};
                for (int mp = 0; mp < w; ++mp) acc += src[mp] * D[l][(size_t)m * w + mp];
                dst[m] = acc;
            }
        }
    }
    return out;
}

// ======================================================================= xcorr
Xi::Xi(int L, std::array<int, 3> s) : l_max(L), shift(s) {
    b.resize(L + 1);
    for (int l = 0; l <= L; ++l) b[l].assign((size_t)(2 * l + 1) * (2 * l + 1), cd{0, 0});
}
double Xi::total_energy() const {
    double e = 0;
    for (const auto& blk : b)
        for (const auto& x : blk) e += std::norm(x);
    return e;
}
// src/xcorr.cpp:129-137
double energy_ratio(const Xi& xi, int l_cut) {
    if (l_cut > xi.l_max) throw std::invalid_argument("energy_ratio: l_cut exceeds band limit");
    const double total = xi.total_energy();
    if (!(total > 0.0)) throw std::domain_error("energy_ratio: zero kernel energy");
    double high = 0.0;
    for (int l = l_cut + 1; l <= xi.l_max; ++l)
        for (const auto& x : xi.b[l]) high += std::norm(x);
    return high / total;
}
// optimize.cpp:179-195: per threshold, the lowest band whose energy above it is small enough
std::vector<int> select_bands(const Xi& xi, const std::vector<double>& thresholds) {
    std::vector<double> ratio(xi.l_max + 1);
    for (int l = 0; l <= xi.l_max; ++l) ratio[l] = energy_ratio(xi, l);
    std::vector<int> bands;
    for (double tau : thresholds)
        for (int l = 0; l <= xi.l_max; ++l)
            if (ratio[l] <= tau) {
                bands.push_back(l);
                break;
            }
    std::sort(bands.begin(), bands.end());
    bands.erase(std::unique(bands.begin(), bands.end()), bands.end());
    return bands;
}

// src/xcorr.cpp:34-50: xi_l = T_l^H F_l, i.e. xi[m,m'] = sum_k conj(t[k,m]) f[k,m']
Xi xi_coefficients(const Expansion& t, const Expansion& f, std::array<int, 3> shift) {
    const Spec& spec = *t.spec;
    if (t.spec != f.spec && (t.spec->l_max != f.spec->l_max || t.spec->lambda_cut != f.spec->lambda_cut ||
                             t.spec->coeff_total != f.spec->coeff_total))
        throw std::invalid_argument("xi_coefficients: template and subtomogram specs differ");
    Xi xi(spec.l_max, shift);
    for (int l = 0; l <= spec.l_max; ++l) {
        const int n_k = spec.radial_count(l);
        if (n_k == 0) continue;
        const int w = 2 * l + 1;
        const cd* tb = t.c.data() + spec.block_off[l];
        const cd* fb = f.c.data() + spec.block_off[l];
        for (int m = 0; m < w; ++m)
            for (int mp = 0; mp < w; ++mp) {
                cd acc{0, 0};
                for (int k = 0; k < n_k; ++k) acc += std::conj(tb[(size_t)k * w + m]) * fb[(size_t)k * w + mp];
                xi.b[l][(size_t)m * w + mp] = acc;
            }
    }
    return xi;
}
// xcorr.cpp:52-105
Deriv correlation_derivatives(const Xi& xi, const Euler& ang, int l_cut, int order) {
    if (l_cut > xi.l_max) throw std::invalid_argument("correlation: l_cut exceeds kernel band");
    const auto st = little_d_stack(l_cut, ang.beta, order);
    std::vector<cd> ua(2 * l_cut + 1), ug(2 * l_cut + 1);
    for (int m = -l_cut; m <= l_cut; ++m) {
        ua[m + l_cut] = std::polar(1.0, -m * ang.alpha);
        ug[m + l_cut] = std::polar(1.0, -m * ang.gamma);
    }
    cd val{}, ga{}, gb{}, gg{}, haa{}, hab{}, hag{}, hbb{}, hbg{}, hgg{};
    for (int l = 0; l <= l_cut; ++l) {
        const auto& blk = xi.b[l];
        const int w = 2 * l + 1;
        const double* dv = st.value[l].data();
        const double* d1 = order >= 1 ? st.d1[l].data() : nullptr;
        const double* d2 = order >= 2 ? st.d2[l].data() : nullptr;
        for (int m = -l; m <= l; ++m) {
            const cd pa = ua[m + l_cut];
            for (int mp = -l; mp <= l; ++mp) {
                const size_t at = (size_t)(m + l) * w + (mp + l);
                const cd z = blk[at] * pa * ug[mp + l_cut];
                const cd t = z * dv[at];
                val += t;
                if (order >= 1) {
                    const cd tb = z * d1[at];
                    ga += cd(m * t.imag(), -m * t.real());
                    gb += tb;
                    gg += cd(mp * t.imag(), -mp * t.real());
                    if (order >= 2) {
                        haa += -static_cast<double>(m) * m * t;
                        hag += -static_cast<double>(m) * mp * t;
                        hgg += -static_cast<double>(mp) * mp * t;
                        hab += cd(m * tb.imag(), -m * tb.real());
                        hbg += cd(mp * tb.imag(), -mp * tb.real());
                        hbb += z * d2[at];
                    }
                }
            }
        }
    }
    Deriv out;
    out.value = val.real();
    out.imag = val.imag();
    if (order >= 1) out.grad = {ga.real(), gb.real(), gg.real()};
    if (order >= 2)
        out.hess = {haa.real(), hab.real(), hag.real(), hab.real(), hbb.real(),
                    hbg.real(), hag.real(), hbg.real(), hgg.real()};
    return out;
}
// xcorr.cpp:149-155: xi~_l = xi_l D^l(a)^T
Xi xi_compose_right(const Xi& xi, const Rot& a, int l_limit) {
    const int top = l_limit < 0 ? xi.l_max : std::min(l_limit, xi.l_max);
    const auto D = wigner_D(top, a);
    Xi out(xi.l_max, xi.shift);
    for (int l = 0; l <= top; ++l) {
        const int w = 2 * l + 1;
        for (int m = 0; m < w; ++m)
            for (int mp = 0; mp < w; ++mp) {
                cd acc{0, 0};
                for (int n = 0; n < w; ++n) acc += xi.b[l][(size_t)m * w + n] * D[l][(size_t)mp * w + n];
                out.b[l][(size_t)m * w + mp] = acc;
            }
    }
    return out;
}

// xcorr.cpp:157-193
static Vec3 cross(const Vec3& a, const Vec3& b) {
    return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
static double norm3(const Vec3& a) { return std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]); }
WedgeMask::WedgeMask(int n_, double theta_deg, Vec3 axis) : n(n_), theta_max_deg(theta_deg) {
    if (!(theta_deg > 0.0) || theta_deg > 90.0)
        throw std::invalid_argument("WedgeMask: theta_max must be in (0, 90]");
    const double an = norm3(axis);
    tilt_axis = {axis[0] / an, axis[1] / an, axis[2] / an};
    all_pass = theta_deg >= 90.0;
    tan_theta = std::tan(theta_deg * kPi / 180.0);
    Vec3 p = cross(tilt_axis, {0, 0, 1});
    const double pn = norm3(p);
    if (pn < 1e-8) throw std::invalid_argument("WedgeMask: tilt axis must not be parallel to the beam");
    perp = {p[0] / pn, p[1] / pn, p[2] / pn};
}
bool WedgeMask::keeps_direction(const Vec3& nu) const {
    if (all_pass) return true;
    const double along_beam = std::abs(nu[2]);
    const double in_plane = std::abs(nu[0] * perp[0] + nu[1] * perp[1] + nu[2] * perp[2]);
    return along_beam <= tan_theta * in_plane;
}
double WedgeMask::kept_fraction() const {
    long kept = 0;
    const int h = n / 2;
    for (int fz = -h; fz < h; ++fz)
        for (int fy = -h; fy < h; ++fy)
            for (int fx = -h; fx < h; ++fx)
                if (keeps(fx, fy, fz)) ++kept;
    return (double)kept / ((double)n * n * n);
}
// xcorr.cpp:195-208
double wedge_keep_profile(const WedgeMask& mask, const Vec3& nu, double taper_deg) {
    if (mask.theta_max_deg >= 90.0) return 1.0;
    if (taper_deg <= 0.0) return mask.keeps_direction(nu) ? 1.0 : 0.0;
    Vec3 p = cross(mask.tilt_axis, {0, 0, 1});
    const double pn = norm3(p);
    p = {p[0] / pn, p[1] / pn, p[2] / pn};
    const double along_beam = std::abs(nu[2]);
    const double in_plane = std::abs(nu[0] * p[0] + nu[1] * p[1] + nu[2] * p[2]);
    if (along_beam == 0.0 && in_plane == 0.0) return 1.0;
    const double a = std::atan2(along_beam, in_plane) * 180.0 / kPi;
    const double x = (mask.theta_max_deg - a) / taper_deg;
    if (x >= 1.0) return 1.0;
    if (x <= 0.0) return 0.0;
    return x * x * (3.0 - 2.0 * x);
}
// xcorr.cpp:210-232
Volume apply_wedge_taper(const Volume& v, const WedgeMask& mask, double taper_deg) {
    if (mask.n != v.n) throw std::invalid_argument("apply_wedge_taper: mask/volume size mismatch");
    const int n = v.n, nh = n / 2 + 1;
    std::vector<cd> spec((size_t)n * n * nh);
    fft_r2c_3d(n, v.d.data(), spec.data());
    auto signed_freq = [n](int i) { return i <= n / 2 ? i : i - n; };
    for (int z = 0; z < n; ++z) {
        const int fz = signed_freq(z);
        for (int y = 0; y < n; ++y) {
            const int fy = signed_freq(y);
            cd* row = spec.data() + ((size_t)z * n + y) * nh;
            for (int x = 0; x < nh; ++x) row[x] *= wedge_keep_profile(mask, {(double)x, (double)fy, (double)fz}, taper_deg);
        }
    }
    Volume out(n);
    fft_c2r_3d(n, spec.data(), out.d.data());
    const double scale = 1.0 / ((double)n * n * n);
    for (double& d : out.d) d *= scale;
    return out;
}
// xcorr.cpp:359-381
Volume apply_wedge(const Volume& v, const WedgeMask& mask) {
    if (mask.n != v.n) throw std::invalid_argument("apply_wedge: mask/volume size mismatch");
    const int n = v.n, nh = n / 2 + 1;
    std::vector<cd> spec((size_t)n * n * nh);
    fft_r2c_3d(n, v.d.data(), spec.data());
    auto signed_freq = [n](int i) { return i <= n / 2 ? i : i - n; };
    for (int z = 0; z < n; ++z) {
        const int fz = signed_freq(z);
        for (int y = 0; y < n; ++y) {
            const int fy = signed_freq(y);
            cd* row = spec.data() + ((size_t)z * n + y) * nh;
            for (int x = 0; x < nh; ++x)
                if (!mask.keeps(x, fy, fz)) row[x] = {0.0, 0.0};
        }
    }
    Volume out(n);
    fft_c2r_3d(n, spec.data(), out.d.data());
    const double scale = 1.0 / ((double)n * n * n);
    for (double& d : out.d) d *= scale;
    return out;
}
// xcorr.cpp:234-341 (the two spherical-harmonic analyses)
WedgePowerFactors wedge_power_factors(const Volume& tmpl, const WedgeMask& mask, int l_max, double taper_deg) {
    WedgePowerFactors wf;
    const size_t n_tri = tri_count(l_max);
    wf.chi_hat.assign(n_tri, cd{0, 0});
    wf.q_hat.assign(n_tri, cd{0, 0});
    if (mask.theta_max_deg >= 90.0) return wf;
    const int n = tmpl.n, np = 2 * n, nph = np / 2 + 1;
    std::vector<double> padded((size_t)np * np * np, 0.0);
    const int off = n / 2;
    for (int z = 0; z < n; ++z)
        for (int y = 0; y < n; ++y)
            for (int x = 0; x < n; ++x)
                padded[((size_t)(z + off) * np + (y + off)) * np + (x + off)] = tmpl.at(x, y, z);
    std::vector<cd> half((size_t)np * np * nph);
    fft_r2c_3d(np, padded.data(), half.data());
    std::vector<double> power((size_t)np * np * np);
    auto wrap = [np](int i) { return (i % np + np) % np; };
    for (int z = 0; z < np; ++z)
        for (int y = 0; y < np; ++y)
            for (int x = 0; x < np; ++x) {
                const size_t at = ((size_t)z * np + y) * np + x;
                if (x < nph) power[at] = std::norm(half[((size_t)z * np + y) * nph + x]);
                else power[at] = std::norm(half[((size_t)wrap(-z) * np + wrap(-y)) * nph + (np - x)]);
            }
    power[0] = 0.0;
    auto power_at = [&](double fx, double fy, double fz) {
        const int ix = (int)std::floor(fx), iy = (int)std::floor(fy), iz = (int)std::floor(fz);
        const double ux = fx - ix, uy = fy - iy, uz = fz - iz;
        double acc = 0.0;
        for (int dz = 0; dz < 2; ++dz)
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) {
                    const double w = (dx ? ux : 1 - ux) * (dy ? uy : 1 - uy) * (dz ? uz : 1 - uz);
                    acc += w * power[((size_t)wrap(iz + dz) * np + wrap(iy + dy)) * np + wrap(ix + dx)];
                }
        return acc;
    };
    const int n_theta = 3 * (l_max + 1), n_phi = 3 * (l_max + 1), n_rad = 2 * n;
    const GL gu = gauss_legendre(n_theta);
    std::vector<double> q((size_t)n_theta * n_phi), chi((size_t)n_theta * n_phi);
    const double r_max = np / 2.0;
#pragma omp parallel for schedule(static)
    for (int t = 0; t < n_theta; ++t) {
        const double u = gu.nodes[t];
        const double st = std::sqrt(std::max(0.0, 1.0 - u * u));
        for (int p = 0; p < n_phi; ++p) {
            const double phi = 2.0 * kPi * p / n_phi;
            const Vec3 dir{st * std::cos(phi), st * std::sin(phi), u};
            double acc = 0.0;
            for (int j = 0; j < n_rad; ++j) {
                const double r = (j + 0.5) * r_max / n_rad;
                acc += r * r * power_at(r * dir[0], r * dir[1], r * dir[2]);
            }
            q[(size_t)t * n_phi + p] = acc;
            chi[(size_t)t * n_phi + p] = 1.0 - wedge_keep_profile(mask, dir, taper_deg);
        }
    }
    std::vector<double> ptab(n_tri);
    double total = 0.0;
    const double wphi = 2.0 * kPi / n_phi;
    for (int t = 0; t < n_theta; ++t) {
        legendre_table(l_max, gu.nodes[t], ptab.data());
        const double wt = gu.weights[t];
        for (int m = 0; m <= l_max; ++m) {
            cd gq{0, 0}, gc{0, 0};
            for (int p = 0; p < n_phi; ++p) {
                const cd e = std::polar(1.0, -m * (2.0 * kPi * p / n_phi));
                gq += q[(size_t)t * n_phi + p] * e;
                gc += chi[(size_t)t * n_phi + p] * e;
            }
            for (int l = m; l <= l_max; ++l) {
                const double pw = ptab[tri_index(l, m)] * wt * wphi;
                wf.q_hat[tri_index(l, m)] += gq * pw;
                wf.chi_hat[tri_index(l, m)] += gc * pw;
            }
        }
        for (int p = 0; p < n_phi; ++p) total += q[(size_t)t * n_phi + p] * wt * wphi;
    }
    wf.total = total;
    return wf;
}
// xcorr.cpp:234-357
Xi wedge_power_kernel(const Volume& tmpl, const WedgeMask& mask, int l_max, double taper_deg) {
    Xi out(l_max, {0, 0, 0});
    if (mask.theta_max_deg >= 90.0) return out;
    const WedgePowerFactors wf = wedge_power_factors(tmpl, mask, l_max, taper_deg);
    if (!(wf.total > 0.0)) return out;
    auto coef = [&](const std::vector<cd>& hat, int l, int m) {
        if (m >= 0) return hat[tri_index(l, m)];
        const cd c = std::conj(hat[tri_index(l, -m)]);
        return (-m) % 2 ? -c : c;
    };
    for (int l = 0; l <= l_max; ++l)
        for (int m = -l; m <= l; ++m)
            for (int mp = -l; mp <= l; ++mp)
                out.at(l, m, mp) = std::conj(coef(wf.chi_hat, l, m)) * coef(wf.q_hat, l, mp) / wf.total;
    return out;
}

// ======================================================================= optimize
namespace {
constexpr double kAnchorMargin = 0.05;  // optimize.cpp:20
struct EulerGrid {                      // optimize.cpp:27-44
    int na = 0, nb = 0, ng = 0;
    static EulerGrid with_step(double step) {
        EulerGrid g;
        g.na = static_cast<int>(std::ceil(2.0 * kPi / step));
        g.ng = g.na;
        g.nb = static_cast<int>(std::ceil(kPi / step)) + 1;
        return g;
    }
    double alpha(int i) const { return 2.0 * kPi * i / na; }
    double beta(int j) const { return nb > 1 ? kPi * j / (nb - 1) : 0.0; }
    double gamma(int k) const { return 2.0 * kPi * k / ng; }
    long size() const { return (long)na * nb * ng; }
    size_t at(int i, int j, int k) const { return ((size_t)j * na + i) * ng + k; }
};
// optimize.cpp:48-97
std::vector<double> grid_scores_impl(const Xi& xi, int l_cut, const EulerGrid& grid) {
    const int w = 2 * l_cut + 1;
    std::vector<cd> ua((size_t)grid.na * w), ug((size_t)grid.ng * w);
    for (int i = 0; i < grid.na; ++i)
        for (int m = -l_cut; m <= l_cut; ++m) ua[(size_t)i * w + (m + l_cut)] = std::polar(1.0, -m * grid.alpha(i));
    for (int k = 0; k < grid.ng; ++k)
        for (int m = -l_cut; m <= l_cut; ++m) ug[(size_t)k * w + (m + l_cut)] = std::polar(1.0, -m * grid.gamma(k));
    std::vector<double> out(grid.size());
    for (int j = 0; j < grid.nb; ++j) {
        const auto st = little_d_stack(l_cut, grid.beta(j), 0);
        std::vector<cd> a((size_t)w * w, cd{0.0, 0.0});
        for (int l = 0; l <= l_cut; ++l) {
            const int wl = 2 * l + 1;
            for (int m = -l; m <= l; ++m)
                for (int mp = -l; mp <= l; ++mp)
                    a[(size_t)(m + l_cut) * w + (mp + l_cut)] +=
                        xi.at(l, m, mp) * st.value[l][(size_t)(m + l) * wl + (mp + l)];
        }
        std::vector<cd> b(w);
        for (int k = 0; k < grid.ng; ++k) {
            const cd* pg = ug.data() + (size_t)k * w;
            for (int m = 0; m < w; ++m) {
                cd acc{0.0, 0.0};
                const cd* row = a.data() + (size_t)m * w;
                for (int mp = 0; mp < w; ++mp) acc += row[mp] * pg[mp];
                b[m] = acc;
            }
            for (int i = 0; i < grid.na; ++i) {
                const cd* pa = ua.data() + (size_t)i * w;
                double acc = 0.0;
                for (int m = 0; m < w; ++m) acc += pa[m].real() * b[m].real() - pa[m].imag() * b[m].imag();
                out[grid.at(i, j, k)] = acc;
            }
        }
    }
    return out;
}
// optimize.cpp:102-131
struct Objective {
    const Xi* corr = nullptr;
    const Xi* wedge_power = nullptr;
    Deriv eval(const Euler& e, int band, int order) const {
        Deriv c = correlation_derivatives(*corr, e, band, order);
        if (!wedge_power) return c;
        const int nband = std::min(band, wedge_power->l_max);
        const Deriv r = correlation_derivatives(*wedge_power, e, nband, order);
        const double v = std::clamp(1.0 - r.value, 0.02, 2.0);
        const double s = 1.0 / std::sqrt(v);
        Deriv f;
        f.value = c.value * s;
        f.imag = c.imag * s;
        if (order >= 1) {
            const Vec3 dv{-r.grad[0], -r.grad[1], -r.grad[2]};
            const double v32 = s / v;
            for (int i = 0; i < 3; ++i) f.grad[i] = c.grad[i] * s - 0.5 * c.value * v32 * dv[i];
            if (order >= 2) {
                const double v52 = v32 / v;
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) {
                        const double hv = -r.hess[i * 3 + j];
                        f.hess[i * 3 + j] = c.hess[i * 3 + j] * s -
                                            0.5 * v32 * (c.grad[i] * dv[j] + dv[i] * c.grad[j] + c.value * hv) +
                                            0.75 * c.value * v52 * dv[i] * dv[j];
                    }
            }
        }
        return f;
    }
};
// Eigen::FullPivLU<Matrix3d> restated (compute / rank / solve); threshold
// = epsilon * diagonalSize relative to the largest pivot (Eigen's default).
struct FullPivLU3 {
    double lu[3][3];
    int rowp[3], colp[3];  // row/col transpositions
    int nonzero_pivots = 3;
    double maxpivot = 0;
    explicit FullPivLU3(const Mat3& m) {
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) lu[i][j] = m[i * 3 + j];
        nonzero_pivots = 3;
        maxpivot = 0;
        for (int k = 0; k < 3; ++k) {
            // biggest |a| in the bottom-right corner, column-major visiting order
            int br = k, bc = k;
            double big = -1.0;
            for (int j = k; j < 3; ++j)
                for (int i = k; i < 3; ++i) {
                    const double a = std::abs(lu[i][j]);
                    if (a > big) {
                        big = a;
                        br = i;
                        bc = j;
                    }
                }
            if (big == 0.0) {
                nonzero_pivots = k;
                for (int i = k; i < 3; ++i) {
                    rowp[i] = i;
                    colp[i] = i;
                }
                break;
            }
            if (big > maxpivot) maxpivot = big;
            rowp[k] = br;
            colp[k] = bc;
            if (k != br)
                for (int j = 0; j < 3; ++j) std::swap(lu[k][j], lu[br][j]);
            if (k != bc)
                for (int i = 0; i < 3; ++i) std::swap(lu[i][k], lu[i][bc]);
            if (k < 2) {
                for (int i = k + 1; i < 3; ++i) lu[i][k] /= lu[k][k];
                for (int i = k + 1; i < 3; ++i)
                    for (int j = k + 1; j < 3; ++j) lu[i][j] -= lu[i][k] * lu[k][j];
            }
        }
    }
    bool invertible() const {
        const double thr = std::numeric_limits<double>::epsilon() * 3.0 * std::abs(maxpivot);
        int rank = 0;
        for (int i = 0; i < nonzero_pivots; ++i)
            if (std::abs(lu[i][i]) > thr) ++rank;
        return rank == 3;
    }
    Vec3 solve(const Vec3& b) const {
        double c[3] = {b[0], b[1], b[2]};
        for (int k = 0; k < 3; ++k)
            if (rowp[k] != k) std::swap(c[k], c[rowp[k]]);
        for (int i = 1; i < 3; ++i)
            for (int j = 0; j < i; ++j) c[i] -= lu[i][j] * c[j];
        for (int i = 2; i >= 0; --i) {
            for (int j = i + 1; j < 3; ++j) c[i] -= lu[i][j] * c[j];
            c[i] /= lu[i][i];
        }
        for (int k = 2; k >= 0; --k)
            if (colp[k] != k) std::swap(c[k], c[colp[k]]);
        return {c[0], c[1], c[2]};
    }
};
bool outcome_better(const ShiftOutcome& a, const ShiftOutcome& b) {  // optimize.cpp:144-149
    if (a.norm_score != b.norm_score) return a.norm_score > b.norm_score;
    if (a.shift != b.shift) return a.shift < b.shift;
    return a.refined.rotation.angle() < b.refined.rotation.angle();
}
}  // namespace

// exhaustive_baseline (optimize.cpp:523-539): first maximum of the full grid
Baseline exhaustive_baseline(const Xi& xi, int l_cut, double step) {
    if (!(step > 0.0)) throw std::invalid_argument("baseline: step must be positive");
    const EulerGrid grid = EulerGrid::with_step(step);
    const std::vector<double> sc = grid_scores_impl(xi, l_cut, grid);
    size_t best = 0;
    for (size_t i = 1; i < sc.size(); ++i)
        if (sc[i] > sc[best]) best = i;
    const int k = (int)(best % grid.ng), i = (int)((best / grid.ng) % grid.na), j = (int)(best / ((size_t)grid.ng * grid.na));
    Baseline b;
    b.rotation = Rot::from_euler_zyz(grid.alpha(i), grid.beta(j), grid.gamma(k));
    b.score = sc[best];
    b.evaluations = grid.size();
    return b;
}
long baseline_evaluation_count(double step) { return EulerGrid::with_step(step).size(); }  // optimize.cpp:541-544

std::vector<double> grid_scores(const Xi& xi, int l_cut, double step) {
    return grid_scores_impl(xi, l_cut, EulerGrid::with_step(step));
}

void Config::validate() const {  // optimize.cpp:153-177
    if (l_max < 0) throw std::invalid_argument("config: l_max must be >= 0");
    for (size_t i = 1; i < band_thresholds.size(); ++i)
        if (!(band_thresholds[i - 1] >= band_thresholds[i]))
            throw std::invalid_argument("config: band thresholds must be strictly decreasing");
    for (double t : band_thresholds)
        if (!(t > 0.0 && t < 1.0)) throw std::invalid_argument("config: band thresholds must lie in (0,1)");
    if (fixed_bands.empty() && !auto_bands)
        throw std::invalid_argument("config: need fixed bands or auto band selection");
    for (size_t i = 0; i < fixed_bands.size(); ++i) {
        if (fixed_bands[i] < 0 || fixed_bands[i] > l_max)
            throw std::invalid_argument("config: bands must lie in [0, l_max]");
        if (i > 0 && fixed_bands[i] <= fixed_bands[i - 1])
            throw std::invalid_argument("config: bands must be strictly increasing");
    }
    if (!(seed_grid_step > 0.0) || seed_grid_step > kPi)
        throw std::invalid_argument("config: seed grid step must be in (0, pi]");
    if (max_candidates < 1 || newton_max_iter < 1)
        throw std::invalid_argument("config: counts must be positive");
    if (!(grad_tol > 0.0) || !(step_damping > 0.0))
        throw std::invalid_argument("config: tolerances must be positive");
    if (shift_radius < 0 || shift_step < 1) throw std::invalid_argument("config: bad shift search parameters");
}

// optimize.cpp:197-253
std::vector<Candidate> seed_candidates(const Xi& xi, int l_low, double step, int max_candidates,
                                       const Xi* wedge_power) {
    if (l_low > xi.l_max) throw std::invalid_argument("seed_candidates: band exceeds l_max");
    const EulerGrid grid = EulerGrid::with_step(step);
    std::vector<double> scores = grid_scores_impl(xi, l_low, grid);
    if (wedge_power) {
        const std::vector<double> rho = grid_scores_impl(*wedge_power, std::min(l_low, wedge_power->l_max), grid);
        for (size_t i = 0; i < scores.size(); ++i) scores[i] /= std::sqrt(std::clamp(1.0 - rho[i], 0.02, 2.0));
    }
    std::vector<std::pair<size_t, double>> maxima;
    for (int j = 0; j < grid.nb; ++j)
        for (int i = 0; i < grid.na; ++i)
            for (int k = 0; k < grid.ng; ++k) {
                const size_t self = grid.at(i, j, k);
                const double s = scores[self];
                bool is_max = true;
                for (int dj = -1; dj <= 1 && is_max; ++dj) {
                    const int jj = j + dj;
                    if (jj < 0 || jj >= grid.nb) continue;
                    for (int di = -1; di <= 1 && is_max; ++di) {
                        const int ii = (i + di + grid.na) % grid.na;
                        for (int dk = -1; dk <= 1; ++dk) {
                            const int kk = (k + dk + grid.ng) % grid.ng;
                            const size_t other = grid.at(ii, jj, kk);
                            if (other == self) continue;
                            const double t = scores[other];
                            if (t > s || (t == s && other < self)) {
                                is_max = false;
                                break;
                            }
                        }
                    }
                }
                if (is_max) maxima.emplace_back(self, s);
            }
    std::sort(maxima.begin(), maxima.end(), [](const auto& a, const auto& b) {
        if (a.second != b.second) return a.second > b.second;
        return a.first < b.first;
    });
    if ((int)maxima.size() > max_candidates) maxima.resize(max_candidates);
    std::vector<Candidate> out;
    for (const auto& [idx, s] : maxima) {
        const int k = (int)(idx % grid.ng);
        const int i = (int)((idx / grid.ng) % grid.na);
        const int j = (int)(idx / ((size_t)grid.ng * grid.na));
        out.push_back({Rot::from_euler_zyz(grid.alpha(i), grid.beta(j), grid.gamma(k)), s, (long)idx});
    }
    return out;
}

// optimize.cpp:255-357
RefineResult refine(const Xi& xi, const Rot& start, const std::vector<int>& bands, const Config& cfg,
                    const Xi* wedge_power) {
    if (bands.empty()) throw std::invalid_argument("refine: band list is empty");
    static const Rot kOffset = Rot::from_euler_zyz(0.0, kPi / 2.0, 0.0);
    RefineResult res;
    Rot g = start, anchor;
    bool anchored = false;
    int anchor_limit = -1;
    Objective obj{&xi, wedge_power};
    Xi owned, owned_wp;
    auto reanchor = [&](const Rot& target, int band) {
        anchor = kOffset.inverse() * target;
        anchor_limit = band;
        owned = xi_compose_right(xi, anchor, band);
        obj.corr = &owned;
        if (wedge_power) {
            owned_wp = xi_compose_right(*wedge_power, anchor, band);
            obj.wedge_power = &owned_wp;
        }
        anchored = true;
    };
    bool diverged = false, band_converged = false;
    double best_score = -std::numeric_limits<double>::infinity();
    Rot best_g = start;
    for (size_t bi = 0; bi < bands.size() && !diverged; ++bi) {
        const int band = bands[bi];
        auto& evals = res.evals[band];
        double lambda = cfg.step_damping;
        band_converged = false;
        if (anchored && band > anchor_limit) reanchor(g, band);
        for (int iter = 0; iter < cfg.newton_max_iter; ++iter) {
            Rot h = g * anchor.inverse();
            Euler e = h.euler_zyz();
            if (e.beta < kAnchorMargin || e.beta > kPi - kAnchorMargin) {
                reanchor(g, band);
                h = kOffset;
                e = h.euler_zyz();
            }
            const Deriv d = obj.eval(e, band, 2);
            ++evals;
            const double scale = std::max(std::abs(d.value), 1e-300);
            const double gnorm = norm3(d.grad);
            res.trace.push_back({band, iter, e.alpha, e.beta, e.gamma, d.value, gnorm});
            if (d.value > best_score) {
                best_score = d.value;
                best_g = g;
            }
            if (gnorm <= cfg.grad_tol * scale) {
                band_converged = true;
                break;
            }
            bool accepted = false;
            double lam = lambda;
            for (int retry = 0; retry < 3 && !accepted; ++retry, lam *= 10.0) {
                Mat3 m = d.hess;
                m[0] -= lam, m[4] -= lam, m[8] -= lam;
                Vec3 p;
                const FullPivLU3 lu(m);
                if (lu.invertible()) {
                    const Vec3 x = lu.solve(d.grad);
                    p = {-x[0], -x[1], -x[2]};
                } else {
                    p = {d.grad[0] / lam, d.grad[1] / lam, d.grad[2] / lam};
                }
                const double pn = norm3(p);
                if (pn > 1.0) {
                    const double s = 1.0 / pn;
                    p = {p[0] * s, p[1] * s, p[2] * s};
                }
                const Rot h_try = Rot::from_euler_zyz(e.alpha + p[0], e.beta + p[1], e.gamma + p[2]);
                const Deriv trial = obj.eval(h_try.euler_zyz(), band, 0);
                ++evals;
                if (trial.value > d.value - 1e-12 * scale) {
                    g = h_try * anchor;
                    lambda = std::max(lam / 10.0, 1e-12);
                    accepted = true;
                    if (trial.value > best_score) {
                        best_score = trial.value;
                        best_g = g;
                    }
                }
            }
            if (!accepted) {
                diverged = true;
                break;
            }
        }
    }
    res.rotation = diverged ? best_g : g;
    const Objective unanchored{&xi, wedge_power};
    res.score = unanchored.eval(res.rotation.euler_zyz(), bands.back(), 0).value;
    ++res.evals[bands.back()];
    res.converged = !diverged && band_converged;
    return res;
}

// optimize.cpp:361-419
ShiftOutcome search_one_shift(const Volume& subtomo, const std::array<int, 3>& s, const Expansion& t_hat,
                              double t_norm, const std::vector<int>& bands, const Config& cfg,
                              const Xi* wedge_power) {
    ShiftOutcome oc;
    oc.shift = s;
    const Volume f_s = shift_volume(subtomo, s);
    const Expansion f_hat = expand(f_s, *t_hat.spec);
    oc.subtomo_norm = f_hat.norm();
    if (!(oc.subtomo_norm > 0.0)) return oc;
    const Xi xi = xi_coefficients(f_hat, t_hat, s);
    auto cands = seed_candidates(xi, bands.front(), cfg.seed_grid_step, cfg.max_candidates, wedge_power);
    const EulerGrid grid = EulerGrid::with_step(cfg.seed_grid_step);
    oc.evals[bands.front()] += grid.size();
    if (cands.empty()) return oc;
    auto run = [&](const Rot& start, const std::vector<int>& schedule) {
        RefineResult r = refine(xi, start, schedule, cfg, wedge_power);
        for (const auto& [band, n] : r.evals) oc.evals[band] += n;
        ++oc.candidates;
        return r;
    };
    RefineResult best;
    bool have = false;
    if (cfg.prune_after_band && bands.size() > 1) {  // optimize.cpp:391-403
        RefineResult low_best;
        bool low_have = false;
        for (const auto& c : cands) {
            RefineResult r = run(c.rotation, {bands.front()});
            if (!low_have || r.score > low_best.score) {
                low_best = std::move(r);
                low_have = true;
            }
        }
        best = run(low_best.rotation, std::vector<int>(bands.begin() + 1, bands.end()));
        have = true;
    } else {
        for (const auto& c : cands) {
            RefineResult r = run(c.rotation, bands);
            if (!have || r.score > best.score ||
                (r.score == best.score && r.rotation.angle() < best.rotation.angle())) {
                best = std::move(r);
                have = true;
            }
        }
    }
    oc.refined = std::move(best);
    oc.raw_score = oc.refined.score;
    oc.norm_score = oc.raw_score / (t_norm * oc.subtomo_norm);
    oc.valid = true;
    return oc;
}

// optimize.cpp:423-521 (fixed bands; the windows of a stage run in parallel)
AlignResult align(const Volume& tmpl, const Volume& subtomo, const Config& cfg,
                  const std::optional<WedgeMask>& wedge) {
    cfg.validate();
    if (tmpl.n != subtomo.n) throw std::invalid_argument("align: template and subtomogram grids differ");
    if (!(volume_l2_norm(tmpl) > 0.0) || !(volume_l2_norm(subtomo) > 0.0))
        throw std::invalid_argument("align: zero-energy input volume");
    AlignResult out;
    const double cut = cfg.lambda_cut > 0.0 ? cfg.lambda_cut : default_lambda_cut(tmpl.n, cfg.l_max);
    const Spec spec = build_spec(cfg.l_max, cut);
    const Volume f_w = wedge ? apply_wedge_taper(subtomo, *wedge) : subtomo;
    const Expansion t_hat = expand(tmpl, spec);
    out.template_norm = t_hat.norm();
    if (!(out.template_norm > 0.0)) throw std::invalid_argument("align: template has no in-ball energy");
    std::optional<Xi> wp;
    if (wedge && wedge->theta_max_deg < 90.0) wp = wedge_power_kernel(tmpl, *wedge, cfg.l_max);
    const Xi* wp_ptr = wp ? &*wp : nullptr;
    std::vector<int> bands = cfg.fixed_bands;
    if (cfg.auto_bands) {  // optimize.cpp:455-460: the zero-shift kernel's energy ratios
        const Expansion f0 = expand(f_w, spec);
        bands = select_bands(xi_coefficients(f0, t_hat, {0, 0, 0}), cfg.band_thresholds);
    }
    out.bands = bands;
#ifdef _OPENMP
    const int n_threads = cfg.threads > 0 ? cfg.threads : omp_get_max_threads();
#endif
    auto run_stage = [&](const std::vector<std::array<int, 3>>& shifts) {
        std::vector<ShiftOutcome> res(shifts.size());
#pragma omp parallel for schedule(dynamic) num_threads(n_threads)
        for (long i = 0; i < (long)shifts.size(); ++i)
            res[i] = search_one_shift(f_w, shifts[i], t_hat, out.template_norm, bands, cfg, wp_ptr);
        return res;
    };
    std::vector<std::array<int, 3>> coarse;
    for (int z = -cfg.shift_radius; z <= cfg.shift_radius; z += cfg.shift_step)
        for (int y = -cfg.shift_radius; y <= cfg.shift_radius; y += cfg.shift_step)
            for (int x = -cfg.shift_radius; x <= cfg.shift_radius; x += cfg.shift_step)
                coarse.push_back({x, y, z});
    std::vector<ShiftOutcome> outcomes = run_stage(coarse);
    const ShiftOutcome* best = nullptr;
    for (const auto& oc : outcomes)
        if (oc.valid && (!best || outcome_better(oc, *best))) best = &oc;
    if (!best) throw std::invalid_argument("align: no usable shift window (empty subtomogram)");
    std::vector<std::array<int, 3>> fine;
    for (int z = -cfg.shift_step; z <= cfg.shift_step; ++z)
        for (int y = -cfg.shift_step; y <= cfg.shift_step; ++y)
            for (int x = -cfg.shift_step; x <= cfg.shift_step; ++x) {
                const std::array<int, 3> s{best->shift[0] + x, best->shift[1] + y, best->shift[2] + z};
                if (std::find(coarse.begin(), coarse.end(), s) == coarse.end()) fine.push_back(s);
            }
    std::vector<ShiftOutcome> fine_outcomes = run_stage(fine);
    for (const auto& oc : fine_outcomes)
        if (oc.valid && outcome_better(oc, *best)) best = &oc;
    for (const auto* set : {&outcomes, &fine_outcomes})
        for (const auto& oc : *set) {
            out.candidates_evaluated += oc.candidates;
            for (const auto& [band, n] : oc.evals) out.evals[band] += n;
        }
    out.windows = (int)(coarse.size() + fine.size());
    out.shift = best->shift;
    out.rotation = best->refined.rotation;
    out.score = best->norm_score;
    out.converged = best->refined.converged;
    out.subtomo_norm = best->subtomo_norm;
    return out;
}

// ======================================================================= volio
Volume rotate_volume_trilinear(const Volume& v, const Rot& g) {  // volio.cpp:195-206
    const Mat3 m = g.matrix();
    Volume out(v.n);
    for (int z = 0; z < v.n; ++z)
        for (int y = 0; y < v.n; ++y)
            for (int x = 0; x < v.n; ++x) {
                const double cx = v.coord(x), cy = v.coord(y), cz = v.coord(z);
                // R^T * c
                const double px = m[0] * cx + m[3] * cy + m[6] * cz;
                const double py = m[1] * cx + m[4] * cy + m[7] * cz;
                const double pz = m[2] * cx + m[5] * cy + m[8] * cz;
                out.at(x, y, z) = sample_trilinear(v, px, py, pz);
            }
    return out;
}
Rot haar_rotation(PhiloxStream& rng) {  // volio.cpp:208-215
    const double u1 = rng.next_unit(), u2 = rng.next_unit(), u3 = rng.next_unit();
    const double a = std::sqrt(1.0 - u1), b = std::sqrt(u1);
    const double t2 = 2.0 * kPi * u2, t3 = 2.0 * kPi * u3;
    return Rot::make(b * std::cos(t3), a * std::sin(t2), a * std::cos(t2), b * std::sin(t3));
}

namespace {
// volio.cpp:285-314: rotate -> shift by -s -> binary wedge -> noise -> f32 rounding
void finish_particle(Phantom& out, std::optional<double> snr, std::optional<double> wedge_deg,
                     uint64_t seed) {
    Volume sub = rotate_volume_trilinear(out.tmpl, out.rotation);
    sub = shift_volume(sub, {-out.shift[0], -out.shift[1], -out.shift[2]});
    if (wedge_deg) sub = apply_wedge(sub, WedgeMask(out.tmpl.n, *wedge_deg));
    const int n = out.tmpl.n;
    if (snr) {
        if (!(*snr > 0.0)) throw std::invalid_argument("make_phantom: snr must be > 0");
        double sum = 0.0, sum2 = 0.0;
        size_t count = 0;
        for (int z = 0; z < n; ++z)
            for (int y = 0; y < n; ++y)
                for (int x = 0; x < n; ++x) {
                    const double cx = sub.coord(x), cy = sub.coord(y), cz = sub.coord(z);
                    if (cx * cx + cy * cy + cz * cz >= 1.0) continue;
                    const double d = sub.at(x, y, z);
                    sum += d;
                    sum2 += d * d;
                    ++count;
                }
        const double mean = sum / (double)count;
        const double var = std::max(0.0, sum2 / (double)count - mean * mean);
        out.noise_sigma = std::sqrt(var / *snr);
        PhiloxStream noise(seed, 3);
        for (double& d : sub.d) d += out.noise_sigma * noise.next_gaussian();
    }
    for (double& d : out.tmpl.d) d = (double)(float)d;
    for (double& d : sub.d) d = (double)(float)d;
    out.sub = std::move(sub);
}
}  // namespace

// volio.cpp:217-317
Phantom make_phantom(const PhantomSpec& spec) {
    if (spec.n < 8 || spec.n % 2 != 0) throw std::invalid_argument("make_phantom: grid size must be even and >= 8");
    if (spec.blobs < 1) throw std::invalid_argument("make_phantom: need at least one blob");
    if (!(spec.support_radius > 0.0 && spec.support_radius < 1.0))
        throw std::invalid_argument("make_phantom: support radius must lie in (0,1)");
    struct Blob {
        Vec3 center;
        Mat3 precision;
        double amplitude;
    };
    PhiloxStream geom(spec.seed, 0);
    std::vector<Blob> blobs;
    for (int b = 0; b < spec.blobs; ++b) {
        const double base = std::exp(geom.next_uniform(std::log(0.028), std::log(0.085)));
        Vec3 sigma;
        for (int i = 0; i < 3; ++i) sigma[i] = base * geom.next_uniform(0.8, 1.25);
        const Rot orient = haar_rotation(geom);
        Vec3 dir{geom.next_gaussian(), geom.next_gaussian(), geom.next_gaussian()};
        if (norm3(dir) < 1e-12) dir = {1, 0, 0};
        const double dn = norm3(dir);
        dir = {dir[0] / dn, dir[1] / dn, dir[2] / dn};
        const double smax = std::max({sigma[0], sigma[1], sigma[2]});
        const double reach = std::max(0.0, spec.support_radius - 3.0 * smax);
        const double radius = reach * std::cbrt(geom.next_unit());
        const double mag = geom.next_uniform(0.5, 1.0) * std::pow(0.05 / base, 0.75);
        const double amp = geom.next_u32() & 1 ? mag : -mag;
        const Mat3 r = orient.matrix();
        Blob blob;
        blob.center = {radius * dir[0], radius * dir[1], radius * dir[2]};
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                double acc = 0;
                for (int q = 0; q < 3; ++q) acc += r[i * 3 + q] * (1.0 / (sigma[q] * sigma[q])) * r[j * 3 + q];
                blob.precision[i * 3 + j] = acc;
            }
        blob.amplitude = amp;
        blobs.push_back(blob);
    }
    Phantom out;
    out.tmpl = Volume(spec.n);
    for (int z = 0; z < spec.n; ++z)
        for (int y = 0; y < spec.n; ++y)
            for (int x = 0; x < spec.n; ++x) {
                const Vec3 p{out.tmpl.coord(x), out.tmpl.coord(y), out.tmpl.coord(z)};
                double val = 0.0;
                for (const auto& blob : blobs) {
                    const Vec3 d{p[0] - blob.center[0], p[1] - blob.center[1], p[2] - blob.center[2]};
                    double q = 0;
                    for (int i = 0; i < 3; ++i) {
                        double row = 0;
                        for (int j = 0; j < 3; ++j) row += blob.precision[i * 3 + j] * d[j];
                        q += d[i] * row;
                    }
                    if (q < 80.0) val += blob.amplitude * std::exp(-0.5 * q);
                }
                out.tmpl.at(x, y, z) = val;
            }
    PhiloxStream rot_stream(spec.seed, 1);
    out.rotation = spec.rotation ? *spec.rotation : haar_rotation(rot_stream);
    PhiloxStream shift_stream(spec.seed, 2);
    if (spec.shift) out.shift = *spec.shift;
    else
        for (int i = 0; i < 3; ++i) out.shift[i] = shift_stream.next_int(-2, 2);
    finish_particle(out, spec.snr, spec.wedge_theta_deg, spec.seed);
    return out;
}

// BASELINE.json template model: sum of isotropic Gaussians, sigma ~ U[1.5,3]
// voxels, amplitude ~ U[0.5,1], centres uniform in the ball of radius 0.6,
// masked to the unit ball; float32-rounded.  Philox stream 0 of `seed`.
Volume gaussian_blob_template(int n, int blobs, uint64_t seed) {
    PhiloxStream geom(seed, 0);
    struct B {
        double cx, cy, cz, s, a;
    };
    std::vector<B> bl;
    for (int b = 0; b < blobs; ++b) {
        const double sig = geom.next_uniform(1.5, 3.0) * (2.0 / n);
        const double amp = geom.next_uniform(0.5, 1.0);
        double dx = geom.next_gaussian(), dy = geom.next_gaussian(), dz = geom.next_gaussian();
        double dn = std::sqrt(dx * dx + dy * dy + dz * dz);
        if (dn < 1e-12) dx = 1, dy = 0, dz = 0, dn = 1;
        const double rad = 0.6 * std::cbrt(geom.next_unit());
        bl.push_back({rad * dx / dn, rad * dy / dn, rad * dz / dn, sig, amp});
    }
    Volume v(n);
    for (int z = 0; z < n; ++z)
        for (int y = 0; y < n; ++y)
            for (int x = 0; x < n; ++x) {
                const double cx = v.coord(x), cy = v.coord(y), cz = v.coord(z);
                if (cx * cx + cy * cy + cz * cz >= 1.0) continue;
                double val = 0.0;
                for (const auto& b : bl) {
                    const double d2 = (cx - b.cx) * (cx - b.cx) + (cy - b.cy) * (cy - b.cy) + (cz - b.cz) * (cz - b.cz);
                    val += b.a * std::exp(-0.5 * d2 / (b.s * b.s));
                }
                v.at(x, y, z) = (double)(float)val;
            }
    return v;
}
// One particle of a BASELINE config: Haar rotation (stream 1), integer shift
// uniform in [-shift_max, shift_max]^3 (stream 2), then the make_phantom
// particle pipeline (volio.cpp:285-314) with noise stream 3 of `seed`.
Phantom make_particle(const Volume& tmpl, uint64_t seed, int shift_max, std::optional<double> snr,
                      std::optional<double> wedge_deg) {
    Phantom out;
    out.tmpl = tmpl;
    PhiloxStream rot_stream(seed, 1);
    out.rotation = haar_rotation(rot_stream);
    PhiloxStream shift_stream(seed, 2);
    for (int i = 0; i < 3; ++i) out.shift[i] = shift_max > 0 ? shift_stream.next_int(-shift_max, shift_max) : 0;
    finish_particle(out, snr, wedge_deg, seed);
    return out;
}

}  // namespace bmo
