// bm_oracle — CPU restatement of the reference (arXiv 2509.01180 "ballmatch")
// alignment hot path.  TEST INFRASTRUCTURE ONLY: used by tests/, by
// __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
// legs as the checker and the CPU baseline.  The product (libballmatch_b200)
// never links or calls this code.
//
// The reference cannot be compiled in this container (Eigen3, FFTW3 and its
// vendored doctest/CLI11/json headers are absent; proj/CMakeLists.txt:10-17),
// so this file restates its algorithms function by function, in FP64, with the
// Eigen/FFTW arithmetic replaced by plain loops (a mixed-radix complex FFT for
// FFTW's r2c/c2r, a 3x3 full-pivot LU with Eigen's rank rule for FullPivLU).
// Each function cites the reference file:line it follows (paths relative to
// the reference's proj/).  The restatement is pinned against the reference's
// own known-answer tests in tests/test_oracle_*.py.
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <map>
#include <optional>
#include <vector>

namespace bmo {

using cd = std::complex<double>;
constexpr double kPi = 3.14159265358979323846;

// ---------------------------------------------------------------- philox
// include/ballmatch/philox.hpp:13-87
struct Philox {
    static std::array<uint32_t, 4> round10(std::array<uint32_t, 4> ctr, std::array<uint32_t, 2> key);
};
class PhiloxStream {
public:
    explicit PhiloxStream(uint64_t seed, uint32_t stream = 0);
    uint32_t next_u32();
    double next_unit();
    double next_uniform(double lo, double hi);
    double next_gaussian();
    int next_int(int lo, int hi);

private:
    std::array<uint32_t, 2> key_;
    uint32_t stream_;
    uint32_t ctr_ = 0;
    std::array<uint32_t, 4> block_{};
    int lane_ = 4;
    double spare_ = 0.0;
    bool have_spare_ = false;
};

// ---------------------------------------------------------------- rotation
// include/ballmatch/rotation.hpp, src/rotation.cpp
struct Euler {
    double alpha = 0, beta = 0, gamma = 0;
};
using Mat3 = std::array<double, 9>;  // row-major
using Vec3 = std::array<double, 3>;
struct Rot {
    double w = 1, x = 0, y = 0, z = 0;
    static Rot make(double w, double x, double y, double z);  // normalizing ctor
    static Rot from_axis_angle(Vec3 axis, double angle);
    static Rot from_euler_zyz(double a, double b, double g);
    Mat3 matrix() const;
    Euler euler_zyz() const;
    Rot inverse() const { return {w, -x, -y, -z}; }
    Rot operator*(const Rot& r) const;
    double angle_to(const Rot& o) const;
    double angle() const { return angle_to(Rot{}); }
};
double geodesic_degrees(const Rot& a, const Rot& b);

// ---------------------------------------------------------------- volume
// include/ballmatch/volume.hpp, src/volume.cpp
struct Volume {
    int n = 0;
    std::vector<double> d;
    Volume() = default;
    explicit Volume(int n_) : n(n_), d((size_t)n_ * n_ * n_, 0.0) {}
    size_t index(int x, int y, int z) const { return ((size_t)z * n + y) * n + x; }
    double at(int x, int y, int z) const { return d[index(x, y, z)]; }
    double& at(int x, int y, int z) { return d[index(x, y, z)]; }
    double coord(int i) const { return (i - n / 2) * (2.0 / n); }
};
double volume_l2_norm(const Volume& v);
double sample_trilinear(const Volume& v, double x, double y, double z);
Volume shift_volume(const Volume& v, const std::array<int, 3>& s);

// ---------------------------------------------------------------- numerics
double sph_jl(int l, double x);
double sph_jl_prime(int l, double x);
double bessel_root(int l, int k);
std::vector<std::vector<double>> bessel_root_table(int l_max, double lambda_cut);
struct GL {
    std::vector<double> nodes, weights;
};
GL gauss_legendre(int n);
GL gauss_legendre01(int n);
inline size_t tri_index(int l, int m) { return (size_t)l * (l + 1) / 2 + m; }
inline size_t tri_count(int l_max) { return (size_t)(l_max + 1) * (l_max + 2) / 2; }
void legendre_table(int l_max, double u, double* out);

// FFT (FFTW semantics: unnormalized forward e^{-2 pi i}, row-major dims, last fastest)
void fft_r2c_3d(int n, const double* in, cd* out);         // out n*n*(n/2+1)
void fft_c2r_3d(int n, const cd* in, double* out);         // unnormalized inverse
void dft_r2c_rows(int n, int count, const double* in, cd* out);

// ---------------------------------------------------------------- basis
// include/ballmatch/basis.hpp, src/basis.cpp
struct Spec {
    int l_max = 0;
    double lambda_cut = 0;
    std::vector<std::vector<double>> roots, norms;  // [l][k-1]
    std::vector<size_t> block_off, pair_off;
    size_t coeff_total = 0, pair_total = 0;
    // ExpandPlan (basis.cpp:25-32, 174-219)
    int n_r = 0, n_theta = 0, n_phi = 0;
    std::vector<double> r, sin_theta, cos_theta, ptab, radial;
    int radial_count(int l) const { return (int)roots[l].size(); }
    size_t index_of(int k, int l, int m) const {
        return block_off[l] + (size_t)(k - 1) * (2 * l + 1) + (m + l);
    }
    void build_plan();
};
Spec build_spec(int l_max, double lambda_cut);
double default_lambda_cut(int n, int l_max);
cd spherical_harmonic(int l, int m, double theta, double phi);

struct Expansion {
    const Spec* spec = nullptr;
    std::vector<cd> c;
    bool real = false;
    double energy() const;
    double norm() const;
};
Expansion expand(const Volume& v, const Spec& spec);
Volume synthesize(const Expansion& e, int n);

// ---------------------------------------------------------------- steer
// src/steer.cpp
struct LittleD {
    int l_max = -1, order = 0;
    std::vector<std::vector<double>> value, d1, d2;  // [l] (2l+1)^2 row-major
};
LittleD little_d_stack(int l_max, double beta, int order);
std::vector<std::vector<cd>> wigner_D(int l_max, const Rot& g);
Expansion rotate_expansion(const Expansion& e, const Rot& g);

// ---------------------------------------------------------------- xcorr
// include/ballmatch/xcorr.hpp, src/xcorr.cpp
struct Xi {
    int l_max = -1;
    std::array<int, 3> shift{0, 0, 0};
    std::vector<std::vector<cd>> b;  // [l] (2l+1)^2 row-major (m row, m' col)
    Xi() = default;
    Xi(int L, std::array<int, 3> s);
    cd& at(int l, int m, int mp) { return b[l][(size_t)(m + l) * (2 * l + 1) + (mp + l)]; }
    cd at(int l, int m, int mp) const { return b[l][(size_t)(m + l) * (2 * l + 1) + (mp + l)]; }
    double total_energy() const;
};
Xi xi_coefficients(const Expansion& t, const Expansion& f, std::array<int, 3> shift = {0, 0, 0});
double energy_ratio(const Xi& xi, int l_cut);
std::vector<int> select_bands(const Xi& xi, const std::vector<double>& thresholds);
struct Deriv {
    double value = 0, imag = 0;
    Vec3 grad{0, 0, 0};
    Mat3 hess{0, 0, 0, 0, 0, 0, 0, 0, 0};
};
Deriv correlation_derivatives(const Xi& xi, const Euler& e, int l_cut, int order);
Xi xi_compose_right(const Xi& xi, const Rot& a, int l_limit = -1);

struct WedgeMask {
    int n = 0;
    double theta_max_deg = 90.0, tan_theta = 0.0;
    bool all_pass = true;
    Vec3 tilt_axis{0, 1, 0}, perp{1, 0, 0};
    WedgeMask() = default;
    WedgeMask(int n, double theta_deg, Vec3 axis = {0, 1, 0});
    bool keeps_direction(const Vec3& nu) const;
    bool keeps(int fx, int fy, int fz) const { return keeps_direction({(double)fx, (double)fy, (double)fz}); }
    double kept_fraction() const;
};
constexpr double kWedgeTaperDeg = 6.0;
double wedge_keep_profile(const WedgeMask& m, const Vec3& nu, double taper_deg);
Volume apply_wedge(const Volume& v, const WedgeMask& m);
Volume apply_wedge_taper(const Volume& v, const WedgeMask& m, double taper_deg = kWedgeTaperDeg);
Xi wedge_power_kernel(const Volume& tmpl, const WedgeMask& m, int l_max,
                      double taper_deg = kWedgeTaperDeg);
// the two SH analyses wedge_power_kernel contracts (rank-1 factors), for the
// product's factored kernel: xi_wp[l][m,m'] = conj(chi_hat[l,m]) q_hat[l,m'] / total
struct WedgePowerFactors {
    std::vector<cd> chi_hat, q_hat;  // tri_count(l_max), m >= 0
    double total = 0;
};
WedgePowerFactors wedge_power_factors(const Volume& tmpl, const WedgeMask& m, int l_max,
                                      double taper_deg = kWedgeTaperDeg);

// ---------------------------------------------------------------- optimize
// include/ballmatch/optimize.hpp, src/optimize.cpp
struct Config {
    int l_max = 42;
    double lambda_cut = 0.0;
    std::vector<int> fixed_bands{7, 12, 33};
    double seed_grid_step = kPi / 8;
    int max_candidates = 20;
    int newton_max_iter = 30;
    double grad_tol = 1e-7;
    double step_damping = 1e-3;
    int shift_radius = 4;
    int shift_step = 2;
    int threads = 0;
    std::vector<double> band_thresholds{0.5, 0.25, 0.05};
    bool auto_bands = false;        // bands from the zero-shift kernel's energy ratios
    bool prune_after_band = false;  // keep only the lowest band's winner for the rest
    void validate() const;
};
struct TraceRow {
    int band, iteration;
    double alpha, beta, gamma, score, grad_norm;
};
struct RefineResult {
    Rot rotation;
    double score = 0;
    bool converged = false;
    std::vector<TraceRow> trace;
    std::map<int, long> evals;
};
struct Candidate {
    Rot rotation;
    double score = 0;
    long flat_index = -1;
};
std::vector<double> grid_scores(const Xi& xi, int l_cut, double step);
struct Baseline {  // BaselineResult (optimize.hpp:96-101)
    Rot rotation;
    double score = 0;
    long evaluations = 0;
};
Baseline exhaustive_baseline(const Xi& xi, int l_cut, double step);
long baseline_evaluation_count(double step);
std::vector<Candidate> seed_candidates(const Xi& xi, int l_low, double step, int max_candidates,
                                       const Xi* wedge_power = nullptr);
RefineResult refine(const Xi& xi, const Rot& start, const std::vector<int>& bands,
                    const Config& cfg, const Xi* wedge_power = nullptr);
struct ShiftOutcome {
    std::array<int, 3> shift{0, 0, 0};
    double norm_score = -1e308 * 10;  // -inf
    double raw_score = 0, subtomo_norm = 0;
    RefineResult refined;
    long candidates = 0;
    std::map<int, long> evals;
    bool valid = false;
};
ShiftOutcome search_one_shift(const Volume& f_w, const std::array<int, 3>& s,
                              const Expansion& t_hat, double t_norm, const std::vector<int>& bands,
                              const Config& cfg, const Xi* wedge_power);
struct AlignResult {
    std::array<int, 3> shift{0, 0, 0};
    Rot rotation;
    double score = 0;
    bool converged = false;
    long candidates_evaluated = 0;
    std::map<int, long> evals;
    double template_norm = 0, subtomo_norm = 0;
    int windows = 0;
    std::vector<int> bands;
};
AlignResult align(const Volume& tmpl, const Volume& sub, const Config& cfg,
                  const std::optional<WedgeMask>& wedge = std::nullopt);

// ---------------------------------------------------------------- volio
// src/volio.cpp:195-317
Volume rotate_volume_trilinear(const Volume& v, const Rot& g);
Rot haar_rotation(PhiloxStream& rng);
struct PhantomSpec {
    int n = 64, blobs = 6;
    double support_radius = 0.8;
    uint64_t seed = 0;
    std::optional<double> snr, wedge_theta_deg;
    std::optional<Rot> rotation;
    std::optional<std::array<int, 3>> shift;
};
struct Phantom {
    Volume tmpl, sub;
    Rot rotation;
    std::array<int, 3> shift{0, 0, 0};
    double noise_sigma = 0;
};
Phantom make_phantom(const PhantomSpec& spec);

// BASELINE.json config generator (isotropic-Gaussian template; the particle
// pipeline of make_phantom, volio.cpp:285-314).  See DESIGN.md "Synthetic inputs".
Volume gaussian_blob_template(int n, int blobs, uint64_t seed);
Phantom make_particle(const Volume& tmpl, uint64_t seed, int shift_max, std::optional<double> snr,
                      std::optional<double> wedge_deg);

}  // namespace bmo
