// C++ parity test of the reference-facing host API (include/ballmatch_b200.hpp)
// against the CPU oracle's C++ API (oracle/bm_oracle.hpp, test infrastructure).
// Written like the reference's doctest suites (tests/test_basis.cpp,
// tests/test_optimize.cpp): same phantoms on both sides, tolerance-based checks.
// Needs a CUDA device; run through tests/test_cpp_shim.py.
#include <cmath>
#include <cstdio>
#include <functional>
#include <numbers>
#include <stdexcept>
#include <string>
#include <vector>

#define BALLMATCH_B200_WITH_NCCL
#include "ballmatch_b200.hpp"
#include "bm_oracle.hpp"

namespace bm = ballmatch_b200;

static int g_failures = 0;
#define CHECK(cond)                                                             \
    do {                                                                        \
        if (!(cond)) {                                                          \
            std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++g_failures;                                                       \
        }                                                                       \
    } while (0)

template <class E>
static bool throws(const std::function<void()>& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// the product takes FP32 voxels: both sides see the same rounded bytes
static bmo::Volume rounded(const bmo::Volume& v) {
    bmo::Volume r = v;
    for (auto& x : r.d) x = static_cast<double>(static_cast<float>(x));
    return r;
}
static bm::Volume to_product(const bmo::Volume& v) {
    bm::Volume r(v.n);
    r.data = v.d;
    return r;
}
static bm::Rotation to_product(const bmo::Rot& q) { return bm::Rotation(q.w, q.x, q.y, q.z); }
static bmo::Rot to_oracle(const bm::Rotation& q) { return bmo::Rot::make(q.w(), q.x(), q.y(), q.z()); }

static double rel_l2(const std::vector<std::complex<double>>& a, const std::vector<std::complex<double>>& b) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += std::norm(a[i] - b[i]);
        den += std::norm(b[i]);
    }
    return std::sqrt(num / den);
}

// test_basis.cpp:139-190 (counts, roots) against the oracle's build_spec
static void basis_matches_oracle() {
    for (int L : {8, 16}) {
        const double cut = L * std::numbers::pi;
        const auto s = bm::build_spec(L, cut);
        const auto o = bmo::build_spec(L, cut);
        CHECK(s.coeff_count() == o.coeff_total);
        for (int l = 0; l <= L; ++l) {
            CHECK(s.radial_count(l) == o.radial_count(l));
            CHECK(s.block_offset(l) == o.block_off[l]);
            for (int k = 1; k <= s.radial_count(l); ++k) {
                CHECK(std::fabs(s.root(l, k) - o.roots[l][k - 1]) <= 1e-12 * o.roots[l][k - 1]);
                CHECK(std::fabs(s.norm(l, k) - o.norms[l][k - 1]) <= 1e-10 * o.norms[l][k - 1]);
            }
        }
    }
    CHECK(std::fabs(bm::default_lambda_cut(64, 16) - bmo::default_lambda_cut(64, 16)) < 1e-12);
}

// expansion coefficients within 1e-5 relative L2 (the contract)
static void expand_matches_oracle() {
    const auto tmpl = rounded(bmo::gaussian_blob_template(32, 20, 1));
    const auto part = bmo::make_particle(tmpl, 7, 2, 0.5, std::nullopt).sub;
    const double cut = 8 * std::numbers::pi;
    const auto s = bm::build_spec(8, cut);
    const auto o = bmo::build_spec(8, cut);
    for (const auto* v : {&tmpl, &part}) {
        const auto got = bm::expand(to_product(*v), s);
        const auto ref = bmo::expand(*v, o);
        const double err = rel_l2(got.coeffs(), ref.c);
        std::printf("  expand rel L2 %.2e\n", err);
        CHECK(err < 1e-5);
        CHECK(got.real_volume());
    }
}

static bmo::Config oracle_cfg(const bm::OptimizerConfig& c) {
    bmo::Config o;
    o.l_max = c.l_max;
    o.lambda_cut = c.lambda_cut;
    o.fixed_bands = c.fixed_bands;
    o.seed_grid_step = c.seed_grid_step;
    o.max_candidates = c.max_candidates;
    o.newton_max_iter = c.newton_max_iter;
    o.grad_tol = c.grad_tol;
    o.step_damping = c.step_damping;
    o.shift_radius = c.shift_radius;
    o.shift_step = c.shift_step;
    return o;
}

// test_optimize.cpp:199-221 (noiseless: exact shift, < 0.5 deg) and :238-252
// (wedge), here against the oracle's align on the same bytes
static void align_matches_oracle() {
    const auto tmpl = rounded(bmo::gaussian_blob_template(32, 20, 3));
    bm::OptimizerConfig cfg;
    cfg.l_max = 8;
    cfg.lambda_cut = 8 * std::numbers::pi;
    cfg.fixed_bands = {4, 8};
    cfg.max_candidates = 8;
    cfg.shift_radius = 2;
    cfg.shift_step = 2;
    const auto ocfg = oracle_cfg(cfg);
    struct Case {
        std::optional<double> snr, wedge;
    };
    for (const Case& c : {Case{std::nullopt, std::nullopt}, Case{1.0, 60.0}}) {
        std::vector<bmo::Phantom> ph;
        std::vector<bm::Volume> subs;
        for (int p = 0; p < 3; ++p) {
            ph.push_back(bmo::make_particle(tmpl, 300 + p, 2, c.snr, c.wedge));
            subs.push_back(to_product(ph.back().sub));
        }
        std::optional<bm::WedgeMask> wm;
        std::optional<bmo::WedgeMask> owm;
        if (c.wedge) {
            wm = bm::build_wedge_mask(32, *c.wedge);
            owm = bmo::WedgeMask(32, *c.wedge);
        }
        const auto got = bm::align_batch(to_product(tmpl), subs, cfg, wm);
        CHECK(got.size() == 3);
        for (int p = 0; p < 3; ++p) {
            const auto ref = bmo::align(tmpl, ph[p].sub, ocfg, owm);
            const double ang = bmo::geodesic_degrees(to_oracle(got[p].rotation), ref.rotation);
            std::printf("  particle %d: shift (%d,%d,%d) vs (%d,%d,%d), %.4f deg, score %.6f vs %.6f\n", p,
                        got[p].shift[0], got[p].shift[1], got[p].shift[2], ref.shift[0], ref.shift[1],
                        ref.shift[2], ang, got[p].score, ref.score);
            CHECK(got[p].shift == ref.shift);
            CHECK(ang < 0.5);
            CHECK(std::fabs(got[p].score - ref.score) <= 1e-4 * std::fabs(ref.score));
            if (!c.snr) {  // noiseless: the truth itself
                CHECK(got[p].shift == ph[p].shift);
                CHECK(bm::geodesic_degrees(got[p].rotation, to_product(ph[p].rotation)) < 0.5);
            }
        }
        // single-particle align() gives the batch's answer
        const auto one = bm::align(to_product(tmpl), subs[0], cfg, wm);
        CHECK(one.shift == got[0].shift);
        CHECK(bm::geodesic_degrees(one.rotation, got[0].rotation) < 1e-6);
    }
}

// average = (1/P) sum_p rotate_expansion(expand(shift_volume(sub_p, s_p)), g_p^-1)
static void average_matches_oracle() {
    const auto tmpl = rounded(bmo::gaussian_blob_template(32, 20, 21));
    bm::OptimizerConfig cfg;
    cfg.l_max = 8;
    cfg.lambda_cut = 8 * std::numbers::pi;
    cfg.fixed_bands = {4, 8};
    cfg.max_candidates = 8;
    cfg.shift_radius = 2;
    std::vector<bm::Volume> subs;
    std::vector<bmo::Volume> osubs;
    for (int p = 0; p < 4; ++p) {
        osubs.push_back(bmo::make_particle(tmpl, 900 + p, 2, 1.0, std::nullopt).sub);
        subs.push_back(to_product(osubs.back()));
    }
    bm::Aligner a(to_product(tmpl), cfg);
    const auto res = a.align_batch(subs);
    a.accumulate_average(subs, res);
    CHECK(a.average_count() == 4);
    const auto avg = a.average();
    const auto o = bmo::build_spec(8, cfg.lambda_cut);
    std::vector<std::complex<double>> ref(o.coeff_total);
    for (int p = 0; p < 4; ++p) {
        const auto f = bmo::expand(bmo::shift_volume(osubs[p], res[p].shift), o);
        const auto r = bmo::rotate_expansion(f, to_oracle(res[p].rotation).inverse());
        for (size_t i = 0; i < ref.size(); ++i) ref[i] += r.c[i] / 4.0;
    }
    const double err = rel_l2(avg.coeffs(), ref);
    std::printf("  average rel L2 %.2e\n", err);
    CHECK(err < 1e-5);
    // the average of aligned particles correlates with the template
    const auto t_hat = bm::expand(to_product(tmpl), a.spec());
    std::complex<double> dot = 0.0;
    for (size_t i = 0; i < ref.size(); ++i) dot += std::conj(t_hat.coeffs()[i]) * avg.coeffs()[i];
    CHECK(dot.real() / (t_hat.norm() * avg.norm()) > 0.5);
}

// One process, one thread per device, NCCL: the multi-device driver
// gives the single-device results bit for bit and the same average, and the world-1
// allreduce of Aligner::allreduce_average leaves the numerator unchanged.
static void multi_device_matches_single() {
#ifdef BALLMATCH_B200_WITH_NCCL
    const auto tmpl = rounded(bmo::gaussian_blob_template(32, 20, 21));
    bm::OptimizerConfig cfg;
    cfg.l_max = 8;
    cfg.lambda_cut = 8 * std::numbers::pi;
    cfg.fixed_bands = {4, 8};
    cfg.max_candidates = 8;
    cfg.shift_radius = 2;
    std::vector<bm::Volume> subs;
    for (int p = 0; p < 7; ++p) subs.push_back(to_product(bmo::make_particle(tmpl, 950 + p, 2, 1.0, std::nullopt).sub));
    bm::Aligner single(to_product(tmpl), cfg);
    const auto ref = single.align_batch(subs);
    single.accumulate_average(subs, ref);
    const auto ref_avg = single.average();
    // world-1 NCCL allreduce through Aligner::allreduce_average: same numerator and count
    {
        ncclComm_t comm;
        int dev = 0;
        CHECK(ncclCommInitAll(&comm, 1, &dev) == ncclSuccess);
        single.allreduce_average(comm, nullptr);
        CHECK(single.average_count() == 7);
        CHECK(rel_l2(single.average().coeffs(), ref_avg.coeffs()) == 0.0);
        ncclCommDestroy(comm);
    }
    int n_dev = 0;
    cudaGetDeviceCount(&n_dev);
    std::vector<int> devs;
    for (int d = 0; d < std::min(n_dev, 8); ++d) devs.push_back(d);
    bm::MultiDeviceAligner multi(to_product(tmpl), cfg, devs, std::nullopt, 2);  // chunks of 2 particles
    const auto res = multi.align_and_average(subs);
    for (size_t p = 0; p < subs.size(); ++p) {
        CHECK(res[p].shift == ref[p].shift);
        CHECK(res[p].rotation.w() == ref[p].rotation.w() && res[p].rotation.x() == ref[p].rotation.x());
        CHECK(res[p].score == ref[p].score);
    }
    long long total = 0;
    for (long long c : multi.particles_per_device()) total += c;
    CHECK(total == 7);
    const double err = rel_l2(multi.average().coeffs(), ref_avg.coeffs());
    std::printf("  %d device(s), average rel L2 vs single device %.2e\n", (int)devs.size(), err);
    CHECK(err < 1e-12);
#else
    std::printf("  built without BALLMATCH_B200_WITH_NCCL\n");
    CHECK(false);
#endif
}

// synthesize (basis.cpp:332-419) of the average against the oracle's, FP64 both sides
static void synthesize_matches_oracle() {
    const auto tmpl = rounded(bmo::gaussian_blob_template(32, 20, 5));
    const double cut = 8 * std::numbers::pi;
    const auto s = bm::build_spec(8, cut);
    const auto o = bmo::build_spec(8, cut);
    const auto e = bm::expand(to_product(tmpl), s);
    const auto v = bm::synthesize(e, 32);
    bmo::Expansion oe;
    oe.spec = &o;
    oe.c = e.coeffs();
    oe.real = true;
    const auto ov = bmo::synthesize(oe, 32);
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < v.data.size(); ++i) {
        num += (v.data[i] - ov.d[i]) * (v.data[i] - ov.d[i]);
        den += ov.d[i] * ov.d[i];
    }
    std::printf("  synthesize rel L2 %.2e\n", std::sqrt(num / den));
    CHECK(std::sqrt(num / den) < 1e-10);
}

// error behaviour mirrors the reference (optimize.cpp:153-177, 423-449)
static void errors_match_reference() {
    const auto tmpl = to_product(rounded(bmo::gaussian_blob_template(32, 20, 1)));
    bm::OptimizerConfig cfg;
    cfg.l_max = 8;
    cfg.lambda_cut = 8 * std::numbers::pi;
    cfg.fixed_bands = {4, 8};
    auto bad = cfg;
    bad.fixed_bands = {8, 4};
    CHECK(throws<std::invalid_argument>([&] { bad.validate(); }));
    bad = cfg;
    bad.fixed_bands = {4, 9};
    CHECK(throws<std::invalid_argument>([&] { bad.validate(); }));
    bad = cfg;
    bad.max_candidates = 0;
    CHECK(throws<std::invalid_argument>([&] { bad.validate(); }));
    bad = cfg;
    bad.seed_grid_step = 4.0;
    CHECK(throws<std::invalid_argument>([&] { bad.validate(); }));
    bm::Volume zero(32);
    CHECK(throws<std::invalid_argument>([&] { bm::align(tmpl, zero, cfg); }));
    CHECK(throws<std::invalid_argument>([&] { bm::align(zero, tmpl, cfg); }));
    CHECK(throws<std::invalid_argument>([&] { bm::align(tmpl, bm::Volume(16), cfg); }));
    CHECK(throws<std::invalid_argument>([&] { bm::build_wedge_mask(32, 0.0); }));
    CHECK(throws<std::invalid_argument>([&] { bm::build_spec(-1, 3.0); }));
    CHECK(throws<std::invalid_argument>([&] { bm::build_spec(4, 3.0); }));  // lambda_cut < pi
    bm::Aligner a(tmpl, cfg);
    CHECK(throws<std::domain_error>([&] { a.average(); }));
}

int main() {
    const std::vector<std::pair<const char*, void (*)()>> tests = {
        {"basis_matches_oracle", basis_matches_oracle},
        {"expand_matches_oracle", expand_matches_oracle},
        {"align_matches_oracle", align_matches_oracle},
        {"average_matches_oracle", average_matches_oracle},
        {"multi_device_matches_single", multi_device_matches_single},
        {"synthesize_matches_oracle", synthesize_matches_oracle},
        {"errors_match_reference", errors_match_reference},
    };
    for (const auto& [name, fn] : tests) {
        const int before = g_failures;
        std::printf("[ RUN ] %s\n", name);
        try {
            fn();
        } catch (const std::exception& e) {
            std::printf("  unexpected exception: %s\n", e.what());
            ++g_failures;
        }
        std::printf("[ %s ] %s\n", g_failures == before ? "OK" : "FAIL", name);
    }
    std::printf("%d failure(s)\n", g_failures);
    return g_failures ? 1 : 0;
}
