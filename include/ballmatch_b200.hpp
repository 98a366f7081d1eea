// ballmatch_b200.hpp — C++ host API of the B200 path, mirroring the reference's
// public alignment API (proj/include/ballmatch/{volume,basis,rotation,xcorr,
// optimize}.hpp) on top of the C ABI in ballmatch_b200.h.
//
// Names, argument meaning and error behaviour follow the reference:
//   build_spec / default_lambda_cut / expand         basis.hpp:60-95
//   Rotation / EulerZyz / geodesic_degrees           rotation.hpp:7-53
//   WedgeMask / build_wedge_mask / apply_wedge_taper xcorr.hpp:82-125
//   OptimizerConfig / AlignmentResult / align        optimize.hpp:15-94
// plus the two entry points the reference lacks: align_batch
// (align() per particle, sharing the template state) and the coefficient-space
// average (sum_p rotate_expansion(f_hat_{p,s_p}, g_p^-1) / P, steer.hpp:39).
// std::invalid_argument / std::domain_error are thrown where the reference
// throws them; CUDA failures throw std::runtime_error.  There is no CPU path:
// every call needs a CUDA device.
//
// Header-only; link with libballmatch_b200.so and cudart.  Define
// BALLMATCH_B200_WITH_NCCL before including to get Aligner::allreduce_average.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numbers>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>
#include <atomic>
#include <exception>

#include "ballmatch_b200.h"

#ifdef BALLMATCH_B200_WITH_NCCL
#include <nccl.h>
#endif

namespace ballmatch_b200 {

using cdouble = std::complex<double>;

// FP32 evaluation defaults: the reference's 1e-12 acceptance
// slack and 1e-7 gradient tolerance assume FP64 scores.
inline constexpr double kFp32AcceptTol = 1e-6;
inline constexpr double kFp32GradTol = 1e-5;
inline constexpr double kWedgeTaperDeg = 6.0;  // xcorr.hpp:114 (fixed on the device path)

namespace detail {

[[noreturn]] inline void raise(int rc, const std::string& what) {
    const std::string msg = what + ": " + bm_last_error();
    switch (rc) {
        case BM_ERR_ARG:
        case BM_ERR_STATE:
            throw std::invalid_argument(msg);
        case BM_ERR_DOMAIN:
            throw std::domain_error(msg);
        default:
            throw std::runtime_error(msg);
    }
}
inline void check(int rc, const char* what) {
    if (rc != BM_OK) raise(rc, what);
}
inline void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
inline int current_device() {
    int d = 0;
    cuda(cudaGetDevice(&d), "cudaGetDevice");
    return d;
}

// caller-side device buffer (RAII)
template <class T>
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(size_t n) { resize(n); }
    ~DeviceBuffer() {
        if (p_) cudaFree(p_);
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    void resize(size_t n) {
        if (n <= n_) return;
        if (p_) cudaFree(p_);
        p_ = nullptr;
        n_ = 0;
        cuda(cudaMalloc(&p_, n * sizeof(T)), "cudaMalloc");
        n_ = n;
    }
    T* get() const { return p_; }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

struct ContextDeleter {
    void operator()(bm_context* c) const { bm_context_destroy(c); }
};
using ContextPtr = std::shared_ptr<bm_context>;

inline ContextPtr make_context(int device, int n, int l_max, double cut) {
    bm_context* c = nullptr;
    check(bm_context_create(device, n, l_max, cut, &c), "build_spec");
    return ContextPtr(c, ContextDeleter{});
}

// Expansion plans are built once per (l_max, lambda_cut, n, device) and
// reused, like the reference's call_once plan cache (basis.cpp:205-219).
struct PlanRegistry {
    std::mutex mu;
    std::map<std::tuple<int, double, int, int>, ContextPtr> plans;
    static PlanRegistry& get() {
        static PlanRegistry r;
        return r;
    }
    ContextPtr plan(int l_max, double cut, int n, int device) {
        std::lock_guard<std::mutex> lock(mu);
        auto& slot = plans[{l_max, cut, n, device}];
        if (!slot) slot = make_context(device, n, l_max, cut);
        return slot;
    }
};

}  // namespace detail

// ------------------------------------------------------------------ Volume (volume.hpp:11-34)
struct Volume {
    int n = 0;
    double voxel_size = 1.0;
    std::vector<double> data;

    Volume() = default;
    Volume(int n_, double voxel_size_ = 1.0)
        : n(n_), voxel_size(voxel_size_), data(static_cast<size_t>(n_) * n_ * n_, 0.0) {
        if (n_ < 2) throw std::invalid_argument("Volume: grid size must be >= 2");
    }
    size_t index(int x, int y, int z) const { return (static_cast<size_t>(z) * n + y) * n + x; }
    double& at(int x, int y, int z) { return data[index(x, y, z)]; }
    double at(int x, int y, int z) const { return data[index(x, y, z)]; }
    double coord(int i) const { return (i - n / 2) * (2.0 / n); }
    size_t size() const { return data.size(); }
};

inline double volume_l2_norm(const Volume& v) {
    double s = 0.0;
    for (double x : v.data) s += x * x;
    return std::sqrt(s);
}

// ------------------------------------------------------------------ rotations (rotation.hpp)
struct EulerZyz {
    double alpha = 0.0, beta = 0.0, gamma = 0.0;
};

class Rotation {
public:
    Rotation() = default;
    Rotation(double w, double x, double y, double z) {
        const double s = std::sqrt(w * w + x * x + y * y + z * z);
        if (!(s > 0.0)) throw std::invalid_argument("Rotation: zero quaternion");
        w_ = w / s, x_ = x / s, y_ = y / s, z_ = z / s;
    }
    static Rotation identity() { return {}; }
    static Rotation from_axis(int axis, double angle) {
        const double h = 0.5 * angle, s = std::sin(h);
        return Rotation(std::cos(h), axis == 0 ? s : 0.0, axis == 1 ? s : 0.0, axis == 2 ? s : 0.0);
    }
    // Rz(alpha) Ry(beta) Rz(gamma), active (rotation.cpp:31-34)
    static Rotation from_euler_zyz(double a, double b, double g) {
        return from_axis(2, a) * from_axis(1, b) * from_axis(2, g);
    }
    static Rotation from_euler_zyz(const EulerZyz& e) { return from_euler_zyz(e.alpha, e.beta, e.gamma); }

    double w() const { return w_; }
    double x() const { return x_; }
    double y() const { return y_; }
    double z() const { return z_; }
    std::array<double, 4> quat() const { return {w_, x_, y_, z_}; }

    // row-major 3x3
    std::array<double, 9> matrix() const {
        const double w = w_, x = x_, y = y_, z = z_;
        return {1 - 2 * (y * y + z * z), 2 * (x * y - w * z),     2 * (x * z + w * y),
                2 * (x * y + w * z),     1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                2 * (x * z - w * y),     2 * (y * z + w * x),     1 - 2 * (x * x + y * y)};
    }
    // beta in [0, pi] with the pole conventions of rotation.cpp:77-93
    EulerZyz euler_zyz() const {
        const auto m = matrix();
        EulerZyz e;
        const double sb = std::hypot(m[2], m[5]);
        e.beta = std::atan2(sb, m[8]);
        if (sb > 1e-12) {
            e.alpha = std::atan2(m[5], m[2]);
            e.gamma = std::atan2(m[7], -m[6]);
        } else if (m[8] > 0.0) {
            e.alpha = std::atan2(m[3], m[0]);
        } else {
            e.alpha = std::atan2(-m[3], -m[0]);
        }
        return e;
    }
    Rotation inverse() const { return raw(w_, -x_, -y_, -z_); }
    // (a * b) applies b first (rotation.cpp:95-100)
    Rotation operator*(const Rotation& b) const {
        return Rotation(w_ * b.w_ - x_ * b.x_ - y_ * b.y_ - z_ * b.z_,
                        w_ * b.x_ + x_ * b.w_ + y_ * b.z_ - z_ * b.y_,
                        w_ * b.y_ - x_ * b.z_ + y_ * b.w_ + z_ * b.x_,
                        w_ * b.z_ + x_ * b.y_ - y_ * b.x_ + z_ * b.w_);
    }
    // geodesic angle, radians in [0, pi] (rotation.cpp:102-107)
    double angle_to(const Rotation& o) const {
        const Rotation d = inverse() * o;
        return 2.0 * std::atan2(std::sqrt(d.x_ * d.x_ + d.y_ * d.y_ + d.z_ * d.z_), std::fabs(d.w_));
    }
    double angle() const { return angle_to({}); }

private:
    static Rotation raw(double w, double x, double y, double z) {
        Rotation r;
        r.w_ = w, r.x_ = x, r.y_ = y, r.z_ = z;
        return r;
    }
    double w_ = 1.0, x_ = 0.0, y_ = 0.0, z_ = 0.0;
};

inline double geodesic_degrees(const Rotation& a, const Rotation& b) {
    return a.angle_to(b) * 180.0 / std::numbers::pi;
}

// ------------------------------------------------------------------ basis (basis.hpp:28-95)
struct BasisIndex {
    int k = 1, l = 0, m = 0;
};

double default_lambda_cut(int n, int l_max);

class BasisSpec {
public:
    BasisSpec() = default;
    int l_max() const { return impl().l_max; }
    double lambda_cut() const { return impl().cut; }
    int radial_count(int l) const { return static_cast<int>(impl().roots.at(l).size()); }
    double root(int l, int k) const { return impl().roots.at(l).at(k - 1); }
    double norm(int l, int k) const { return impl().norms.at(l).at(k - 1); }
    size_t coeff_count() const { return impl().coeffs; }
    size_t pair_count() const { return impl().pairs; }
    size_t block_offset(int l) const { return impl().block_off.at(l); }
    size_t index_of(const BasisIndex& i) const {
        return block_offset(i.l) + static_cast<size_t>(i.k - 1) * (2 * i.l + 1) + (i.m + i.l);
    }
    bool compatible(const BasisSpec& o) const {
        return valid() && o.valid() && l_max() == o.l_max() && lambda_cut() == o.lambda_cut();
    }
    bool valid() const { return m_impl != nullptr; }

    // device expansion plan (operator for an n^3 grid on `device`, built once)
    bm_context* plan(int n, int device = -1) const {
        return detail::PlanRegistry::get().plan(l_max(), lambda_cut(), n, device < 0 ? detail::current_device() : device)
            .get();
    }

    struct Impl {
        int l_max = 0;
        double cut = 0.0;
        std::vector<std::vector<double>> roots, norms;
        std::vector<size_t> block_off;
        size_t coeffs = 0, pairs = 0;
    };
    const Impl& impl() const {
        if (!m_impl) throw std::invalid_argument("BasisSpec: not built (use build_spec)");
        return *m_impl;
    }

private:
    friend BasisSpec build_spec(int, double);
    std::shared_ptr<const Impl> m_impl;
};

// build_spec (basis.cpp:88-115): retained (l, k) with lambda_lk <= lambda_cut
inline BasisSpec build_spec(int l_max, double lambda_cut) {
    if (l_max < 0) throw std::invalid_argument("build_spec: l_max must be >= 0");
    // basis-only device context (n = 0): roots and norms come from the library
    auto ctx = detail::PlanRegistry::get().plan(l_max, lambda_cut, 0, detail::current_device());
    auto impl = std::make_shared<BasisSpec::Impl>();
    impl->l_max = l_max;
    impl->cut = lambda_cut;
    impl->roots.resize(l_max + 1);
    impl->norms.resize(l_max + 1);
    impl->block_off.resize(l_max + 1);
    for (int l = 0; l <= l_max; ++l) {
        const int k = bm_context_roots(ctx.get(), l, nullptr, nullptr);
        if (k < 0) detail::raise(BM_ERR_STATE, "build_spec");
        std::vector<double> r(k), c(k);
        bm_context_roots(ctx.get(), l, r.data(), c.data());
        impl->roots[l] = r;
        impl->norms[l] = c;
        impl->block_off[l] = impl->coeffs;
        impl->coeffs += static_cast<size_t>(k) * (2 * l + 1);
        impl->pairs += k;
    }
    BasisSpec s;
    s.m_impl = impl;
    return s;
}

inline double default_lambda_cut(int n, int l_max) { return bm_default_lambda_cut(n, l_max); }

// complex coefficients over the retained index set (basis.hpp:67-91)
class BallExpansion {
public:
    BallExpansion() = default;
    explicit BallExpansion(BasisSpec spec, bool real_volume = false)
        : m_spec(std::move(spec)), m_coeffs(m_spec.coeff_count()), m_real(real_volume) {}
    const BasisSpec& spec() const { return m_spec; }
    bool real_volume() const { return m_real; }
    void set_real_volume(bool r) { m_real = r; }
    cdouble operator[](const BasisIndex& i) const { return m_coeffs[m_spec.index_of(i)]; }
    cdouble& operator[](const BasisIndex& i) { return m_coeffs[m_spec.index_of(i)]; }
    const std::vector<cdouble>& coeffs() const { return m_coeffs; }
    std::vector<cdouble>& coeffs() { return m_coeffs; }
    const cdouble* block(int l) const { return m_coeffs.data() + m_spec.block_offset(l); }
    cdouble* block(int l) { return m_coeffs.data() + m_spec.block_offset(l); }
    double energy() const {
        double s = 0.0;
        for (const auto& c : m_coeffs) s += std::norm(c);
        return s;
    }
    double norm() const { return std::sqrt(energy()); }

private:
    BasisSpec m_spec;
    std::vector<cdouble> m_coeffs;
    bool m_real = false;
};

namespace detail {
inline std::vector<float> to_f32(const Volume& v) {
    std::vector<float> f(v.data.size());
    for (size_t i = 0; i < f.size(); ++i) f[i] = static_cast<float>(v.data[i]);
    return f;
}
}  // namespace detail

// expand (basis.cpp:254-328): the volume is rounded to FP32 (the reference's
// MRC inputs are FP32, volio.cpp:312-314) and expanded on the device.
inline BallExpansion expand(const Volume& v, const BasisSpec& spec) {
    if (v.n < 8) throw std::invalid_argument("expand: grid too small for the device path");
    bm_context* ctx = spec.plan(v.n);
    const auto f = detail::to_f32(v);
    detail::DeviceBuffer<float> d_in(f.size());
    detail::DeviceBuffer<double> d_out(2 * spec.coeff_count());
    detail::cuda(cudaMemcpy(d_in.get(), f.data(), f.size() * sizeof(float), cudaMemcpyHostToDevice), "expand H2D");
    detail::check(bm_expand(ctx, d_in.get(), 1, nullptr, d_out.get(), nullptr), "expand");
    BallExpansion e(spec, true);
    detail::cuda(cudaMemcpy(e.coeffs().data(), d_out.get(), spec.coeff_count() * sizeof(cdouble),
                            cudaMemcpyDeviceToHost),
                 "expand D2H");
    return e;
}

// synthesize (basis.hpp:99, basis.cpp:332-419): voxel map of a coefficient set,
// zero outside the unit ball; FP64 on the device
inline Volume synthesize(const BallExpansion& e, int n, double voxel_size = 1.0) {
    if (n < 8) throw std::invalid_argument("synthesize: grid size must be >= 8");
    const BasisSpec& spec = e.spec();
    bm_context* ctx = spec.plan(0);
    detail::DeviceBuffer<double> d_c(2 * spec.coeff_count()), d_out(static_cast<size_t>(n) * n * n);
    detail::cuda(cudaMemcpy(d_c.get(), e.coeffs().data(), spec.coeff_count() * sizeof(cdouble), cudaMemcpyHostToDevice),
                 "synthesize H2D");
    detail::check(bm_synthesize(ctx, d_c.get(), e.real_volume() ? 1 : 0, n, d_out.get(), nullptr), "synthesize");
    Volume v(n, voxel_size);
    detail::cuda(cudaMemcpy(v.data.data(), d_out.get(), v.data.size() * sizeof(double), cudaMemcpyDeviceToHost),
                 "synthesize D2H");
    return v;
}

// ------------------------------------------------------------------ wedge (xcorr.hpp:82-125)
struct WedgeMask {
    int n = 0;
    double theta_max_deg = 90.0;  // tilt axis y, beam z (xcorr.hpp:107)
    bool all_pass() const { return theta_max_deg >= 90.0; }
};
inline WedgeMask build_wedge_mask(int n, double theta_max_deg) {
    if (!(theta_max_deg > 0.0 && theta_max_deg <= 90.0))
        throw std::invalid_argument("WedgeMask: theta_max must be in (0, 90]");
    return {n, theta_max_deg};
}

// ------------------------------------------------------------------ optimizer (optimize.hpp:15-94)
struct OptimizerConfig {
    int l_max = 42;
    double lambda_cut = 0.0;  // 0 = default for the grid size
    std::vector<double> band_thresholds{0.5, 0.25, 0.05};
    std::vector<int> fixed_bands{7, 12, 33};
    bool auto_bands = false;  // per-particle bands from the zero-shift kernel (select_bands)
    double seed_grid_step = std::numbers::pi / 8;
    int max_candidates = 20;
    int newton_max_iter = 30;
    double grad_tol = 1e-7;
    double step_damping = 1e-3;
    int shift_radius = 4;
    int shift_step = 2;
    bool prune_after_band = false;  // keep each window's first-band winner for the rest
    int threads = 0;                // host threads: unused (the device does the work)
    // device path only
    int device = -1;          // -1: current device
    double accept_tol = 0.0;  // 0: FP32 default (kFp32AcceptTol, grad_tol floored at kFp32GradTol)

    // optimize.cpp:153-177
    void validate() const {
        if (l_max < 0) throw std::invalid_argument("config: l_max must be >= 0");
        for (size_t i = 1; i < band_thresholds.size(); ++i)
            if (!(band_thresholds[i - 1] >= band_thresholds[i]))
                throw std::invalid_argument("config: band thresholds must be strictly decreasing");
        for (double t : band_thresholds)
            if (!(t > 0.0 && t < 1.0)) throw std::invalid_argument("config: band thresholds must lie in (0,1)");
        if (band_thresholds.size() > 8) throw std::invalid_argument("config: at most 8 band thresholds");
        if (fixed_bands.empty() && !auto_bands)
            throw std::invalid_argument("config: need fixed bands or auto band selection");
        if (fixed_bands.size() > 16) throw std::invalid_argument("config: at most 16 bands");
        for (size_t i = 0; i < fixed_bands.size(); ++i) {
            if (fixed_bands[i] < 0 || fixed_bands[i] > l_max)
                throw std::invalid_argument("config: bands must lie in [0, l_max]");
            if (i > 0 && fixed_bands[i] <= fixed_bands[i - 1])
                throw std::invalid_argument("config: bands must be strictly increasing");
        }
        if (!(seed_grid_step > 0.0 && seed_grid_step <= std::numbers::pi))
            throw std::invalid_argument("config: seed grid step must be in (0, pi]");
        if (max_candidates < 1 || newton_max_iter < 1) throw std::invalid_argument("config: counts must be positive");
        if (!(grad_tol > 0.0) || !(step_damping > 0.0))
            throw std::invalid_argument("config: tolerances must be positive");
        if (shift_radius < 0 || shift_step < 1) throw std::invalid_argument("config: bad shift search parameters");
    }
    bm_align_config to_c() const {
        bm_align_config c{};
        c.n_bands = static_cast<int>(fixed_bands.size());
        for (size_t i = 0; i < fixed_bands.size(); ++i) c.bands[i] = fixed_bands[i];
        c.seed_grid_step = seed_grid_step;
        c.max_candidates = max_candidates;
        c.newton_max_iter = newton_max_iter;
        c.grad_tol = accept_tol > 0.0 ? grad_tol : std::max(grad_tol, kFp32GradTol);
        c.step_damping = step_damping;
        c.shift_radius = shift_radius;
        c.shift_step = shift_step;
        c.accept_tol = accept_tol > 0.0 ? accept_tol : kFp32AcceptTol;
        c.auto_bands = auto_bands ? 1 : 0;
        c.prune_after_band = prune_after_band ? 1 : 0;
        c.n_thresholds = static_cast<int>(band_thresholds.size());
        for (size_t i = 0; i < band_thresholds.size(); ++i) c.thresholds[i] = band_thresholds[i];
        return c;
    }
};

struct AlignmentResult {
    std::array<int, 3> shift{0, 0, 0};
    Rotation rotation;  // template -> re-centred subtomogram
    double score = 0.0;
    bool converged = false;
    long candidates_evaluated = 0;
    long evaluations = 0;  // all bands (the reference splits them per band)
    std::vector<int> bands;
    double template_norm = 0.0;
    double subtomo_norm = 0.0;
    double wall_time_s = 0.0;  // of the whole batch call
    int windows = 0;
    std::map<int, long> evaluations_per_band;  // band -> evaluations (the seed grid counts at the first band)
    double expand_template_s = 0.0;  // phase timings of the batch call (the particles share them)
    double coarse_search_s = 0.0;
    double fine_search_s = 0.0;
};

// Batched alignment against one template (the reference's align() semantics per
// particle; t_hat, the wedge filter and the wedge-power kernel are built once).
// Also accumulates the coefficient-space average of aligned particles.
class Aligner {
public:
    Aligner(const Volume& tmpl, const OptimizerConfig& cfg, const std::optional<WedgeMask>& wedge = std::nullopt)
        : cfg_(cfg), n_(tmpl.n) {
        cfg_.validate();
        if (!(volume_l2_norm(tmpl) > 0.0)) throw std::invalid_argument("align: zero-energy input volume");
        if (wedge && wedge->n != tmpl.n) throw std::invalid_argument("apply_wedge_taper: mask/volume size mismatch");
        device_ = cfg.device < 0 ? detail::current_device() : cfg.device;
        detail::cuda(cudaSetDevice(device_), "cudaSetDevice");
        const double cut = cfg.lambda_cut > 0.0 ? cfg.lambda_cut : default_lambda_cut(tmpl.n, cfg.l_max);
        spec_ = build_spec(cfg.l_max, cut);
        // own context: the template state must not be shared with other aligners
        ctx_ = detail::make_context(device_, n_, cfg.l_max, cut);
        const auto f = detail::to_f32(tmpl);
        detail::DeviceBuffer<float> d(f.size());
        detail::cuda(cudaMemcpy(d.get(), f.data(), f.size() * sizeof(float), cudaMemcpyHostToDevice), "H2D");
        const double theta = (wedge && !wedge->all_pass()) ? wedge->theta_max_deg : 0.0;
        detail::check(bm_set_template(ctx_.get(), d.get(), theta, nullptr), "align");
        detail::cuda(cudaDeviceSynchronize(), "set_template");
        ccfg_ = cfg_.to_c();
    }

    const BasisSpec& spec() const { return spec_; }
    double template_norm() const { return bm_template_norm(ctx_.get()); }
    bm_context* context() const { return ctx_.get(); }

    // device-resident particles (count x n^3 float32), stream-ordered
    std::vector<AlignmentResult> align_batch_device(const float* d_particles, int count, cudaStream_t stream = nullptr) {
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<bm_align_result> raw(static_cast<size_t>(count));
        detail::check(bm_align_batch(ctx_.get(), d_particles, count, &ccfg_, raw.data(), stream), "align");
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::vector<AlignmentResult> out(raw.size());
        for (size_t i = 0; i < raw.size(); ++i) {
            const auto& r = raw[i];
            auto& o = out[i];
            o.shift = {r.shift[0], r.shift[1], r.shift[2]};
            o.rotation = Rotation(r.quat[0], r.quat[1], r.quat[2], r.quat[3]);
            o.score = r.score;
            o.converged = r.converged != 0;
            o.candidates_evaluated = static_cast<long>(r.candidates);
            for (int j = 0; j < r.n_bands && j < 16; ++j) o.evaluations_per_band[r.bands[j]] = static_cast<long>(r.evaluations_per_band[j]);
            o.expand_template_s = r.expand_template_s;
            o.coarse_search_s = r.coarse_search_s;
            o.fine_search_s = r.fine_search_s;
            o.evaluations = static_cast<long>(r.evaluations);
            o.bands.assign(r.bands, r.bands + r.n_bands);
            o.template_norm = template_norm();
            o.subtomo_norm = r.subtomo_norm;
            o.wall_time_s = wall;
            o.windows = r.windows;
        }
        return out;
    }

    // host volumes, uploaded in chunks of `chunk` particles
    std::vector<AlignmentResult> align_batch(const std::vector<Volume>& subtomos, int chunk = 1024) {
        std::vector<AlignmentResult> out;
        out.reserve(subtomos.size());
        const size_t vox = static_cast<size_t>(n_) * n_ * n_;
        detail::DeviceBuffer<float> d(vox * std::min<size_t>(chunk, std::max<size_t>(subtomos.size(), 1)));
        std::vector<float> staging;
        for (size_t p0 = 0; p0 < subtomos.size(); p0 += chunk) {
            const size_t cnt = std::min<size_t>(chunk, subtomos.size() - p0);
            upload(subtomos, p0, cnt, d.get(), staging);
            auto r = align_batch_device(d.get(), static_cast<int>(cnt));
            out.insert(out.end(), r.begin(), r.end());
        }
        return out;
    }

    // average numerator += sum_p rotate_expansion(expand(shift_volume(f_w,p, s_p)), g_p^-1)
    void accumulate_average_device(const float* d_particles, int count, const std::vector<AlignmentResult>& res,
                                   cudaStream_t stream = nullptr) {
        if (res.size() != static_cast<size_t>(count)) throw std::invalid_argument("average: result count mismatch");
        ensure_sum();
        std::vector<bm_align_result> raw(res.size());
        for (size_t i = 0; i < res.size(); ++i) {
            for (int j = 0; j < 3; ++j) raw[i].shift[j] = res[i].shift[j];
            const auto q = res[i].rotation.quat();
            for (int j = 0; j < 4; ++j) raw[i].quat[j] = q[j];
        }
        detail::check(bm_average_accumulate(ctx_.get(), d_particles, count, raw.data(), sum_.get(), stream),
                      "average");
        count_ += count;
    }
    void accumulate_average(const std::vector<Volume>& subtomos, const std::vector<AlignmentResult>& res,
                            int chunk = 1024) {
        if (res.size() != subtomos.size()) throw std::invalid_argument("average: result count mismatch");
        const size_t vox = static_cast<size_t>(n_) * n_ * n_;
        detail::DeviceBuffer<float> d(vox * std::min<size_t>(chunk, std::max<size_t>(subtomos.size(), 1)));
        std::vector<float> staging;
        for (size_t p0 = 0; p0 < subtomos.size(); p0 += chunk) {
            const size_t cnt = std::min<size_t>(chunk, subtomos.size() - p0);
            upload(subtomos, p0, cnt, d.get(), staging);
            std::vector<AlignmentResult> r(res.begin() + p0, res.begin() + p0 + cnt);
            accumulate_average_device(d.get(), static_cast<int>(cnt), r);
        }
    }
    // device FP64 numerator (coeff_count complex, reference layout) and local count
    double* average_numerator_device() {
        ensure_sum();
        return sum_.get();
    }
    long long& average_count() { return count_; }

#ifdef BALLMATCH_B200_WITH_NCCL
    // the one collective of the path: sum the numerators and counts over ranks
    void allreduce_average(ncclComm_t comm, cudaStream_t stream) {
        ensure_sum();
        detail::DeviceBuffer<double> cnt(1);
        const double c = static_cast<double>(count_);
        detail::cuda(cudaMemcpyAsync(cnt.get(), &c, sizeof(double), cudaMemcpyHostToDevice, stream), "H2D");
        if (ncclAllReduce(sum_.get(), sum_.get(), 2 * spec_.coeff_count(), ncclDouble, ncclSum, comm, stream) !=
                ncclSuccess ||
            ncclAllReduce(cnt.get(), cnt.get(), 1, ncclDouble, ncclSum, comm, stream) != ncclSuccess)
            throw std::runtime_error("average: ncclAllReduce failed");
        double total = 0.0;
        detail::cuda(cudaMemcpyAsync(&total, cnt.get(), sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H");
        detail::cuda(cudaStreamSynchronize(stream), "allreduce");
        count_ = static_cast<long long>(std::llround(total));
    }
#endif

    // avg_hat = numerator / count
    BallExpansion average() {
        if (count_ <= 0) throw std::domain_error("average: no particles accumulated");
        ensure_sum();
        BallExpansion e(spec_, true);
        detail::cuda(cudaDeviceSynchronize(), "average");
        detail::cuda(cudaMemcpy(e.coeffs().data(), sum_.get(), spec_.coeff_count() * sizeof(cdouble),
                                cudaMemcpyDeviceToHost),
                     "average D2H");
        for (auto& c : e.coeffs()) c /= static_cast<double>(count_);
        return e;
    }

private:
    void upload(const std::vector<Volume>& v, size_t p0, size_t cnt, float* d, std::vector<float>& staging) const {
        const size_t vox = static_cast<size_t>(n_) * n_ * n_;
        staging.resize(vox * cnt);
        for (size_t i = 0; i < cnt; ++i) {
            const Volume& s = v[p0 + i];
            if (s.n != n_) throw std::invalid_argument("align: template and subtomogram grids differ");
            if (!(volume_l2_norm(s) > 0.0)) throw std::invalid_argument("align: zero-energy input volume");
            for (size_t k = 0; k < vox; ++k) staging[i * vox + k] = static_cast<float>(s.data[k]);
        }
        detail::cuda(cudaMemcpy(d, staging.data(), staging.size() * sizeof(float), cudaMemcpyHostToDevice), "H2D");
    }
    void ensure_sum() {
        if (sum_.get()) return;
        sum_.resize(2 * spec_.coeff_count());
        detail::cuda(cudaMemset(sum_.get(), 0, 2 * spec_.coeff_count() * sizeof(double)), "memset");
    }

    OptimizerConfig cfg_;
    bm_align_config ccfg_{};
    int n_ = 0, device_ = 0;
    BasisSpec spec_;
    detail::ContextPtr ctx_;
    detail::DeviceBuffer<double> sum_;
    long long count_ = 0;
};

#ifdef BALLMATCH_B200_WITH_NCCL
// Multi-GPU alignment + averaging in ONE process: one
// Aligner (context, template state) and one host thread per device, NCCL
// communicators from ncclCommInitAll.  Particles are handed out in chunks from a
// shared atomic counter (dynamic assignment: a device that draws cheap
// particles -- fewer fine windows, shorter Newton runs -- simply takes more
// chunks), each device accumulates the average numerator of its own particles,
// and the only collective is the allreduce of those numerators and counts.
class MultiDeviceAligner {
public:
    MultiDeviceAligner(const Volume& tmpl, const OptimizerConfig& cfg, const std::vector<int>& devices,
                       const std::optional<WedgeMask>& wedge = std::nullopt, int chunk = 256)
        : chunk_(chunk), devices_(devices) {
        if (devices_.empty()) throw std::invalid_argument("multi-device: no devices");
        if (chunk_ < 1) throw std::invalid_argument("multi-device: chunk must be >= 1");
        for (int d : devices_) {
            OptimizerConfig c = cfg;
            c.device = d;
            aligners_.push_back(std::make_unique<Aligner>(tmpl, c, wedge));
        }
        comms_.resize(devices_.size());
        if (ncclCommInitAll(comms_.data(), static_cast<int>(devices_.size()), devices_.data()) != ncclSuccess)
            throw std::runtime_error("multi-device: ncclCommInitAll failed");
    }
    ~MultiDeviceAligner() {
        for (auto c : comms_)
            if (c) ncclCommDestroy(c);
    }
    MultiDeviceAligner(const MultiDeviceAligner&) = delete;
    MultiDeviceAligner& operator=(const MultiDeviceAligner&) = delete;

    int devices() const { return static_cast<int>(devices_.size()); }
    // particles each device aligned in the last call (load-balance evidence)
    const std::vector<long long>& particles_per_device() const { return per_device_; }

    // align every particle (results in input order) and leave the allreduced
    // average numerator on every device
    std::vector<AlignmentResult> align_and_average(const std::vector<Volume>& subtomos) {
        const size_t total = subtomos.size();
        std::vector<AlignmentResult> out(total);
        std::atomic<size_t> next{0};
        per_device_.assign(devices_.size(), 0);
        std::vector<std::exception_ptr> err(devices_.size());
        auto work = [&](size_t i) {
            try {
                detail::cuda(cudaSetDevice(devices_[i]), "cudaSetDevice");
                Aligner& al = *aligners_[i];
                const int n = subtomos.empty() ? 0 : subtomos[0].n;
                const size_t vox = static_cast<size_t>(n) * n * n;
                detail::DeviceBuffer<float> d(vox * static_cast<size_t>(chunk_));
                std::vector<float> staging;
                for (size_t p0; (p0 = next.fetch_add(static_cast<size_t>(chunk_))) < total;) {
                    const size_t cnt = std::min<size_t>(static_cast<size_t>(chunk_), total - p0);
                    staging.resize(vox * cnt);
                    for (size_t k = 0; k < cnt; ++k) {
                        const Volume& v = subtomos[p0 + k];
                        if (v.n != n) throw std::invalid_argument("align: template and subtomogram grids differ");
                        for (size_t x = 0; x < vox; ++x) staging[k * vox + x] = static_cast<float>(v.data[x]);
                    }
                    detail::cuda(cudaMemcpy(d.get(), staging.data(), staging.size() * sizeof(float),
                                            cudaMemcpyHostToDevice), "H2D");
                    auto r = al.align_batch_device(d.get(), static_cast<int>(cnt));
                    al.accumulate_average_device(d.get(), static_cast<int>(cnt), r);
                    for (size_t k = 0; k < cnt; ++k) out[p0 + k] = r[k];
                    per_device_[i] += static_cast<long long>(cnt);
                }
                detail::cuda(cudaDeviceSynchronize(), "align");
            } catch (...) {
                err[i] = std::current_exception();
            }
        };
        run_all(work);
        for (auto& e : err)
            if (e) std::rethrow_exception(e);
        // the one collective: every device's numerator and count summed over devices
        auto reduce = [&](size_t i) {
            try {
                detail::cuda(cudaSetDevice(devices_[i]), "cudaSetDevice");
                aligners_[i]->allreduce_average(comms_[i], nullptr);
            } catch (...) {
                err[i] = std::current_exception();
            }
        };
        run_all(reduce);
        for (auto& e : err)
            if (e) std::rethrow_exception(e);
        return out;
    }

    // avg_hat of every particle aligned so far (device 0's allreduced numerator)
    BallExpansion average() {
        detail::cuda(cudaSetDevice(devices_[0]), "cudaSetDevice");
        return aligners_[0]->average();
    }
    Aligner& aligner(int i) { return *aligners_.at(static_cast<size_t>(i)); }

private:
    template <class F>
    void run_all(F& f) {
        std::vector<std::thread> th;
        for (size_t i = 1; i < devices_.size(); ++i) th.emplace_back(f, i);
        f(0);
        for (auto& t : th) t.join();
    }
    int chunk_;
    std::vector<int> devices_;
    std::vector<std::unique_ptr<Aligner>> aligners_;
    std::vector<ncclComm_t> comms_;
    std::vector<long long> per_device_;
};
#endif

// align (optimize.cpp:423-521): one template, one subtomogram
inline AlignmentResult align(const Volume& tmpl, const Volume& subtomo, const OptimizerConfig& cfg,
                             const std::optional<WedgeMask>& wedge = std::nullopt) {
    cfg.validate();
    if (tmpl.n != subtomo.n) throw std::invalid_argument("align: template and subtomogram grids differ");
    if (!(volume_l2_norm(tmpl) > 0.0) || !(volume_l2_norm(subtomo) > 0.0))
        throw std::invalid_argument("align: zero-energy input volume");
    Aligner a(tmpl, cfg, wedge);
    return a.align_batch({subtomo}).at(0);
}

// align() for many particles against one template
inline std::vector<AlignmentResult> align_batch(const Volume& tmpl, const std::vector<Volume>& subtomos,
                                                const OptimizerConfig& cfg,
                                                const std::optional<WedgeMask>& wedge = std::nullopt) {
    Aligner a(tmpl, cfg, wedge);
    return a.align_batch(subtomos);
}

// coefficient-space average of aligned particles (single device)
inline BallExpansion average(const Volume& tmpl, const std::vector<Volume>& subtomos,
                             const std::vector<AlignmentResult>& results, const OptimizerConfig& cfg,
                             const std::optional<WedgeMask>& wedge = std::nullopt) {
    Aligner a(tmpl, cfg, wedge);
    a.accumulate_average(subtomos, results);
    return a.average();
}

}  // namespace ballmatch_b200
