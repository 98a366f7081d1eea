// extern "C" surface of the CPU oracle, for ctypes in tests/ and bench.py's
// cpu-baseline legs.  TEST INFRASTRUCTURE ONLY.
//
// Complex arrays are interleaved (re, im) doubles.  XiBlocks are packed as the
// concatenation of the (2l+1)^2 row-major blocks, l = 0..L.
#include <cstring>
#include <stdexcept>
#include <string>

#include "bm_oracle.hpp"

using namespace bmo;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}
size_t xi_count(int L) { return (size_t)(L + 1) * (2 * L + 1) * (2 * L + 3) / 3; }
Xi unpack_xi(int L, const double* p) {
    Xi xi(L, {0, 0, 0});
    size_t o = 0;
    for (int l = 0; l <= L; ++l)
        for (auto& v : xi.b[l]) {
            v = cd(p[2 * o], p[2 * o + 1]);
            ++o;
        }
    return xi;
}
void pack_xi(const Xi& xi, double* p) {
    size_t o = 0;
    for (int l = 0; l <= xi.l_max; ++l)
        for (const auto& v : xi.b[l]) {
            p[2 * o] = v.real();
            p[2 * o + 1] = v.imag();
            ++o;
        }
}
Volume make_vol(int n, const double* d) {
    Volume v(n);
    std::memcpy(v.d.data(), d, sizeof(double) * v.d.size());
    return v;
}
Rot rot_of(const double* q) { return Rot{q[0], q[1], q[2], q[3]}; }
void put_rot(const Rot& r, double* q) {
    q[0] = r.w;
    q[1] = r.x;
    q[2] = r.y;
    q[3] = r.z;
}
Expansion exp_of(const Spec* s, const double* c) {
    Expansion e;
    e.spec = s;
    e.real = true;
    e.c.resize(s->coeff_total);
    for (size_t i = 0; i < e.c.size(); ++i) e.c[i] = cd(c[2 * i], c[2 * i + 1]);
    return e;
}
void put_exp(const Expansion& e, double* c) {
    for (size_t i = 0; i < e.c.size(); ++i) {
        c[2 * i] = e.c[i].real();
        c[2 * i + 1] = e.c[i].imag();
    }
}
}  // namespace

extern "C" {

// Mirrors OptimizerConfig (include/ballmatch/optimize.hpp:15-32), fixed bands.
struct bmo_config {
    int l_max;
    double lambda_cut;
    int n_bands;
    int bands[16];
    double seed_grid_step;
    int max_candidates;
    int newton_max_iter;
    double grad_tol;
    double step_damping;
    int shift_radius;
    int shift_step;
    int threads;
    int auto_bands;
    int prune_after_band;
    int n_thresholds;
    double thresholds[8];
};
struct bmo_align_out {
    int shift[3];
    double quat[4];
    double score;
    int converged;
    long long candidates_evaluated;
    long long evaluations;
    double template_norm;
    double subtomo_norm;
    int windows;
    int n_bands;
    int bands[16];
};

static Config cfg_of(const bmo_config* c) {
    Config cfg;
    cfg.l_max = c->l_max;
    cfg.lambda_cut = c->lambda_cut;
    cfg.fixed_bands.assign(c->bands, c->bands + c->n_bands);
    cfg.seed_grid_step = c->seed_grid_step;
    cfg.max_candidates = c->max_candidates;
    cfg.newton_max_iter = c->newton_max_iter;
    cfg.grad_tol = c->grad_tol;
    cfg.step_damping = c->step_damping;
    cfg.shift_radius = c->shift_radius;
    cfg.shift_step = c->shift_step;
    cfg.threads = c->threads;
    cfg.auto_bands = c->auto_bands != 0;
    cfg.prune_after_band = c->prune_after_band != 0;
    if (c->n_thresholds > 0) cfg.band_thresholds.assign(c->thresholds, c->thresholds + c->n_thresholds);
    return cfg;
}

const char* bmo_last_error(void) { return g_err.c_str(); }

void bmo_philox_round10(const unsigned* ctr, const unsigned* key, unsigned* out) {
    auto r = Philox::round10({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
    for (int i = 0; i < 4; ++i) out[i] = r[i];
}
void bmo_philox_u32(unsigned long long seed, unsigned stream, long long n, unsigned* out) {
    PhiloxStream s(seed, stream);
    for (long long i = 0; i < n; ++i) out[i] = s.next_u32();
}
void bmo_philox_gaussian(unsigned long long seed, unsigned stream, long long n, double* out) {
    PhiloxStream s(seed, stream);
    for (long long i = 0; i < n; ++i) out[i] = s.next_gaussian();
}
double bmo_sph_jl(int l, double x) { return sph_jl(l, x); }
double bmo_bessel_root(int l, int k) { return bessel_root(l, k); }
double bmo_default_lambda_cut(int n, int l_max) { return default_lambda_cut(n, l_max); }
void bmo_spherical_harmonic(int l, int m, double theta, double phi, double* out) {
    const cd y = spherical_harmonic(l, m, theta, phi);
    out[0] = y.real();
    out[1] = y.imag();
}
void bmo_gauss_legendre(int n, double* nodes, double* weights) {
    GL g = gauss_legendre(n);
    std::memcpy(nodes, g.nodes.data(), sizeof(double) * n);
    std::memcpy(weights, g.weights.data(), sizeof(double) * n);
}
void bmo_legendre_table(int l_max, double u, double* out) { legendre_table(l_max, u, out); }

void* bmo_spec_create(int l_max, double lambda_cut) {
    try {
        return new Spec(build_spec(l_max, lambda_cut));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void bmo_spec_destroy(void* s) { delete static_cast<Spec*>(s); }
// info: [l_max, coeff_total, pair_total, n_r, n_theta, n_phi]
void bmo_spec_info(void* h, long long* info) {
    const Spec* s = static_cast<Spec*>(h);
    info[0] = s->l_max;
    info[1] = (long long)s->coeff_total;
    info[2] = (long long)s->pair_total;
    info[3] = s->n_r;
    info[4] = s->n_theta;
    info[5] = s->n_phi;
}
int bmo_spec_radial_count(void* h, int l) { return static_cast<Spec*>(h)->radial_count(l); }
double bmo_spec_root(void* h, int l, int k) { return static_cast<Spec*>(h)->roots[l][k - 1]; }
double bmo_spec_norm(void* h, int l, int k) { return static_cast<Spec*>(h)->norms[l][k - 1]; }
// plan tables: r[n_r], cos_theta[n_theta], ptab[tri*n_theta], radial[pairs*n_r]
void bmo_spec_plan(void* h, double* r, double* cos_theta, double* ptab, double* radial) {
    const Spec* s = static_cast<Spec*>(h);
    std::memcpy(r, s->r.data(), sizeof(double) * s->r.size());
    std::memcpy(cos_theta, s->cos_theta.data(), sizeof(double) * s->cos_theta.size());
    std::memcpy(ptab, s->ptab.data(), sizeof(double) * s->ptab.size());
    std::memcpy(radial, s->radial.data(), sizeof(double) * s->radial.size());
}

int bmo_expand(void* h, int n, const double* vol, double* out) {
    try {
        const Spec* s = static_cast<Spec*>(h);
        put_exp(expand(make_vol(n, vol), *s), out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}
// expand many volumes (OpenMP over volumes): the cfg-3 CPU baseline
int bmo_expand_many(void* h, int n, int count, const double* vols, double* out, int threads) {
    const Spec* s = static_cast<Spec*>(h);
    const size_t nv = (size_t)n * n * n;
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : 1)
    for (int i = 0; i < count; ++i)
        put_exp(expand(make_vol(n, vols + nv * i), *s), out + 2 * s->coeff_total * i);
    return 0;
}
int bmo_synthesize(void* h, const double* coeffs, int n, double* out) {
    try {
        const Spec* s = static_cast<Spec*>(h);
        Volume v = synthesize(exp_of(s, coeffs), n);
        std::memcpy(out, v.d.data(), sizeof(double) * v.d.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}
void bmo_rotate_expansion(void* h, const double* coeffs, const double* quat, double* out) {
    const Spec* s = static_cast<Spec*>(h);
    put_exp(rotate_expansion(exp_of(s, coeffs), rot_of(quat)), out);
}
void bmo_little_d(int l_max, double beta, int order, double* out) {
    LittleD st = little_d_stack(l_max, beta, order);
    size_t o = 0;
    for (int d = 0; d <= order; ++d) {
        const auto& t = d == 0 ? st.value : (d == 1 ? st.d1 : st.d2);
        for (int l = 0; l <= l_max; ++l)
            for (double v : t[l]) out[o++] = v;
    }
}
void bmo_wigner_D(int l_max, const double* quat, double* out) {
    auto D = wigner_D(l_max, rot_of(quat));
    size_t o = 0;
    for (int l = 0; l <= l_max; ++l)
        for (const auto& v : D[l]) {
            out[2 * o] = v.real();
            out[2 * o + 1] = v.imag();
            ++o;
        }
}
int bmo_xi(void* h, const double* t, const double* f, double* out) {
    const Spec* s = static_cast<Spec*>(h);
    pack_xi(xi_coefficients(exp_of(s, t), exp_of(s, f)), out);
    return 0;
}
// out: value, imag, grad[3], hess[9]
int bmo_corr_deriv(int L, const double* xi, const double* euler, int l_cut, int order, double* out) {
    try {
        const Xi x = unpack_xi(L, xi);
        const Deriv d = correlation_derivatives(x, {euler[0], euler[1], euler[2]}, l_cut, order);
        out[0] = d.value;
        out[1] = d.imag;
        for (int i = 0; i < 3; ++i) out[2 + i] = d.grad[i];
        for (int i = 0; i < 9; ++i) out[5 + i] = d.hess[i];
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}
// many (pair, rotation) evaluations: cfg-4 CPU baseline (OpenMP over pairs)
int bmo_corr_deriv_many(int L, int n_xi, const double* xis, int n_rot, const double* eulers, int l_cut,
                        int order, double* out, int threads) {
    std::vector<Xi> xs;
    for (int p = 0; p < n_xi; ++p) xs.push_back(unpack_xi(L, xis + 2 * xi_count(L) * p));
#pragma omp parallel for collapse(2) schedule(static) num_threads(threads > 0 ? threads : 1)
    for (int p = 0; p < n_xi; ++p)
        for (int g = 0; g < n_rot; ++g) {
            const double* e = eulers + 3 * g;
            const Deriv d = correlation_derivatives(xs[p], {e[0], e[1], e[2]}, l_cut, order);
            double* o = out + 4 * ((size_t)p * n_rot + g);
            o[0] = d.value;
            o[1] = d.grad[0];
            o[2] = d.grad[1];
            o[3] = d.grad[2];
        }
    return 0;
}
void bmo_xi_compose_right(int L, const double* xi, const double* quat, int l_limit, double* out) {
    pack_xi(xi_compose_right(unpack_xi(L, xi), rot_of(quat), l_limit), out);
}
int bmo_exhaustive_baseline(int L, const double* xi, int l_cut, double step, double* quat, double* score,
                            long long* evals) {
    try {
        const Baseline b = exhaustive_baseline(unpack_xi(L, xi), l_cut, step);
        quat[0] = b.rotation.w, quat[1] = b.rotation.x, quat[2] = b.rotation.y, quat[3] = b.rotation.z;
        *score = b.score;
        *evals = b.evaluations;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
long long bmo_baseline_evaluation_count(double step) { return baseline_evaluation_count(step); }
void bmo_grid_scores(int L, const double* xi, int l_cut, double step, double* out) {
    auto s = grid_scores(unpack_xi(L, xi), l_cut, step);
    std::memcpy(out, s.data(), sizeof(double) * s.size());
}
// returns count; out_quat[4*max], out_score[max], out_index[max]
int bmo_seed_candidates(int L, const double* xi, int l_low, double step, int max_c, int L_wp,
                        const double* wp, double* out_quat, double* out_score, long long* out_index) {
    try {
        const Xi x = unpack_xi(L, xi);
        Xi w;
        if (wp) w = unpack_xi(L_wp, wp);
        auto c = seed_candidates(x, l_low, step, max_c, wp ? &w : nullptr);
        for (size_t i = 0; i < c.size(); ++i) {
            put_rot(c[i].rotation, out_quat + 4 * i);
            out_score[i] = c[i].score;
            out_index[i] = c[i].flat_index;
        }
        return (int)c.size();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}
// out_trace: rows of [band, iter, alpha, beta, gamma, score, gnorm] (max_trace rows)
// energy_ratio / select_bands (xcorr.cpp:129-137, optimize.cpp:179-195)
int bmo_energy_ratio(int L, const double* xi, int l_cut, double* out) {
    try {
        *out = energy_ratio(unpack_xi(L, xi), l_cut);
        return 0;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
int bmo_select_bands(int L, const double* xi, const double* thresholds, int n_thr, int* out_bands) {
    try {
        const auto b = select_bands(unpack_xi(L, xi), std::vector<double>(thresholds, thresholds + n_thr));
        for (size_t i = 0; i < b.size(); ++i) out_bands[i] = b[i];
        return (int)b.size();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int bmo_refine(int L, const double* xi, const double* start, const bmo_config* c, int L_wp,
               const double* wp, double* out_quat, double* out_score, int* out_converged,
               double* out_trace, int max_trace, int* n_trace, long long* n_evals) {
    try {
        const Xi x = unpack_xi(L, xi);
        Xi w;
        if (wp) w = unpack_xi(L_wp, wp);
        const Config cfg = cfg_of(c);
        RefineResult r = refine(x, rot_of(start), cfg.fixed_bands, cfg, wp ? &w : nullptr);
        put_rot(r.rotation, out_quat);
        *out_score = r.score;
        *out_converged = r.converged ? 1 : 0;
        int nt = 0;
        for (const auto& row : r.trace) {
            if (nt >= max_trace) break;
            double* o = out_trace + 7 * nt;
            o[0] = row.band;
            o[1] = row.iteration;
            o[2] = row.alpha;
            o[3] = row.beta;
            o[4] = row.gamma;
            o[5] = row.score;
            o[6] = row.grad_norm;
            ++nt;
        }
        *n_trace = nt;
        long long ev = 0;
        for (const auto& [b, n] : r.evals) ev += n;
        *n_evals = ev;
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}
int bmo_align(int n, const double* tmpl, const double* sub, const bmo_config* c, double wedge_deg,
              bmo_align_out* out) {
    try {
        const Config cfg = cfg_of(c);
        std::optional<WedgeMask> wedge;
        if (wedge_deg > 0.0) wedge = WedgeMask(n, wedge_deg);
        AlignResult r = align(make_vol(n, tmpl), make_vol(n, sub), cfg, wedge);
        for (int i = 0; i < 3; ++i) out->shift[i] = r.shift[i];
        put_rot(r.rotation, out->quat);
        out->score = r.score;
        out->converged = r.converged;
        out->candidates_evaluated = r.candidates_evaluated;
        long long ev = 0;
        for (const auto& [b, k] : r.evals) ev += k;
        out->evaluations = ev;
        out->template_norm = r.template_norm;
        out->subtomo_norm = r.subtomo_norm;
        out->windows = r.windows;
        out->n_bands = (int)std::min<size_t>(r.bands.size(), 16);
        for (int b = 0; b < out->n_bands; ++b) out->bands[b] = r.bands[b];
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}
// one window end-to-end (search_one_shift) with an already-expanded template
int bmo_search_window(void* h, int n, const double* tmpl, const double* sub, const int* shift,
                      const bmo_config* c, double wedge_deg, double* out_quat, double* out_norm_score,
                      double* out_raw_score, double* out_sub_norm, int* out_converged) {
    try {
        const Spec* s = static_cast<Spec*>(h);
        const Config cfg = cfg_of(c);
        const Volume tv = make_vol(n, tmpl);
        Volume f = make_vol(n, sub);
        std::optional<Xi> wp;
        if (wedge_deg > 0.0 && wedge_deg < 90.0) {
            const WedgeMask m(n, wedge_deg);
            f = apply_wedge_taper(f, m);
            wp = wedge_power_kernel(tv, m, cfg.l_max);
        }
        const Expansion t_hat = expand(tv, *s);
        ShiftOutcome oc = search_one_shift(f, {shift[0], shift[1], shift[2]}, t_hat, t_hat.norm(),
                                           cfg.fixed_bands, cfg, wp ? &*wp : nullptr);
        put_rot(oc.refined.rotation, out_quat);
        *out_norm_score = oc.norm_score;
        *out_raw_score = oc.raw_score;
        *out_sub_norm = oc.subtomo_norm;
        *out_converged = oc.refined.converged;
        return oc.valid ? 0 : 3;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}
int bmo_apply_wedge(int n, const double* v, double theta, double* out) {
    try {
        Volume r = apply_wedge(make_vol(n, v), WedgeMask(n, theta));
        std::memcpy(out, r.d.data(), sizeof(double) * r.d.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}
int bmo_apply_wedge_taper(int n, const double* v, double theta, double taper, double* out) {
    try {
        Volume r = apply_wedge_taper(make_vol(n, v), WedgeMask(n, theta), taper);
        std::memcpy(out, r.d.data(), sizeof(double) * r.d.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}
double bmo_wedge_kept_fraction(int n, double theta) { return WedgeMask(n, theta).kept_fraction(); }
double bmo_wedge_keep_profile(int n, double theta, const double* nu, double taper) {
    return wedge_keep_profile(WedgeMask(n, theta), {nu[0], nu[1], nu[2]}, taper);
}
int bmo_wedge_power_kernel(int n, const double* tmpl, double theta, int l_max, double* out) {
    try {
        pack_xi(wedge_power_kernel(make_vol(n, tmpl), WedgeMask(n, theta), l_max), out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}
// rank-1 factors: chi_hat, q_hat (tri_count complex each), total
int bmo_wedge_power_factors(int n, const double* tmpl, double theta, int l_max, double* chi, double* q,
                            double* total) {
    try {
        auto f = wedge_power_factors(make_vol(n, tmpl), WedgeMask(n, theta), l_max);
        for (size_t i = 0; i < f.chi_hat.size(); ++i) {
            chi[2 * i] = f.chi_hat[i].real();
            chi[2 * i + 1] = f.chi_hat[i].imag();
            q[2 * i] = f.q_hat[i].real();
            q[2 * i + 1] = f.q_hat[i].imag();
        }
        *total = f.total;
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}
void bmo_fft_r2c_3d(int n, const double* in, double* out) {
    fft_r2c_3d(n, in, reinterpret_cast<cd*>(out));
}
double bmo_sample_trilinear(int n, const double* v, double x, double y, double z) {
    return sample_trilinear(make_vol(n, v), x, y, z);
}
void bmo_shift_volume(int n, const double* v, const int* s, double* out) {
    Volume r = shift_volume(make_vol(n, v), {s[0], s[1], s[2]});
    std::memcpy(out, r.d.data(), sizeof(double) * r.d.size());
}
void bmo_rotate_volume_trilinear(int n, const double* v, const double* quat, double* out) {
    Volume r = rotate_volume_trilinear(make_vol(n, v), rot_of(quat));
    std::memcpy(out, r.d.data(), sizeof(double) * r.d.size());
}
void bmo_euler_zyz(const double* quat, double* out) {
    const Euler e = rot_of(quat).euler_zyz();
    out[0] = e.alpha;
    out[1] = e.beta;
    out[2] = e.gamma;
}
void bmo_from_euler_zyz(const double* e, double* quat) { put_rot(Rot::from_euler_zyz(e[0], e[1], e[2]), quat); }
double bmo_geodesic_degrees(const double* q1, const double* q2) { return geodesic_degrees(rot_of(q1), rot_of(q2)); }
void bmo_haar_rotation(unsigned long long seed, unsigned stream, double* quat) {
    PhiloxStream s(seed, stream);
    put_rot(haar_rotation(s), quat);
}
// make_phantom with the reference's anisotropic-blob model (tests that mirror
// the reference's own fixtures).  wedge <= 0 / snr <= 0: off.  shift/quat may be NULL (drawn).
int bmo_make_phantom(int n, int blobs, unsigned long long seed, double snr, double wedge,
                     const double* quat, const int* shift, double* tmpl, double* sub, double* out_quat,
                     int* out_shift) {
    try {
        PhantomSpec ps;
        ps.n = n;
        ps.blobs = blobs;
        ps.seed = seed;
        if (snr > 0) ps.snr = snr;
        if (wedge > 0) ps.wedge_theta_deg = wedge;
        if (quat) ps.rotation = rot_of(quat);
        if (shift) ps.shift = std::array<int, 3>{shift[0], shift[1], shift[2]};
        Phantom ph = make_phantom(ps);
        std::memcpy(tmpl, ph.tmpl.d.data(), sizeof(double) * ph.tmpl.d.size());
        std::memcpy(sub, ph.sub.d.data(), sizeof(double) * ph.sub.d.size());
        put_rot(ph.rotation, out_quat);
        for (int i = 0; i < 3; ++i) out_shift[i] = ph.shift[i];
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}
void bmo_gaussian_blob_template(int n, int blobs, unsigned long long seed, double* out) {
    Volume v = gaussian_blob_template(n, blobs, seed);
    std::memcpy(out, v.d.data(), sizeof(double) * v.d.size());
}
int bmo_make_particle(int n, const double* tmpl, unsigned long long seed, int shift_max, double snr,
                      double wedge, double* sub, double* out_quat, int* out_shift) {
    try {
        Phantom ph = make_particle(make_vol(n, tmpl), seed, shift_max, snr > 0 ? std::optional<double>(snr) : std::nullopt,
                                   wedge > 0 ? std::optional<double>(wedge) : std::nullopt);
        std::memcpy(sub, ph.sub.d.data(), sizeof(double) * ph.sub.d.size());
        put_rot(ph.rotation, out_quat);
        for (int i = 0; i < 3; ++i) out_shift[i] = ph.shift[i];
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

}  // extern "C"
