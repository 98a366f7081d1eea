// Host alignment driver of the B200 path (kernel K7 orchestration + the
// coarse-to-fine shift search of align(), src/optimize.cpp:423-521).
//
// Per stage (coarse shift grid, then the unit-step fine cube): all windows of
// all particles in the batch are expanded by the tcgen05 GEMM, seeded on the
// Euler grid, refined band by band (the host raises L between launches =
// frequency marching), and reduced to one outcome per window on the device.
// The host only picks the best window per particle (outcome_better) and builds
// the fine window list.
#include <algorithm>
#include <array>
#include <cfloat>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <thread>
#include <chrono>

#include <nvtx3/nvToolsExt.h>

#include "context.hpp"
#include "refine.cuh"
#include "rotation.cuh"
#include "seed.cuh"
#include "tables.hpp"
#include "wedge.hpp"

namespace bmb {

namespace {
void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

void AlignConfig::validate(int l_max) const {
    for (size_t i = 1; i < band_thresholds.size(); ++i)
        if (!(band_thresholds[i - 1] >= band_thresholds[i]))
            throw std::invalid_argument("config: band thresholds must be strictly decreasing");
    for (double t : band_thresholds)
        if (!(t > 0.0 && t < 1.0)) throw std::invalid_argument("config: band thresholds must lie in (0,1)");
    if (bands.empty() && !auto_bands) throw std::invalid_argument("config: need fixed bands or auto band selection");
    for (size_t i = 0; i < bands.size(); ++i) {
        if (bands[i] < 0 || bands[i] > l_max) throw std::invalid_argument("config: bands must lie in [0, l_max]");
        if (i > 0 && bands[i] <= bands[i - 1]) throw std::invalid_argument("config: bands must be strictly increasing");
    }
    if (!(seed_grid_step > 0.0) || seed_grid_step > kPiH)
        throw std::invalid_argument("config: seed grid step must be in (0, pi]");
    if (max_candidates < 1 || newton_max_iter < 1) throw std::invalid_argument("config: counts must be positive");
    if (max_candidates > 256) throw std::invalid_argument("config: max_candidates above 256 is not supported on the device path");
    if (!(grad_tol > 0.0) || !(step_damping > 0.0)) throw std::invalid_argument("config: tolerances must be positive");
    if (!std::isfinite(accept_tol) || accept_tol < 0.0)
        throw std::invalid_argument("config: accept_tol must be finite and non-negative");
    if (shift_radius < 0 || shift_step < 1) throw std::invalid_argument("config: bad shift search parameters");
}

BandTables BandDev::view() const {
    BandTables t;
    t.L = L;
    t.n_items = n_items;
    t.n_groups = n_groups;
    t.rows = rows;
    t.row_off = row_off.as<int>();
    t.item_mm = item_mm.as<char2>();
    t.item_pm = item_pm.as<char2>();
    t.item_w = item_w.as<float2>();
    t.item_len = item_len.as<int>();
    t.bfac = bfac.as<float>();
    t.bexp = bexp.as<int>();
    t.PQR = PQR.as<float4>();
    t.item_of = item_of.as<int>();
    t.out_pos = out_pos.as<int>();
    t.at_desc = at_desc.as<int2>();
    t.wedge = has_wedge ? wedge.as<float4>() : nullptr;
    t.wedge_side = has_wedge ? wedge_side.as<float4>() : nullptr;
    return t;
}

BandDev& Context::band(int L) {
    auto it = bands_.find(L);
    if (it != bands_.end()) {
        BandDev& b = *it->second;
        if (wedge_active() && !b.has_wedge) {
            BandTablesHost h = build_band_tables(L);
            upload(b.wedge, wedge_band_entries(h, chi_hat, q_hat, wp_total), stream);
            upload(b.wedge_side, wedge_band_entries(h, chi_hat, q_side, wp_total), stream);
            b.has_wedge = true;
            ck(cudaStreamSynchronize(stream), "band wedge tables");
        }
        return b;
    }
    auto b = std::make_unique<BandDev>();
    BandTablesHost h = build_band_tables(L);
    b->L = L;
    b->n_items = h.n_items;
    b->n_groups = h.n_groups;
    b->rows = h.rows;
    upload(b->row_off, h.row_off, stream);
    upload(b->item_mm, h.item_mm, stream);
    upload(b->item_pm, h.item_pm, stream);
    upload(b->item_w, h.item_w, stream);
    upload(b->item_len, h.item_len, stream);
    upload(b->bfac, h.bfac, stream);
    upload(b->bexp, h.bexp, stream);
    std::vector<float4> pqr(h.P.size());
    for (size_t i = 0; i < pqr.size(); ++i) pqr[i] = make_float4(h.P[i], h.Q[i], h.R[i], 0.0f);
    upload(b->PQR, pqr, stream);
    upload(b->item_of, h.item_of, stream);
    upload(b->out_pos, h.out_pos, stream);
    upload(b->at_desc, h.at_desc, stream);
    std::vector<int> rg(h.rows);
    for (int g = 0; g < h.n_groups; ++g)
        for (int r = h.row_off[g]; r < h.row_off[g + 1]; ++r) rg[r] = g;
    upload(b->row_group, rg, stream);
    if (wedge_active()) {
        upload(b->wedge, wedge_band_entries(h, chi_hat, q_hat, wp_total), stream);
        upload(b->wedge_side, wedge_band_entries(h, chi_hat, q_side, wp_total), stream);
        b->has_wedge = true;
    }
    ck(cudaStreamSynchronize(stream), "band tables");
    return *bands_.emplace(L, std::move(b)).first->second;
}

SeedDev& Context::seed_tables(int L, double step) {
    const long long key_step = (long long)std::llround(step * 1e12);
    auto key = std::make_pair(L, key_step);
    auto it = seeds_.find(key);
    if (it != seeds_.end() && it->second->has_wedge == wedge_active()) return *it->second;
    auto s = std::make_unique<SeedDev>();
    s->L_low = L;
    s->step = step;
    // EulerGrid::with_step (optimize.cpp:30-36)
    s->na = s->ng = (int)std::ceil(2.0 * kPiH / step);
    s->nb = (int)std::ceil(kPiH / step) + 1;
    s->nxi = (L + 1) * (2 * L + 1) * (2 * L + 3) / 3;
    const int wd = 2 * L + 1;
    std::vector<double> dgrid;
    std::vector<std::vector<double>> dj(s->nb);
    for (int j = 0; j < s->nb; ++j) {
        const double beta = s->nb > 1 ? kPiH * j / (s->nb - 1) : 0.0;
        dj[j] = little_d_full(L, beta);
        dgrid.insert(dgrid.end(), dj[j].begin(), dj[j].end());
    }
    std::vector<double2> ua((size_t)s->na * wd), ug((size_t)s->ng * wd);
    for (int i = 0; i < s->na; ++i)
        for (int m = -L; m <= L; ++m) {
            const std::complex<double> z = std::polar(1.0, -m * (2.0 * kPiH * i / s->na));
            ua[(size_t)i * wd + (m + L)] = double2{z.real(), z.imag()};
        }
    for (int k = 0; k < s->ng; ++k)
        for (int m = -L; m <= L; ++m) {
            const std::complex<double> z = std::polar(1.0, -m * (2.0 * kPiH * k / s->ng));
            ug[(size_t)k * wd + (m + L)] = double2{z.real(), z.imag()};
        }
    upload(s->dgrid, dgrid, stream);
    upload(s->ua, ua, stream);
    upload(s->ug, ug, stream);
    if (wedge_active()) {
        // rho on the grid from the wedge-power kernel at min(L, l_max) (optimize.cpp:202-206)
        const int Lw = std::min(L, basis.l_max);
        auto coef = [](const std::vector<std::complex<double>>& hat, int l, int m) {
            if (m >= 0) return hat[host::tri(l, m)];
            const std::complex<double> c = std::conj(hat[host::tri(l, -m)]);
            return ((-m) % 2) ? -c : c;
        };
        const int w2 = 2 * Lw + 1;
        std::vector<double> sq((size_t)s->na * s->nb * s->ng);
        for (int j = 0; j < s->nb; ++j) {
            const std::vector<double>& d = dj[j];
            std::vector<std::complex<double>> A((size_t)w2 * w2, {0.0, 0.0});
            for (int l = 0; l <= Lw; ++l) {
                const int wl = 2 * l + 1;
                const size_t off = (size_t)l * (2 * l - 1) * (2 * l + 1) / 3;
                for (int m = -l; m <= l; ++m)
                    for (int mp = -l; mp <= l; ++mp)
                        A[(size_t)(m + Lw) * w2 + (mp + Lw)] +=
                            std::conj(coef(chi_hat, l, m)) * coef(q_hat, l, mp) / wp_total *
                            d[off + (size_t)(m + l) * wl + (mp + l)];
            }
            for (int k = 0; k < s->ng; ++k)
                for (int i = 0; i < s->na; ++i) {
                    double acc = 0.0;
                    for (int m = 0; m < w2; ++m) {
                        std::complex<double> b{0.0, 0.0};
                        for (int mp = 0; mp < w2; ++mp)
                            b += A[(size_t)m * w2 + mp] * std::polar(1.0, -(mp - Lw) * (2.0 * kPiH * k / s->ng));
                        const std::complex<double> pa = std::polar(1.0, -(m - Lw) * (2.0 * kPiH * i / s->na));
                        acc += pa.real() * b.real() - pa.imag() * b.imag();
                    }
                    sq[((size_t)j * s->na + i) * s->ng + k] = std::sqrt(std::clamp(1.0 - acc, 0.02, 2.0));
                }
        }
        upload(s->wedge_sqrt, sq, stream);
        s->has_wedge = true;
    }
    ck(cudaStreamSynchronize(stream), "seed tables");
    auto& ref = seeds_[key];
    ref = std::move(s);
    return *ref;
}

void Context::set_template(const float* tmpl, double wedge_theta) {
    if (geo.support == 0) throw std::invalid_argument("set_template: context has no operator (n = 0)");
    const auto t0 = std::chrono::steady_clock::now();
    struct Stamp {
        double& out;
        std::chrono::steady_clock::time_point t0;
        ~Stamp() { out = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
    } stamp{template_s_, t0};
    // template expansion through the same tensor-core path (align: t_hat = expand(tmpl))
    std::vector<int> wv{0}, ws{0, 0, 0};
    expand_windows(tmpl, (long long)n * n * n, 1, wv, ws);
    t_hat.reserve(sizeof(float) * geo.m_pad);
    ck(cudaMemcpyAsync(t_hat.p, coef.p, sizeof(float) * geo.m_pad, cudaMemcpyDeviceToDevice, stream), "t_hat");
    norms.reserve(sizeof(double));
    launch_window_norms(coef.as<float>(), 1, geo.m_pad, geo, norms.as<double>(), stream);
    ck(cudaMemcpyAsync(&t_norm, norms.p, sizeof(double), cudaMemcpyDeviceToHost, stream), "t_norm");
    ck(cudaStreamSynchronize(stream), "set_template");
    if (!(t_norm > 0.0)) throw std::invalid_argument("align: template has no in-ball energy");
    wedge_deg = wedge_theta;
    wedge.reset();
    chi_hat.clear();
    q_hat.clear();
    wp_total = 0.0;
    if (wedge_theta > 0.0 && wedge_theta < 90.0) {
        wedge = std::make_unique<WedgeFilter>(n, wedge_theta, kWedgeTaperDeg);
        WedgePowerFactors f = wedge_power_factors(tmpl, n, basis.l_max, wedge_theta, kWedgeTaperDeg, stream);
        chi_hat = std::move(f.chi_hat);
        q_hat = std::move(f.q_hat);
        wp_total = f.total;
    }
    build_side_template();
    // band tables carry the wedge entries of this template: rebuild lazily
    bands_.clear();
    seeds_.clear();
    has_template = true;
    // the lanes re-adopt the template on their next use
    tmpl_copy_.reserve(sizeof(float) * (size_t)n * n * n);
    ck(cudaMemcpyAsync(tmpl_copy_.p, tmpl, sizeof(float) * (size_t)n * n * n, cudaMemcpyDeviceToDevice, stream),
       "template copy");
    ck(cudaStreamSynchronize(stream), "template copy");
    lanes_stale_ = true;
}

// Template side of the side kernels (refine.cu chart_transform): t' = D(K^-1) t
// (rotate_expansion) and q' = D(K^-1) q, K = ZYZ(0, pi/2, 0), in FP64 on the host.
void Context::build_side_template() {
    const Euler3 e = q_euler(q_inv(q_from_euler(0.0, kPiH / 2.0, 0.0)));
    const std::vector<std::complex<double>> D = wigner_D_blocks(basis.l_max, e.a, e.b, e.g);
    std::vector<float> t(geo.m_pad, 0.0f);
    ck(cudaMemcpyAsync(t.data(), t_hat.p, sizeof(float) * geo.m_pad, cudaMemcpyDeviceToHost, stream), "t_hat");
    ck(cudaStreamSynchronize(stream), "t_hat");
    upload(t_side, rotate_real_packed(t, basis, D), stream);
    q_side.clear();
    if (!q_hat.empty()) q_side = rotate_tri(q_hat, basis.l_max, D);
    ck(cudaStreamSynchronize(stream), "side template");
}

// Bulk-synchronous damped Newton over every candidate of every window
// (refine(), src/optimize.cpp:255-357), band by band; windows are processed in
// chunks so the window + side kernels of a chunk stay within a memory budget.
void Context::refine_windows(int nw, int maxc, const AlignConfig& cfg, const Quat& koff, long long grid_evals) {
    work_.reserve(sizeof(CandWork) * (size_t)nw * maxc);
    counters_.reserve(sizeof(int) * 8);
    int* d_counts = counters_.as<int>();  // CNT_L2, -, CNT_T0, CNT_T1, -, -, start counts
    int* h_active = pinned_counts();
    const bool wedge = wedge_active();
    const int Lmax_band = cfg.bands.back();
    BandDev& btop = band(Lmax_band);
    const size_t kernel_bytes = sizeof(float4) * (size_t)btop.rows * 32;
    const int per_chunk = (int)std::max<size_t>(1, pool_budget_ / (2 * kernel_bytes));
    for (int w0 = 0; w0 < nw; w0 += per_chunk) {
        const int cnt = std::min(per_chunk, nw - w0);
        for (size_t bi = 0; bi < cfg.bands.size(); ++bi) {
            const int L = cfg.bands[bi];
            BandDev& bd = band(L);
            const size_t len = (size_t)bd.rows * 32;
            // NVTX range per band ("bmb_band16"): profilers select one band's launches
            char range[32];
            snprintf(range, sizeof(range), "bmb_band%d", L);
            nvtxRangePushA(range);
            struct RangePop {
                ~RangePop() { nvtxRangePop(); }
            } pop_range;
            StageArgs a;
            a.T = bd.view();
            a.row_group = bd.row_group.as<int>();
            // window kernels xi(f, t) and side kernels xi(f, D(K^-1) t) of this band
            xi_win_.reserve(sizeof(float4) * len * cnt);
            xi_side_.reserve(sizeof(float4) * len * cnt);
            XiArgs xa;
            xa.T = a.T;
            xa.row_group = a.row_group;
            xa.f = coef.as<float>() + (size_t)w0 * geo.m_pad;
            xa.ldf = geo.m_pad;
            xa.t = t_hat.as<float>();
            xa.ldt = 0;
            xa.block_off = geo.block_off;
            xa.radial_count = geo.radial_count;
            xa.n = cnt;
            xa.out = xi_win_.as<float4>();
            xa.nf = L < basis.l_max ? basis.block_off[L + 1] : geo.coeffs;
            for (int l = 0; l <= L; ++l) xa.npairs += basis.radial_count(l) * (l + 1);
            cudaEvent_t r0 = timer.begin(stream);
            cudaEvent_t rb = timer.begin(stream);
            timer.band = (int)bi;
            cudaEvent_t x0 = timer.begin(stream);
            xa.t2 = t_side.as<float>();
            xa.out2 = xi_side_.as<float4>();
            if (launch_build_xi(xa, stream) != 0) throw std::runtime_error("build_xi launch failed");
            timer.end(K_XI, x0, stream);
            timer.launches += 1;
            a.xi_win = xi_win_.as<float4>();
            a.xi_side = xi_side_.as<float4>();
            a.cand = cand_.as<CandState>() + (size_t)w0 * maxc;
            a.work = work_.as<CandWork>() + (size_t)w0 * maxc;
            a.cand_count = cand_count_.as<int>() + w0;
            a.max_cand = maxc;
            a.n_win = cnt;
            a.prm.band = L;
            a.prm.band_index = (int)bi;
            a.prm.newton_max_iter = cfg.newton_max_iter;
            a.prm.grad_tol = cfg.grad_tol;
            a.prm.accept_tol = cfg.accept_tol;
            a.prm.step_damping = cfg.step_damping;
            a.prm.koffset[0] = koff.w;
            a.prm.koffset[1] = koff.x;
            a.prm.koffset[2] = koff.y;
            a.prm.koffset[3] = koff.z;
            a.prm.max_cand = maxc;
            a.prm.has_wedge = wedge ? 1 : 0;
            const long long slots = (long long)cnt * maxc;
            // lists: fresh[2] (candidates whose iteration needs an order-2 evaluation at g),
            // trial[2] (pending trials), start (band start); counts d_counts[0..1] fresh,
            // [2..3] trial, [4] start
            lists_.reserve(sizeof(int) * 5 * (size_t)slots);
            int* lbase = lists_.as<int>();
            int* fresh[2] = {lbase, lbase + slots};
            int* trial[2] = {lbase + 2 * slots, lbase + 3 * slots};
            int* start = lbase + 4 * slots;
            int* c_fresh[2] = {d_counts, d_counts + 1};
            int* c_trial[2] = {d_counts + 2, d_counts + 3};
            int* c_start = d_counts + 4;
            a.list2 = fresh[0];  // iter_begin / final_prep append to list2 with count CNT_L2 = c_fresh[0]
            a.counts = d_counts;
            a.eval_stats = eval_stats();
            ck(cudaMemsetAsync(d_counts, 0, sizeof(int) * 5, stream), "counts");
            cudaEvent_t b0 = timer.begin(stream);
            launch_band_begin(a, start, c_start, stream);
            launch_iter_begin(a, start, c_start, (int)slots, stream);  // band start: all need an evaluation
            timer.end(K_NEWTON, b0, stream);
            timer.launches += 2;
            // rounds: evaluate and step the fresh candidates, evaluate every pending trial
            // at order 2, then accept / retry / advance each to its next iteration
            int cur = 0;
            const int max_rounds = 4 * cfg.newton_max_iter + 8;
            // The list lengths come back to the host to size the launches and to stop.
            // Candidates only ever leave the lists, so once few are left (the long
            // tail: after ~20 of ~60 rounds under 2% remain) the host reads the counts
            // every round_check_-th round only and sizes the rounds in between by the
            // last sum (an upper bound); the kernels take the true lengths from device
            // memory, and a round on empty lists is a few empty launches.
            int bound = (int)slots, since_check = 0;
            int nf = 0, nt = 0;
            for (int round = 0; round < max_rounds; ++round) {
                const bool check = debug_iters_ || round_check_ <= 1 || bound > kTailCandidates ||
                                   since_check + 1 >= round_check_;
                if (check) {
                    ck(cudaMemcpyAsync(h_active, d_counts, sizeof(int) * 4, cudaMemcpyDeviceToHost, stream), "active");
                    ck(cudaStreamSynchronize(stream), "round");
                    nf = h_active[cur], nt = h_active[2 + cur];
                    if (debug_iters_)
                        fprintf(stderr, "[refine] band %d round %d fresh %d trials %d\n", L, round, nf, nt);
                    if (nf == 0 && nt == 0) break;
                    bound = nf + nt;
                    since_check = 0;
                } else {
                    nf = bound, nt = 0;  // launch bounds only (nt_max below = bound)
                    ++since_check;
                }
                ck(cudaMemsetAsync(c_fresh[cur ^ 1], 0, sizeof(int), stream), "next fresh count");
                ck(cudaMemsetAsync(c_trial[cur ^ 1], 0, sizeof(int), stream), "next trial count");
                if (nf > 0) {
                    cudaEvent_t e2 = timer.begin(stream);
                    launch_eval(a, 2, fresh[cur], c_fresh[cur], nf, stream);
                    timer.end(K_EVAL2, e2, stream);
                    cudaEvent_t n0 = timer.begin(stream);
                    launch_step(a, fresh[cur], c_fresh[cur], trial[cur], c_trial[cur], nf, stream);
                    timer.end(K_NEWTON, n0, stream);
                    timer.launches += 2;
                }
                const int nt_max = nt + nf;
                if (nt_max > 0) {
                    cudaEvent_t e0 = timer.begin(stream);
                    launch_eval(a, 2, trial[cur], c_trial[cur], nt_max, stream, true);
                    timer.end(K_EVAL0, e0, stream);
                    cudaEvent_t n1 = timer.begin(stream);
                    launch_advance(a, trial[cur], c_trial[cur], trial[cur ^ 1], c_trial[cur ^ 1], fresh[cur ^ 1],
                                   c_fresh[cur ^ 1], nt_max, stream);
                    timer.end(K_NEWTON, n1, stream);
                    timer.launches += 2;
                }
                cur ^= 1;
            }
            const bool prune_now = cfg.prune_after_band && cfg.bands.size() > 1 && bi == 0;
            if (bi + 1 == cfg.bands.size() || prune_now) {
                // final unanchored score at the top band (optimize.cpp:349-352), or at
                // the first band before prune_after_band keeps each window's winner
                a.list2 = fresh[0];
                ck(cudaMemsetAsync(d_counts, 0, sizeof(int), stream), "final count");
                launch_final_prep(a, stream);
                cudaEvent_t ef = timer.begin(stream);
                launch_eval(a, 0, a.list2, d_counts + CNT_L2, (int)slots, stream);
                timer.end(K_EVAL0, ef, stream);
                launch_final_score(a, (int)slots, stream);
                timer.launches += 3;
                if (prune_now) {
                    launch_prune(a, stream);
                    ++timer.launches;
                }
            }
            ++timer.refine_launches;
            timer.band = -1;
            timer.end(K_REFINE, r0, stream);
            timer.end(K_REFINE_B0 + (int)std::min<size_t>(bi, 3), rb, stream);
        }
        ReduceArgs ra;
        ra.cand = cand_.as<CandState>() + (size_t)w0 * maxc;
        ra.work = work_.as<CandWork>() + (size_t)w0 * maxc;
        ra.cand_count = cand_count_.as<int>() + w0;
        ra.max_cand = maxc;
        ra.n_win = cnt;
        ra.sub_norm = sub_norm_.as<double>() + w0;
        ra.t_norm = t_norm;
        ra.win_particle = win_vol.as<int>() + w0;
        ra.win_shift = win_shift.as<int>() + 3 * w0;
        ra.grid_evals = grid_evals;
        ra.extra_candidates = (cfg.prune_after_band && cfg.bands.size() > 1) ? 1 : 0;
        ra.out = outcome_.as<WindowOutcome>() + w0;
        launch_window_reduce(ra, stream);
        ++timer.launches;
    }
}

// seed_candidates (optimize.cpp:197-253) for n_f device coefficient sets
// (complex128, reference layout) against the template: candidate rotations
// (quaternions, rank order) and counts to host
void Context::seed_candidates(const double* f, int n_f, int L_low, double step, int max_cand, double* quats,
                              int* counts, double* scores) {
    if (n_f <= 0) return;
    if (!has_template) throw std::invalid_argument("seed: set_template first");
    if (L_low < 0 || L_low > basis.l_max) throw std::invalid_argument("seed: band outside [0, l_max]");
    if (max_cand < 1 || max_cand > 256) throw std::invalid_argument("seed: max_candidates must be 1..256");
    if (!(step > 0.0) || step > kPiH) throw std::invalid_argument("seed: grid step must be in (0, pi]");
    const int ld = geo.m_pad;
    work_f.reserve(sizeof(float) * (size_t)n_f * ld);
    launch_from_complex(f, n_f, geo, work_f.as<float>(), ld, stream);
    SeedDev& sd = seed_tables(L_low, step);
    SeedArgs sa;
    sa.coef = work_f.as<float>();
    sa.ldc = ld;
    sa.t_hat = t_hat.as<float>();
    sa.block_off = geo.block_off;
    sa.radial_count = geo.radial_count;
    sa.L_low = sd.L_low;
    sa.rows_low = sd.L_low + 1 <= basis.l_max ? basis.block_off[sd.L_low + 1] : geo.coeffs;
    sa.nxi = sd.nxi;
    sa.na = sd.na;
    sa.nb = sd.nb;
    sa.ng = sd.ng;
    sa.dgrid = sd.dgrid.as<double>();
    sa.ua = sd.ua.as<double2>();
    sa.ug = sd.ug.as<double2>();
    sa.wedge_sqrt = sd.has_wedge ? sd.wedge_sqrt.as<double>() : nullptr;
    sa.max_cand = max_cand;
    cand_.reserve(sizeof(CandState) * (size_t)n_f * max_cand);
    cand_count_.reserve(sizeof(int) * n_f);
    sub_norm_.reserve(sizeof(double) * (size_t)n_f * max_cand);
    sa.cand = cand_.as<CandState>();
    sa.cand_count = cand_count_.as<int>();
    sa.seed_score = scores ? sub_norm_.as<double>() : nullptr;
    if (seed_needs_scratch(sa)) {
        sa.scratch_windows = 4096;
        seed_scratch_.reserve(sizeof(double2) * (size_t)sa.scratch_windows * sa.nxi);
        sa.xi_scratch = seed_scratch_.as<double2>();
    }
    if (launch_seed(sa, n_f, stream) != 0) throw std::runtime_error("seed kernel launch failed");
    std::vector<CandState> cs((size_t)n_f * max_cand);
    ck(cudaMemcpyAsync(cs.data(), cand_.p, sizeof(CandState) * cs.size(), cudaMemcpyDeviceToHost, stream), "cands");
    ck(cudaMemcpyAsync(counts, cand_count_.p, sizeof(int) * n_f, cudaMemcpyDeviceToHost, stream), "counts");
    if (scores)
        ck(cudaMemcpyAsync(scores, sub_norm_.p, sizeof(double) * (size_t)n_f * max_cand, cudaMemcpyDeviceToHost,
                           stream), "scores");
    ck(cudaStreamSynchronize(stream), "seed");
    for (size_t i = 0; i < cs.size(); ++i)
        for (int k = 0; k < 4; ++k) quats[4 * i + k] = cs[i].g[k];
}

// Objective::eval of the refinement (bm_objective_eval): kernels of one
// coefficient set f against t (null: the template; its side template is rebuilt
// for an explicit t), at band L, n chart points
void Context::objective_eval(const double* f, const double* t, const double* euler, const double* anchors, int n,
                             int L, int order, double* out) {
    if (n <= 0) return;
    if (L < 0 || L > basis.l_max) throw std::invalid_argument("objective: band outside [0, l_max]");
    if (order != 0 && order != 2) throw std::invalid_argument("objective: order must be 0 or 2");
    if (!t && !has_template) throw std::invalid_argument("objective: set_template first (or pass t)");
    const int ld = geo.m_pad;
    work_f.reserve(sizeof(float) * (size_t)3 * ld);
    float* fr = work_f.as<float>();
    const float* tr = t_hat.as<float>();
    const float* ts = t_side.as<float>();
    launch_from_complex(f, 1, geo, fr, ld, stream);
    if (t) {
        float* tt = fr + ld;
        cudaMemsetAsync(tt, 0, sizeof(float) * 2 * ld, stream);
        launch_from_complex(t, 1, geo, tt, ld, stream);
        std::vector<float> th(ld);
        ck(cudaMemcpyAsync(th.data(), tt, sizeof(float) * ld, cudaMemcpyDeviceToHost, stream), "t");
        ck(cudaStreamSynchronize(stream), "t");
        const Euler3 e = q_euler(q_inv(q_from_euler(0.0, kPiH / 2.0, 0.0)));
        const std::vector<float> side = rotate_real_packed(th, basis, wigner_D_blocks(basis.l_max, e.a, e.b, e.g));
        ck(cudaMemcpyAsync(tt + ld, side.data(), sizeof(float) * ld, cudaMemcpyHostToDevice, stream), "t side");
        tr = tt;
        ts = tt + ld;
    }
    BandDev& bd = band(L);
    const size_t len = (size_t)bd.rows * 32;
    xi_win_.reserve(sizeof(float4) * len);
    xi_side_.reserve(sizeof(float4) * len);
    XiArgs xa;
    xa.T = bd.view();
    xa.row_group = bd.row_group.as<int>();
    xa.f = fr;
    xa.ldf = ld;
    xa.t = tr;
    xa.ldt = 0;
    xa.block_off = geo.block_off;
    xa.radial_count = geo.radial_count;
    xa.n = 1;
    xa.out = xi_win_.as<float4>();
    xa.nf = L < basis.l_max ? basis.block_off[L + 1] : geo.coeffs;
    if (launch_build_xi(xa, stream) != 0) throw std::runtime_error("build_xi launch failed");
    xa.t = ts;
    xa.out = xi_side_.as<float4>();
    if (launch_build_xi(xa, stream) != 0) throw std::runtime_error("build_xi launch failed");
    StageArgs a;
    a.T = bd.view();
    a.row_group = xa.row_group;
    a.xi_win = xi_win_.as<float4>();
    a.xi_side = xi_side_.as<float4>();
    cand_.reserve(sizeof(CandState) * (size_t)n);
    work_.reserve(sizeof(CandWork) * (size_t)n);
    lists_.reserve(sizeof(int) * (size_t)n);
    counters_.reserve(sizeof(int) * 8);
    a.cand = cand_.as<CandState>();
    a.work = work_.as<CandWork>();
    a.list2 = lists_.as<int>();
    a.counts = counters_.as<int>();
    a.max_cand = n;
    a.n_win = 1;
    const Quat koff = q_from_euler(0.0, kPiH / 2.0, 0.0);
    a.prm.band = L;
    a.prm.band_index = 0;
    a.prm.koffset[0] = koff.w;
    a.prm.koffset[1] = koff.x;
    a.prm.koffset[2] = koff.y;
    a.prm.koffset[3] = koff.z;
    a.prm.max_cand = n;
    a.prm.has_wedge = wedge_active() ? 1 : 0;
    if (launch_objective_eval(a, euler, anchors, n, order, out, stream) != 0)
        throw std::runtime_error("objective launch failed");
    ck(cudaStreamSynchronize(stream), "objective");
}

std::vector<WindowOutcome> Context::run_windows(const float* vols, int n_vol, const std::vector<int>& wvol,
                                                const std::vector<int>& wshift, const AlignConfig& cfg) {
    if (!has_template) throw std::invalid_argument("align: set_template first");
    cfg.validate(basis.l_max);
    const int nw = (int)wvol.size();
    std::vector<WindowOutcome> res(nw);
    if (nw == 0) return res;
    const long long vstride = (long long)n * n * n;
    expand_windows(vols, vstride, n_vol, wvol, wshift);
    sub_norm_.reserve(sizeof(double) * nw);
    cudaEvent_t t0 = timer.begin(stream);
    launch_window_norms(coef.as<float>(), nw, geo.m_pad, geo, sub_norm_.as<double>(), stream);
    ++timer.launches;
    timer.end(K_MISC, t0, stream);

    const int maxc = cfg.max_candidates;
    cand_.reserve(sizeof(CandState) * (size_t)nw * maxc);
    cand_count_.reserve(sizeof(int) * nw);
    outcome_.reserve(sizeof(WindowOutcome) * nw);
    win_counter_.reserve(sizeof(int));
    SeedDev& sd = seed_tables(cfg.bands.front(), cfg.seed_grid_step);
    SeedArgs sa;
    sa.coef = coef.as<float>();
    sa.ldc = geo.m_pad;
    sa.t_hat = t_hat.as<float>();
    sa.block_off = geo.block_off;
    sa.radial_count = geo.radial_count;
    sa.L_low = sd.L_low;
    sa.rows_low = sd.L_low + 1 <= basis.l_max ? basis.block_off[sd.L_low + 1] : geo.coeffs;
    sa.nxi = sd.nxi;
    sa.na = sd.na;
    sa.nb = sd.nb;
    sa.ng = sd.ng;
    sa.dgrid = sd.dgrid.as<double>();
    sa.ua = sd.ua.as<double2>();
    sa.ug = sd.ug.as<double2>();
    sa.wedge_sqrt = sd.has_wedge ? sd.wedge_sqrt.as<double>() : nullptr;
    sa.max_cand = maxc;
    sa.cand = cand_.as<CandState>();
    sa.cand_count = cand_count_.as<int>();
    if (seed_needs_scratch(sa)) {
        sa.scratch_windows = 4096;
        seed_scratch_.reserve(sizeof(double2) * (size_t)sa.scratch_windows * sa.nxi);
        sa.xi_scratch = seed_scratch_.as<double2>();
    }
    cudaEvent_t s0 = timer.begin(stream);
    if (launch_seed(sa, nw, stream) != 0) throw std::runtime_error("seed kernel launch failed");
    ++timer.launches;
    timer.end(K_SEED, s0, stream);

    const Quat koff = q_from_euler(0.0, kPiH / 2.0, 0.0);
    const long long grid_evals = (long long)sd.na * sd.nb * sd.ng;
    refine_windows(nw, maxc, cfg, koff, grid_evals);
    ck(cudaMemcpyAsync(res.data(), outcome_.p, sizeof(WindowOutcome) * nw, cudaMemcpyDeviceToHost, stream),
       "outcomes");
    ck(cudaStreamSynchronize(stream), "run_windows");
    timer.collect();
    return res;
}

namespace {
// outcome_better (optimize.cpp:144-149): score, then lexicographic shift, then angle
bool better(const WindowOutcome& a, const WindowOutcome& b) {
    if (a.norm_score != b.norm_score) return a.norm_score > b.norm_score;
    for (int i = 0; i < 3; ++i)
        if (a.shift[i] != b.shift[i]) return a.shift[i] < b.shift[i];
    return q_angle(Quat{a.quat[0], a.quat[1], a.quat[2], a.quat[3]}) <
           q_angle(Quat{b.quat[0], b.quat[1], b.quat[2], b.quat[3]});
}
}  // namespace

namespace {
bool host_pointer(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();  // unregistered host memory on older drivers
        return true;
    }
    return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}
}  // namespace

const float* Context::device_particles(const float* particles, int count) {
    if (count <= 0 || !host_pointer(particles)) return particles;
    const size_t bytes = sizeof(float) * (size_t)n * n * n * count;
    // the copy staged by the last bm_align_batch serves this call only when the
    // caller opted in (bm_context_set_stage_reuse), only for the same buffer and
    // count, and only once; otherwise the host buffer is staged again
    const bool reuse = stage_reuse_ && staged_valid_ && particles == staged_src_ && count == staged_count_;
    staged_valid_ = false;
    staged_src_ = nullptr;
    if (!reuse) {
        staged_.reserve(bytes);
        ck(cudaMemcpyAsync(staged_.p, particles, bytes, cudaMemcpyHostToDevice, stream), "stage particles");
    }
    return staged_.as<float>();
}

std::vector<ParticleResult> Context::align_batch(const float* particles, int count, const AlignConfig& cfg) {
    // any earlier staged copy is stale from here on, whatever happens below
    staged_valid_ = false;
    staged_src_ = nullptr;
    std::vector<ParticleResult> out = align_batch_impl(particles, count, cfg);
    if (count > 0 && host_pointer(particles)) {  // complete: the staged copy holds these bytes
        staged_src_ = particles;
        staged_count_ = count;
        staged_valid_ = true;
    }
    return out;
}

std::vector<ParticleResult> Context::align_batch_impl(const float* particles, int count, const AlignConfig& cfg) {
    if (!has_template) throw std::invalid_argument("align: set_template first");
    cfg.validate(basis.l_max);
    const int k = std::max(1, std::min(lanes, count / std::max(1, lane_min_particles)));
    const bool host = count > 0 && host_pointer(particles);
    float* stage = nullptr;
    if (host) {
        staged_.reserve(sizeof(float) * (size_t)n * n * n * count);
        stage = staged_.as<float>();
    }
    // slice [o, o + c) of the batch on the device: staged on stream s when host-resident
    auto slice = [&](int o, int c, cudaStream_t s) -> const float* {
        const long long vs = (long long)n * n * n;
        if (!host) return particles + o * vs;
        ck(cudaMemcpyAsync(stage + o * vs, particles + o * vs, sizeof(float) * vs * c, cudaMemcpyHostToDevice, s),
           "stage particles");
        return stage + o * vs;
    };
    if (k <= 1) return align_batch_lane(slice(0, count, stream), count, cfg);
    ensure_lanes();
    // the lanes start after the work already queued on this context's stream
    cudaEvent_t ready;
    ck(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "lane event");
    ck(cudaEventRecord(ready, stream), "lane event");
    const long long vstride = (long long)n * n * n;
    std::vector<int> off(k + 1, 0);
    for (int i = 0; i < k; ++i) off[i + 1] = off[i] + count / k + (i < count % k ? 1 : 0);
    std::vector<std::vector<ParticleResult>> part(k);
    std::vector<std::exception_ptr> err(k);
    std::vector<std::thread> threads;
    // host particles: stage the slices in lane order, each copy after the previous
    // one, so lane 0 starts computing after its own slice instead of after all
    std::vector<const float*> dev_slice(k);
    if (host) {
        cudaEvent_t prev = ready;
        std::vector<cudaEvent_t> done(k);
        for (int i = 0; i < k; ++i) {
            cudaStream_t s = i == 0 ? stream : lane_ctx_[i - 1]->stream;
            ck(cudaStreamWaitEvent(s, prev, 0), "stage order");
            dev_slice[i] = slice(off[i], off[i + 1] - off[i], s);
            ck(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "stage event");
            ck(cudaEventRecord(done[i], s), "stage event");
            prev = done[i];
        }
        for (auto& e : done) cudaEventDestroy(e);  // released once their work completes
    } else {
        for (int i = 0; i < k; ++i) dev_slice[i] = particles + off[i] * vstride;
    }
    for (int i = 1; i < k; ++i)
        threads.emplace_back([&, i] {
            try {
                Context& c = *lane_ctx_[i - 1];
                ck(cudaSetDevice(device), "lane device");
                ck(cudaStreamWaitEvent(c.stream, ready, 0), "lane wait");
                c.timer.on = timer.on;
                part[i] = c.align_batch_lane(dev_slice[i], off[i + 1] - off[i], cfg);
            } catch (...) {
                err[i] = std::current_exception();
            }
        });
    try {
        part[0] = align_batch_lane(dev_slice[0], off[1], cfg);
    } catch (...) {
        err[0] = std::current_exception();
    }
    for (auto& t : threads) t.join();
    cudaEventDestroy(ready);
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
    std::vector<ParticleResult> out;
    out.reserve(count);
    for (int i = 0; i < k; ++i) {
        out.insert(out.end(), part[i].begin(), part[i].end());
        if (i > 0) timer.absorb(lane_ctx_[i - 1]->timer);
    }
    return out;
}

void Context::ensure_lanes() {
    while ((int)lane_ctx_.size() < lanes - 1) {
        auto c = std::make_unique<Context>(device, n, basis.l_max, basis.lambda_cut);
        c->lanes = 1;
        lane_ctx_.push_back(std::move(c));
    }
    for (auto& c : lane_ctx_) {
        c->expand_mode = expand_mode;
        c->pairs_mode = pairs_mode;
        c->pool_budget_ = pool_budget_;  // each lane allocates only what its slice needs
    }
    // lanes created after set_template (a larger set_lanes) adopt it too
    for (auto& c : lane_ctx_)
        if (lanes_stale_ || !c->has_template) c->adopt_template(*this);
    lanes_stale_ = false;
}

// a lane's template state: its own expansion of the template and wedge filter,
// the wedge-power factors copied from the main context
void Context::adopt_template(const Context& src) {
    std::vector<int> wv{0}, ws{0, 0, 0};
    expand_windows(src.tmpl_copy_.as<float>(), (long long)n * n * n, 1, wv, ws);
    t_hat.reserve(sizeof(float) * geo.m_pad);
    ck(cudaMemcpyAsync(t_hat.p, coef.p, sizeof(float) * geo.m_pad, cudaMemcpyDeviceToDevice, stream), "t_hat");
    t_norm = src.t_norm;
    wedge_deg = src.wedge_deg;
    wedge.reset();
    chi_hat = src.chi_hat;
    q_hat = src.q_hat;
    wp_total = src.wp_total;
    if (src.wedge) wedge = std::make_unique<WedgeFilter>(n, wedge_deg, kWedgeTaperDeg);
    ck(cudaStreamSynchronize(stream), "adopt template");
    build_side_template();
    bands_.clear();
    seeds_.clear();
    has_template = true;
}

std::vector<ParticleResult> Context::align_batch_lane(const float* particles, int count, const AlignConfig& cfg) {
    std::vector<ParticleResult> out(count);
    if (count == 0) return out;
    const long long vstride = (long long)n * n * n;
    const float* fw = particles;
    if (wedge) {  // missing-wedge restriction before any window (optimize.cpp:445)
        filtered.reserve(sizeof(float) * vstride * count);
        cudaEvent_t w0 = timer.begin(stream);
        wedge->apply(particles, filtered.as<float>(), count, stream);
        ++timer.launches;  // the profile multiply (cuFFT kernels are library launches)
        timer.end(K_WEDGE, w0, stream);
        fw = filtered.as<float>();
    }
    if (!cfg.auto_bands) {
        std::vector<int> all(count);
        for (int p = 0; p < count; ++p) all[p] = p;
        align_group(fw, count, all, cfg, out);
        return out;
    }
    // auto_bands (optimize.cpp:455-460): each particle's schedule from its zero-shift
    // kernel; particles sharing a schedule are aligned together
    const std::vector<std::vector<int>> sched = auto_band_schedules(fw, count, cfg.band_thresholds);
    std::map<std::vector<int>, std::vector<int>> groups;
    for (int p = 0; p < count; ++p) groups[sched[p]].push_back(p);
    for (const auto& [bands, members] : groups) {
        AlignConfig c = cfg;
        c.auto_bands = false;
        c.bands = bands;
        c.validate(basis.l_max);
        align_group(fw, count, members, c, out);
    }
    return out;
}

// select_bands (optimize.cpp:179-195) of xi_coefficients(expand(f_w), t_hat) for every
// particle: band energies ||xi_l||^2 in FP64 on the host from the FP32 expansions
std::vector<std::vector<int>> Context::auto_band_schedules(const float* fw, int count,
                                                           const std::vector<double>& thresholds) {
    const long long vstride = (long long)n * n * n;
    std::vector<int> wv(count), ws(3 * (size_t)count, 0);
    for (int p = 0; p < count; ++p) wv[p] = p;
    expand_windows(fw, vstride, count, wv, ws);
    const int ld = geo.m_pad, C = geo.coeffs, L = basis.l_max;
    std::vector<float> f((size_t)count * ld), t(ld);
    ck(cudaMemcpyAsync(f.data(), coef.p, sizeof(float) * f.size(), cudaMemcpyDeviceToHost, stream), "auto bands f");
    ck(cudaMemcpyAsync(t.data(), t_hat.p, sizeof(float) * ld, cudaMemcpyDeviceToHost, stream), "auto bands t");
    ck(cudaStreamSynchronize(stream), "auto bands");
    (void)C;
    std::vector<std::vector<int>> out(count);
    int zero_energy = 0;
#pragma omp parallel for schedule(dynamic) reduction(| : zero_energy)
    for (int p = 0; p < count; ++p) {
        const float* fp = f.data() + (size_t)p * ld;
        std::vector<double> energy(L + 1, 0.0);
        std::vector<std::complex<double>> Fm, Tm;
        for (int l = 0; l <= L; ++l) {
            const int nk = basis.radial_count(l), w = 2 * l + 1;
            Fm.assign((size_t)nk * w, 0.0);
            Tm.assign((size_t)nk * w, 0.0);
            for (int k = 0; k < nk; ++k)
                for (int m = -l; m <= l; ++m) {
                    const int am = m < 0 ? -m : m;
                    auto val = [&](const float* src) {
                        const float* row = src + basis.block_off[l] + k * w;
                        std::complex<double> z = am == 0 ? std::complex<double>(row[0], 0.0)
                                                         : std::complex<double>(row[2 * am - 1], row[2 * am]);
                        if (m < 0) z = ((am & 1) ? -1.0 : 1.0) * std::conj(z);  // real-volume symmetry
                        return z;
                    };
                    Fm[(size_t)k * w + (m + l)] = val(fp);
                    Tm[(size_t)k * w + (m + l)] = val(t.data());
                }
            double e = 0.0;
            for (int m = 0; m < w; ++m)
                for (int mp = 0; mp < w; ++mp) {
                    std::complex<double> x = 0.0;
                    for (int k = 0; k < nk; ++k) x += std::conj(Fm[(size_t)k * w + m]) * Tm[(size_t)k * w + mp];
                    e += std::norm(x);
                }
            energy[l] = e;
        }
        double total = 0.0;
        for (double e : energy) total += e;
        if (!(total > 0.0)) {
            zero_energy = 1;
            continue;
        }
        std::vector<double> ratio(L + 1, 0.0);
        for (int l = 0; l <= L; ++l) {
            double high = 0.0;
            for (int j = l + 1; j <= L; ++j) high += energy[j];
            ratio[l] = high / total;
        }
        std::vector<int> bands;
        for (double tau : thresholds)
            for (int l = 0; l <= L; ++l)
                if (ratio[l] <= tau) {
                    bands.push_back(l);
                    break;
                }
        std::sort(bands.begin(), bands.end());
        bands.erase(std::unique(bands.begin(), bands.end()), bands.end());
        out[p] = bands;
    }
    if (zero_energy) throw std::domain_error("energy_ratio: zero kernel energy");
    return out;
}

// coarse + fine shift stages of align() (optimize.cpp:463-521) for the listed
// particles (indices into the n_vol volumes at fw), all with cfg.bands
void Context::align_group(const float* fw, int n_vol, const std::vector<int>& parts, const AlignConfig& cfg,
                          std::vector<ParticleResult>& out) {
    std::vector<std::array<int, 3>> coarse;
    for (int z = -cfg.shift_radius; z <= cfg.shift_radius; z += cfg.shift_step)
        for (int y = -cfg.shift_radius; y <= cfg.shift_radius; y += cfg.shift_step)
            for (int x = -cfg.shift_radius; x <= cfg.shift_radius; x += cfg.shift_step) coarse.push_back({x, y, z});
    std::vector<int> wv, ws;
    for (int p : parts)
        for (const auto& s : coarse) {
            wv.push_back(p);
            ws.insert(ws.end(), s.begin(), s.end());
        }
    // the coarse and fine passes read the same volumes: one x-paired copy serves both
    struct PairHold {
        Context& c;
        explicit PairHold(Context& x) : c(x) { c.pairs_hold_ = true; c.pairs_src_ = nullptr; c.quads_src_ = nullptr; }
        ~PairHold() { c.pairs_hold_ = c.quads_hold_ = false; c.pairs_src_ = c.quads_src_ = nullptr; }
    } hold(*this);
    const auto t_coarse = std::chrono::steady_clock::now();
    std::vector<WindowOutcome> oc = run_windows(fw, n_vol, wv, ws, cfg);
    const double coarse_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_coarse).count();
    std::vector<int> best(n_vol, -1);
    std::vector<long long> cand(n_vol, 0), evals(n_vol, 0);
    std::vector<std::array<long long, kMaxBands>> band_evals(n_vol);
    for (auto& b : band_evals) b.fill(0);
    std::vector<int> nwin(n_vol, 0);
    for (size_t i = 0; i < oc.size(); ++i) {
        const int p = oc[i].particle;
        cand[p] += oc[i].n_cand;
        evals[p] += oc[i].evals;
        for (int b = 0; b < kMaxBands; ++b) band_evals[p][b] += oc[i].band_evals[b];
        ++nwin[p];
        if (oc[i].valid && (best[p] < 0 || better(oc[i], oc[best[p]]))) best[p] = (int)i;
    }
    for (int p : parts)
        if (best[p] < 0) throw std::invalid_argument("align: no usable shift window (empty subtomogram)");
    // fine pass: unit-step cube around the coarse winner, minus coarse points (optimize.cpp:490-501)
    std::vector<int> fv, fs;
    for (int p : parts) {
        const int* b = oc[best[p]].shift;
        for (int z = -cfg.shift_step; z <= cfg.shift_step; ++z)
            for (int y = -cfg.shift_step; y <= cfg.shift_step; ++y)
                for (int x = -cfg.shift_step; x <= cfg.shift_step; ++x) {
                    const std::array<int, 3> s{b[0] + x, b[1] + y, b[2] + z};
                    if (std::find(coarse.begin(), coarse.end(), s) != coarse.end()) continue;
                    fv.push_back(p);
                    fs.insert(fs.end(), s.begin(), s.end());
                }
    }
    const auto t_fine = std::chrono::steady_clock::now();
    std::vector<WindowOutcome> fo = run_windows(fw, n_vol, fv, fs, cfg);
    const double fine_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_fine).count();
    std::vector<WindowOutcome> bestw(n_vol);
    for (int p : parts) bestw[p] = oc[best[p]];
    for (const auto& o : fo) {
        const int p = o.particle;
        cand[p] += o.n_cand;
        evals[p] += o.evals;
        for (int b = 0; b < kMaxBands; ++b) band_evals[p][b] += o.band_evals[b];
        ++nwin[p];
        if (o.valid && better(o, bestw[p])) bestw[p] = o;
    }
    for (int p : parts) {
        ParticleResult& r = out[p];
        for (int i = 0; i < 3; ++i) r.shift[i] = bestw[p].shift[i];
        for (int i = 0; i < 4; ++i) r.quat[i] = bestw[p].quat[i];
        r.score = bestw[p].norm_score;
        r.converged = bestw[p].converged;
        r.candidates = cand[p];
        r.evaluations = evals[p];
        r.subtomo_norm = bestw[p].sub_norm;
        r.windows = nwin[p];
        r.bands = cfg.bands;
        r.evaluations_per_band.assign(band_evals[p].begin(), band_evals[p].begin() + cfg.bands.size());
        r.coarse_search_s = coarse_s;  // of the whole group (the stages run batched)
        r.fine_search_s = fine_s;
        r.expand_template_s = template_s_;
    }
}

void Context::read_eval_stats(long long* evals, double* flops, bool reset) {
    std::vector<unsigned long long> h(kEvalStats, 0ull);
    ck(cudaMemcpyAsync(h.data(), eval_stats(), sizeof(unsigned long long) * kEvalStats, cudaMemcpyDeviceToHost,
                       stream),
       "eval stats");
    ck(cudaStreamSynchronize(stream), "eval stats");
    long long e2 = 0, e0 = 0;
    double fl = 0.0;
    for (int L = 0; L <= kMaxL; ++L)
        for (int o = 0; o < 2; ++o)
            for (int w = 0; w < 2; ++w) {
                const unsigned long long c = h[((size_t)L * 2 + o) * 2 + w];
                (o ? e2 : e0) += (long long)c;
                fl += (double)c * eval_flops(L, o ? 2 : 0, w != 0);
            }
    for (auto& c : lane_ctx_) {
        long long le[2] = {0, 0};
        double lf = 0.0;
        c->read_eval_stats(le, &lf, reset);
        e2 += le[0];
        e0 += le[1];
        fl += lf;
    }
    if (evals) evals[0] = e2, evals[1] = e0;
    if (flops) *flops = fl;
    if (reset) ck(cudaMemsetAsync(eval_stats(), 0, sizeof(unsigned long long) * kEvalStats, stream), "eval stats");
}

void Context::eval_counts(int L, long long* out) {
    std::vector<unsigned long long> h(kEvalStats);
    ck(cudaMemcpyAsync(h.data(), eval_stats(), sizeof(unsigned long long) * kEvalStats, cudaMemcpyDeviceToHost,
                       stream), "eval counts");
    ck(cudaStreamSynchronize(stream), "eval counts");
    out[0] = (long long)(h[((size_t)L * 2 + 1) * 2] + h[((size_t)L * 2 + 1) * 2 + 1]);
    out[1] = (long long)(h[((size_t)L * 2) * 2] + h[((size_t)L * 2) * 2 + 1]);
    for (auto& c : lane_ctx_) {
        long long o[2];
        c->eval_counts(L, o);
        out[0] += o[0];
        out[1] += o[1];
    }
}

}  // namespace bmb
