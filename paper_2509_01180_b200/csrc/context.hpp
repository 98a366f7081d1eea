// Per-device context of the B200 alignment path: basis + operator resident in
// HBM, template state, per-band evaluation tables and grown-on-demand work
// buffers.  One context per device; calls on a context are stream-ordered on
// its stream and not thread-safe (one host thread per device).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cufft.h>

#include <complex>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "basis_host.hpp"
#include "bmb_internal.hpp"
#include "expand_factored.hpp"
#include "kernels.cuh"
#include "rotation.cuh"

namespace bmb {

// RAII device buffer
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    // grow (never shrink); contents are not preserved
    void reserve(size_t b) {
        if (b <= bytes) return;
        release();
        if (cudaMalloc(&p, b) != cudaSuccess) {
            p = nullptr;
            throw std::bad_alloc();
        }
        bytes = b;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

template <class T>
void upload(DevBuf& d, const std::vector<T>& h, cudaStream_t s) {
    d.reserve(sizeof(T) * (h.size() ? h.size() : 1));
    if (!h.empty())
        cudaMemcpyAsync(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, s);
}

struct WedgeFilter;

// device storage of one band's evaluation tables (+ the wedge entries)
struct BandDev {
    int L = 0;
    int n_items = 0, n_groups = 0, rows = 0;
    DevBuf row_off, item_mm, item_pm, item_w, item_len, bfac, bexp, PQR, item_of, out_pos, at_desc, row_group, wedge,
        wedge_side;
    bool has_wedge = false;
    BandTables view() const;
};

// seed-grid tables for one (L_low, grid step) and the current template
struct SeedDev {
    int L_low = 0, na = 0, nb = 0, ng = 0, nxi = 0;
    double step = 0.0;
    DevBuf dgrid, ua, ug, wedge_sqrt;
    bool has_wedge = false;
};

struct AlignConfig {
    std::vector<int> bands;
    double seed_grid_step;
    int max_candidates;
    int newton_max_iter;
    double grad_tol;
    double step_damping;
    int shift_radius;
    int shift_step;
    double accept_tol;
    bool auto_bands = false;
    bool prune_after_band = false;
    std::vector<double> band_thresholds{0.5, 0.25, 0.05};
    void validate(int l_max) const;  // OptimizerConfig::validate (optimize.cpp:153-177)
};

struct ParticleResult {
    int shift[3];
    double quat[4];
    double score;
    int converged;
    long long candidates;
    long long evaluations;
    double subtomo_norm;
    int windows;
    std::vector<int> bands;
    std::vector<long long> evaluations_per_band;  // aligned with bands (AlignmentResult, optimize.hpp:83)
    double expand_template_s = 0.0, coarse_search_s = 0.0, fine_search_s = 0.0;  // phase timings (batch level)
};

// Per-kernel-class CUDA-event timing on the context stream (bench evidence).
enum KClass { K_GATHER = 0, K_GEMM, K_SEED, K_REFINE, K_WEDGE, K_MISC, K_REFINE_B0, K_REFINE_B1, K_REFINE_B2, K_REFINE_B3, K_EVAL2, K_EVAL0, K_COMPOSE, K_NEWTON, K_XI, K_COUNT };
struct KernelTimer {
    bool on = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    double ms[K_COUNT] = {0};
    double band_ms[4][K_COUNT] = {{0}};  // per band index (refinement classes; last slot: bands >= 3)
    int band = -1;                        // band index of the launches being timed (-1: none)
    long long launches = 0;        // kernels of this library launched (always counted)
    long long windows_expanded = 0;
    long long gemm_launches = 0, refine_launches = 0;
    cudaEvent_t begin(cudaStream_t s) {
        if (!on) return nullptr;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        return e;
    }
    void end(int cls, cudaEvent_t b, cudaStream_t s) {
        if (!on || !b) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        pending.push_back({cls + (band >= 0 ? K_COUNT * (1 + (band < 3 ? band : 3)) : 0), {b, e}});
    }
    void collect() {
        for (auto& p : pending) {
            float t = 0.f;
            cudaEventSynchronize(p.second.second);
            cudaEventElapsedTime(&t, p.second.first, p.second.second);
            const int cls = p.first % K_COUNT, bi = p.first / K_COUNT - 1;
            ms[cls] += t;
            if (bi >= 0) band_ms[bi][cls] += t;
            cudaEventDestroy(p.second.first);
            cudaEventDestroy(p.second.second);
        }
        pending.clear();
    }
    void reset() {
        collect();
        for (double& x : ms) x = 0.0;
        for (auto& r : band_ms)
            for (double& x : r) x = 0.0;
        launches = windows_expanded = gemm_launches = refine_launches = 0;
    }
    // add another timer's totals (a lane's) and clear it
    void absorb(KernelTimer& o) {
        o.collect();
        for (int i = 0; i < K_COUNT; ++i) ms[i] += o.ms[i];
        for (int b = 0; b < 4; ++b)
            for (int i = 0; i < K_COUNT; ++i) band_ms[b][i] += o.band_ms[b][i];
        launches += o.launches;
        windows_expanded += o.windows_expanded;
        gemm_launches += o.gemm_launches;
        refine_launches += o.refine_launches;
        o.reset();
    }
};

class Context {
public:
    KernelTimer timer;
    Context(int device, int n, int l_max, double lambda_cut);
    ~Context();

    int device = 0;
    cudaStream_t stream = nullptr;
    int n = 0;
    host::Basis basis;
    Geometry geo;
    std::vector<int> voxels_host;

    // resident operator + geometry tables
    DevBuf E_hi, E_lo, row_scale, voxels, block_off, radial_count, row_weight, row_lkm;

    // work buffers
    DevBuf B_hi, B_lo, col_scale, coef, win_vol, win_shift, vol_scale, norms;
    DevBuf vol_pairs;  // x-paired particle volumes for the expansion gathers (many windows per volume)
    DevBuf vol_quads;  // zero-padded quad copy (kernel K2q) and its CTA pair list
    DevBuf win_pairs;
    bool quads_hold_ = false;
    const float* quads_src_ = nullptr;
    int quads_nvol_ = 0;
    long long quads_stride_ = 0;
    int pairs_mode = 1;                 // 0 off, 1 auto (>= 4 windows per volume), 2 always x-pairs, 3 always quads
    static constexpr size_t kMaxPairBytes = size_t(8) << 30;  // larger batches gather directly
    bool pairs_hold_ = false;           // inside align_group: vol_pairs may be reused for pairs_src_
    const float* pairs_src_ = nullptr;
    int pairs_nvol_ = 0;
    long long pairs_stride_ = 0;

    // expansion of `count` windows (volume index + integer shift) of volumes
    // already on the device; real-packed FP32 coefficients into ctx.coef
    // (row stride geo.m_pad), returns the number of windows.
    void expand_windows(const float* vols, long long vol_stride, int n_vol,
                        const std::vector<int>& wvol, const std::vector<int>& wshift);

    int expand_mode = 0;          // 0: factored expansion (K2f), 1: dense operator GEMM (K1 + K2)
    bool operator_ready = false;
    void ensure_operator();
    void build_factored_tables();
    FactoredTables fx;
    DevBuf fx_r, fx_samp, fx_tw, fx_ptab, fx_trilm, fx_radial, fx_rowmap;
    int gemm_block_n = 128;
    int gemm_kchunk = 4;
    long long max_chunk_windows = 8192;  // windows expanded per GEMM chunk

    // ---------------------------------------------------------- template
    DevBuf t_hat;          // real-packed FP32 template coefficients
    DevBuf t_side;         // D(K^-1) t_hat: template of the side kernels (refine.cu chart_transform)
    void build_side_template();
    double t_norm = 0.0;
    bool has_template = false;
    double template_s_ = 0.0;  // wall time of the last set_template
    double wedge_deg = 0.0;                // <= 0 or >= 90: no wedge
    std::unique_ptr<WedgeFilter> wedge;    // tapered filter for the particles
    std::vector<std::complex<double>> chi_hat, q_hat;  // wedge power factors
    std::vector<std::complex<double>> q_side;         // D(K^-1) q_hat (side wedge kernel)
    double wp_total = 0.0;
    bool wedge_active() const { return wedge_deg > 0.0 && wedge_deg < 90.0 && wp_total > 0.0; }
    void set_template(const float* tmpl, double wedge_deg);

    BandDev& band(int L);
    SeedDev& seed_tables(int L_low, double step);

    // seed_candidates for device coefficient sets (bm_seed_candidates)
    void seed_candidates(const double* f, int n_f, int L_low, double step, int max_cand, double* quats, int* counts,
                         double* scores);
    // Objective::eval of the refinement at n chart points (bm_objective_eval)
    void objective_eval(const double* f, const double* t, const double* euler, const double* anchors, int n, int L,
                        int order, double* out);

    // one window stage: search_one_shift for every (volume, shift) window
    std::vector<WindowOutcome> run_windows(const float* vols, int n_vol, const std::vector<int>& wvol,
                                           const std::vector<int>& wshift, const AlignConfig& cfg);
    // align() for a batch of particles (coarse + fine shift stages)
    // particles: device or host memory (host: each lane stages its own slice on
    // its stream right before aligning it, so the copies overlap other lanes'
    // work; the staged copy serves a following average of the same buffer)
    std::vector<ParticleResult> align_batch(const float* particles, int count, const AlignConfig& cfg);
    const float* device_particles(const float* particles, int count);  // staged copy of host particles
    DevBuf staged_;
    const float* staged_src_ = nullptr;
    int staged_count_ = 0;
    bool staged_valid_ = false;  // staged_ holds staged_src_'s bytes (set by a completed align_batch)
    bool stage_reuse_ = false;   // caller opt-in: bm_context_set_stage_reuse
    std::vector<ParticleResult> align_batch_impl(const float* particles, int count, const AlignConfig& cfg);
    std::vector<ParticleResult> align_batch_lane(const float* particles, int count, const AlignConfig& cfg);
    // concurrent lanes: sub-contexts with their own stream and buffers that align
    // slices of a large batch from their own host threads (overlapping the
    // low-occupancy tails of each lane's Newton loop)
    int lanes = 4;
    int lane_min_particles = 64;  // per lane
    std::vector<std::unique_ptr<Context>> lane_ctx_;
    DevBuf tmpl_copy_;
    bool lanes_stale_ = true;
    void ensure_lanes();
    void adopt_template(const Context& src);
    void align_group(const float* fw, int n_vol, const std::vector<int>& parts, const AlignConfig& cfg,
                     std::vector<ParticleResult>& out);
    std::vector<std::vector<int>> auto_band_schedules(const float* fw, int count, const std::vector<double>& thresholds);

    // rotate-score-gradient sweep (config 4): kernels from coefficient pairs
    DevBuf work_f, work_xi, filtered;

    bool debug_iters_ = std::getenv("BMB_DEBUG_ITERS") != nullptr;
    // Newton rounds: host reads of the list lengths in the tail (align.cpp run_windows)
    static constexpr int kTailCandidates = 8192;
    int round_check_ = [] {
        const char* e = std::getenv("BMB_ROUND_CHECK");
        return e ? std::atoi(e) : 4;
    }();
    // pinned host words for the per-iteration list counts (allocated once:
    // cudaMallocHost / cudaFreeHost per call stall the host unpredictably)
    int* pinned_ = nullptr;
    int* pinned_counts() {
        if (!pinned_ && cudaMallocHost(&pinned_, sizeof(int) * 16) != cudaSuccess) throw std::bad_alloc();
        return pinned_;
    }
    // synthesize() radial table (basis.cpp:221-245), built on first use
    DevBuf synth_table_, synth_pair_off_;
    void synthesize(const double* coef, bool real_volume, int n_out, double* out);
    DevBuf seed_scratch_;                   // seed xi when it does not fit in shared memory
    DevBuf eval_stats_;                     // [kMaxL+1][order 0/2][wedge 0/1] evaluation counts
    static constexpr size_t kEvalStats = (size_t)(kMaxL + 1) * 4;
    unsigned long long* eval_stats() {
        if (!eval_stats_.p) {
            eval_stats_.reserve(sizeof(unsigned long long) * kEvalStats);
            cudaMemsetAsync(eval_stats_.p, 0, sizeof(unsigned long long) * kEvalStats, stream);
        }
        return eval_stats_.as<unsigned long long>();
    }
    // evaluations (order 2, order 0) and their algorithmic FLOPs since the last reset
    void read_eval_stats(long long* evals, double* flops, bool reset);
    void eval_counts(int L, long long* out);  // (order 2, order 0) evaluations at band L
    // bytes of window + side kernels per refinement chunk (BMB_POOL_GB overrides)
    size_t pool_budget_ = [] {
        const char* e = std::getenv("BMB_POOL_GB");
        return (e && std::atoi(e) > 0) ? (size_t)std::atoi(e) << 30 : 24ull << 30;
    }();

private:
    void refine_windows(int nw, int maxc, const AlignConfig& cfg, const Quat& koff, long long grid_evals);
    DevBuf work_, counters_, xi_win_, xi_side_, lists_;
    std::map<int, std::unique_ptr<BandDev>> bands_;
    std::map<std::pair<int, long long>, std::unique_ptr<SeedDev>> seeds_;
    DevBuf cand_, cand_count_, outcome_, win_counter_, sub_norm_;
};

}  // namespace bmb
