// ballmatch-b200: command-line front end of the B200 alignment path (SURVEY §8(f)
// row 3), following the reference CLI's contract (tools/main.cpp:25-26, 41-77,
// 221-268):
// - exit codes: 0 success, 2 usage, 3 non-convergence, 4 I/O, 1 other;
// - JSON reports with the reference's keys;
// - the same align flags.
//
// Subcommands:
//   align        one template / one subtomogram (cmd_align)
//   align-batch  one template / a stack of subtomograms (new): per-particle results,
//                optional coefficient-space average written as an MRC map
//   expand       ball-harmonic expansion report (cmd_expand)
//
// Not ported: phantom (the data generator), bandscan and bench (the exhaustive
// baseline) — control plane outside the hot path.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <numbers>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "ballmatch_b200.hpp"
#include "ballmatch_b200_io.hpp"

namespace bm = ballmatch_b200;

namespace {

constexpr const char* kVersion = "0.1.0-b200";
constexpr double kPi = std::numbers::pi;
enum ExitCode : int { kOk = 0, kUsage = 2, kNoConverge = 3, kIo = 4 };

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ tiny JSON writer
struct Json {
    std::ostringstream s;
    bool first = true;
    static std::string esc(const std::string& v) {
        std::string o = "\"";
        for (char c : v) {
            if (c == '"' || c == '\\') o += '\\';
            o += c;
        }
        return o + "\"";
    }
    static std::string num(double v) {
        std::ostringstream t;
        t << std::setprecision(17) << v;
        return t.str();
    }
    template <class T>
    static std::string arr(const std::vector<T>& v) {
        std::string o = "[";
        for (size_t i = 0; i < v.size(); ++i) o += (i ? ", " : "") + num(static_cast<double>(v[i]));
        return o + "]";
    }
};
struct Obj {
    std::vector<std::pair<std::string, std::string>> kv;
    Obj& add(const std::string& k, const std::string& raw) {
        kv.emplace_back(k, raw);
        return *this;
    }
    Obj& num(const std::string& k, double v) { return add(k, Json::num(v)); }
    Obj& str(const std::string& k, const std::string& v) { return add(k, Json::esc(v)); }
    Obj& flag(const std::string& k, bool v) { return add(k, v ? "true" : "false"); }
    std::string dump(int indent = 0) const {
        const std::string pad(indent + 2, ' ');
        std::string o = "{\n";
        for (size_t i = 0; i < kv.size(); ++i)
            o += pad + Json::esc(kv[i].first) + ": " + kv[i].second + (i + 1 < kv.size() ? ",\n" : "\n");
        return o + std::string(indent, ' ') + "}";
    }
};

void write_text(const std::string& text, const std::string& path) {
    std::ofstream out(path, std::ios::trunc);
    if (!out) throw bm::io_error("cannot open " + path + " for writing");
    out << text << "\n";
    if (!out) throw bm::io_error("write failed for " + path);
}

// ------------------------------------------------------------------ flags
struct Args {
    std::map<std::string, std::string> kv;
    std::vector<std::string> switches;
    bool has(const std::string& k) const { return kv.count(k) != 0; }
    bool on(const std::string& k) const {
        for (const auto& s : switches)
            if (s == k) return true;
        return false;
    }
    std::string get(const std::string& k, const std::string& def = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? def : it->second;
    }
    double d(const std::string& k, double def) const {
        if (!has(k)) return def;
        try {
            return std::stod(get(k));
        } catch (...) {
            throw UsageError("--" + k + " expects a number");
        }
    }
    int i(const std::string& k, int def) const {
        if (!has(k)) return def;
        try {
            return std::stoi(get(k));
        } catch (...) {
            throw UsageError("--" + k + " expects an integer");
        }
    }
    template <class T>
    std::vector<T> list(const std::string& k, std::vector<T> def) const {
        if (!has(k)) return def;
        std::vector<T> out;
        std::stringstream ss(get(k));
        std::string tok;
        while (std::getline(ss, tok, ',')) {
            try {
                out.push_back(static_cast<T>(std::stod(tok)));
            } catch (...) {
                throw UsageError("--" + k + " expects a comma-separated list");
            }
        }
        return out;
    }
};

Args parse(int argc, char** argv, int from, const std::vector<std::string>& switches) {
    Args a;
    for (int k = from; k < argc; ++k) {
        std::string s = argv[k];
        if (s.rfind("--", 0) != 0) throw UsageError("unexpected argument " + s);
        s = s.substr(2);
        bool is_switch = false;
        for (const auto& w : switches) is_switch |= (w == s);
        if (is_switch) {
            a.switches.push_back(s);
            continue;
        }
        if (k + 1 >= argc) throw UsageError("--" + s + " needs a value");
        a.kv[s] = argv[++k];
    }
    return a;
}

struct AlignFlags {
    bm::OptimizerConfig cfg;
    double wedge_theta = 0.0;
    std::string report, truth;
    void read(const Args& a) {
        cfg.fixed_bands = a.list<int>("bands", {7, 12, 33});
        cfg.l_max = a.i("lmax", 42);
        cfg.lambda_cut = a.d("lambda-cut", 0.0);
        cfg.auto_bands = a.on("auto-bands");
        cfg.band_thresholds = a.list<double>("band-thresholds", {0.5, 0.25, 0.05});
        wedge_theta = a.d("wedge", 0.0);
        cfg.shift_radius = a.i("shift-radius", 4);
        cfg.shift_step = a.i("shift-step", 2);
        cfg.seed_grid_step = a.d("grid-step-deg", 22.5) * kPi / 180.0;
        cfg.max_candidates = a.i("max-candidates", 20);
        cfg.newton_max_iter = a.i("newton-max-iter", 30);
        cfg.threads = a.i("threads", 0);
        cfg.prune_after_band = a.on("prune-after-band");
        cfg.device = a.i("device", -1);
        report = a.get("report");
        truth = a.get("truth");
    }
    std::optional<bm::WedgeMask> wedge(int n) const {
        if (wedge_theta <= 0.0) return std::nullopt;
        return bm::build_wedge_mask(n, wedge_theta);
    }
};
const std::vector<std::string> kAlignSwitches{"auto-bands", "prune-after-band"};

std::string rotation_json(const bm::Rotation& g) {
    const bm::EulerZyz e = g.euler_zyz();
    return Obj()
        .add("quaternion_wxyz", Json::arr(std::vector<double>{g.w(), g.x(), g.y(), g.z()}))
        .add("euler_zyz_deg", Json::arr(std::vector<double>{e.alpha * 180 / kPi, e.beta * 180 / kPi, e.gamma * 180 / kPi}))
        .dump(4);
}

std::string config_json(const bm::OptimizerConfig& c, double wedge, double cut_eff) {
    Obj o;
    o.num("l_max", c.l_max)
        .num("lambda_cut", c.lambda_cut)
        .add("bands", Json::arr(c.fixed_bands))
        .flag("auto_bands", c.auto_bands)
        .add("band_thresholds", Json::arr(c.band_thresholds))
        .num("seed_grid_step_deg", c.seed_grid_step * 180.0 / kPi)
        .num("max_candidates", c.max_candidates)
        .num("newton_max_iter", c.newton_max_iter)
        .num("grad_tol", c.grad_tol)
        .num("step_damping", c.step_damping)
        .num("shift_radius", c.shift_radius)
        .num("shift_step", c.shift_step)
        .num("threads", c.threads)
        .flag("prune_after_band", c.prune_after_band)
        .str("generator", "ballmatch-b200 (B200 sm_100a)")
        .num("lambda_cut_effective", cut_eff);
    if (wedge > 0.0) o.num("wedge_theta_deg", wedge);
    return o.dump(2);
}

std::string result_json(const bm::AlignmentResult& r, int indent) {
    Obj per_band;
    for (const auto& [band, n] : r.evaluations_per_band) per_band.num(std::to_string(band), static_cast<double>(n));
    return Obj()
        .add("shift_voxels", Json::arr(std::vector<int>{r.shift[0], r.shift[1], r.shift[2]}))
        .add("rotation", rotation_json(r.rotation))
        .num("score", r.score)
        .flag("converged", r.converged)
        .num("candidates_evaluated", static_cast<double>(r.candidates_evaluated))
        .num("evaluations", static_cast<double>(r.evaluations))
        .add("evaluations_per_band", per_band.dump(indent + 2))
        .add("bands", Json::arr(r.bands))
        .num("template_norm", r.template_norm)
        .num("subtomo_norm", r.subtomo_norm)
        .num("windows", r.windows)
        .add("timings", Obj()
                            .num("expand_template_s", r.expand_template_s)
                            .num("coarse_search_s", r.coarse_search_s)
                            .num("fine_search_s", r.fine_search_s)
                            .num("wall_s", r.wall_time_s)
                            .dump(indent + 2))
        .dump(indent);
}

// truth.json of the reference's phantom command: rotation.quaternion_wxyz, shift_voxels
std::vector<double> json_numbers_after(const std::string& text, const std::string& key) {
    const size_t k = text.find("\"" + key + "\"");
    if (k == std::string::npos) return {};
    const size_t b = text.find('[', k), e = text.find(']', b);
    if (b == std::string::npos || e == std::string::npos) return {};
    std::vector<double> out;
    std::stringstream ss(text.substr(b + 1, e - b - 1));
    std::string tok;
    while (std::getline(ss, tok, ',')) out.push_back(std::stod(tok));
    return out;
}

std::string truth_comparison(const std::string& path, const bm::AlignmentResult& r) {
    std::ifstream in(path);
    if (!in) throw bm::io_error("cannot open " + path);
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    const auto q = json_numbers_after(text, "quaternion_wxyz");
    if (q.size() != 4) throw bm::io_error("truth: no rotation.quaternion_wxyz in " + path);
    Obj o;
    o.num("geodesic_error_deg", bm::geodesic_degrees(r.rotation, bm::Rotation(q[0], q[1], q[2], q[3])));
    const auto s = json_numbers_after(text, "shift_voxels");
    if (s.size() == 3) {
        std::vector<int> d(3);
        bool exact = true;
        for (int i = 0; i < 3; ++i) {
            d[i] = r.shift[i] - static_cast<int>(s[i]);
            exact &= d[i] == 0;
        }
        o.add("shift_error_voxels", Json::arr(d)).flag("shift_exact", exact);
    }
    return o.dump(2);
}

// ------------------------------------------------------------------ commands
int cmd_align(const Args& a) {
    if (!a.has("template") || !a.has("subtomo")) throw UsageError("align needs --template and --subtomo");
    AlignFlags f;
    f.read(a);
    const bm::Volume tmpl = bm::read_mrc(a.get("template"));
    const bm::Volume sub = bm::read_mrc(a.get("subtomo"));
    f.cfg.validate();
    const bm::AlignmentResult res = bm::align(tmpl, sub, f.cfg, f.wedge(tmpl.n));
    const double cut = f.cfg.lambda_cut > 0.0 ? f.cfg.lambda_cut : bm::default_lambda_cut(tmpl.n, f.cfg.l_max);
    Obj rep;
    rep.str("version", kVersion).str("command", "align").add("config", config_json(f.cfg, f.wedge_theta, cut));
    rep.add("result", result_json(res, 2));
    if (!f.truth.empty()) rep.add("truth_comparison", truth_comparison(f.truth, res));
    if (!f.report.empty()) write_text(rep.dump(), f.report);
    const bm::EulerZyz e = res.rotation.euler_zyz();
    std::cout << "align: shift = (" << res.shift[0] << ", " << res.shift[1] << ", " << res.shift[2]
              << ")  euler_zyz_deg = (" << e.alpha * 180.0 / kPi << ", " << e.beta * 180.0 / kPi << ", "
              << e.gamma * 180.0 / kPi << ")  score = " << res.score
              << "  converged = " << (res.converged ? "yes" : "no") << "\n";
    return res.converged ? kOk : kNoConverge;
}

int cmd_align_batch(const Args& a) {
    if (!a.has("template") || (!a.has("stack") && !a.has("subtomos")))
        throw UsageError("align-batch needs --template and --stack (or --subtomos a.mrc,b.mrc,...)");
    AlignFlags f;
    f.read(a);
    const bm::Volume tmpl = bm::read_mrc(a.get("template"));
    std::vector<bm::Volume> subs;
    if (a.has("stack")) {
        subs = bm::read_mrc_stack(a.get("stack"));
    } else {
        std::stringstream ss(a.get("subtomos"));
        std::string p;
        while (std::getline(ss, p, ',')) subs.push_back(bm::read_mrc(p));
    }
    f.cfg.validate();
    const int chunk = a.i("chunk", 1024);
    bm::Aligner al(tmpl, f.cfg, f.wedge(tmpl.n));
    const auto res = al.align_batch(subs, chunk);
    const double cut = f.cfg.lambda_cut > 0.0 ? f.cfg.lambda_cut : bm::default_lambda_cut(tmpl.n, f.cfg.l_max);
    std::string results = "[\n";
    int converged = 0;
    for (size_t p = 0; p < res.size(); ++p) {
        results += "    " + result_json(res[p], 4) + (p + 1 < res.size() ? ",\n" : "\n");
        converged += res[p].converged ? 1 : 0;
    }
    results += "  ]";
    Obj rep;
    rep.str("version", kVersion)
        .str("command", "align-batch")
        .add("config", config_json(f.cfg, f.wedge_theta, cut))
        .num("particles", static_cast<double>(res.size()))
        .num("converged", converged)
        .add("results", results);
    if (a.has("average")) {  // coefficient-space average, synthesized onto the template grid
        al.accumulate_average(subs, res, chunk);
        const bm::BallExpansion avg = al.average();
        bm::Volume map = bm::synthesize(avg, tmpl.n, tmpl.voxel_size);
        bm::write_mrc(map, a.get("average"));
        rep.str("average_map", a.get("average"));
    }
    if (!f.report.empty()) write_text(rep.dump(), f.report);
    std::cout << "align-batch: " << res.size() << " particles, " << converged << " converged";
    if (!res.empty()) std::cout << ", wall " << res[0].wall_time_s << " s";
    std::cout << "\n";
    return converged == static_cast<int>(res.size()) ? kOk : kNoConverge;
}

int cmd_expand(const Args& a) {
    if (!a.has("in") || !a.has("out")) throw UsageError("expand needs --in and --out");
    const bm::Volume v = bm::read_mrc(a.get("in"));
    const int l_max = a.i("lmax", 42);
    const double cut = a.d("lambda-cut", 0.0) > 0.0 ? a.d("lambda-cut", 0.0) : bm::default_lambda_cut(v.n, l_max);
    const bm::BasisSpec spec = bm::build_spec(l_max, cut);
    const bm::BallExpansion e = bm::expand(v, spec);
    std::string per_band = "[\n";
    for (int l = 0; l <= l_max; ++l) {
        double en = 0.0;
        const size_t cnt = static_cast<size_t>(spec.radial_count(l)) * (2 * l + 1);
        for (size_t i = 0; i < cnt; ++i) en += std::norm(e.block(l)[i]);
        per_band += "    " + Obj().num("band", l).num("energy", en).num("radial_count", spec.radial_count(l)).dump(4) +
                    (l < l_max ? ",\n" : "\n");
    }
    per_band += "  ]";
    Obj j;
    j.str("version", kVersion)
        .str("command", "expand")
        .num("n", v.n)
        .num("l_max", l_max)
        .num("lambda_cut", cut)
        .num("coeff_count", static_cast<double>(e.coeffs().size()))
        .num("energy", e.energy())
        .add("energy_per_band", per_band);
    if (a.has("coeffs-bin")) {
        std::ofstream bin(a.get("coeffs-bin"), std::ios::binary | std::ios::trunc);
        if (!bin) throw bm::io_error("cannot open " + a.get("coeffs-bin"));
        bin.write(reinterpret_cast<const char*>(e.coeffs().data()),
                  static_cast<std::streamsize>(e.coeffs().size() * sizeof(bm::cdouble)));
        j.str("coeffs_bin", a.get("coeffs-bin"))
            .str("coeffs_layout", "per degree l: k rows of 2l+1 complex<double> (m = -l..l), little-endian");
    }
    write_text(j.dump(), a.get("out"));
    std::cout << "expand: " << e.coeffs().size() << " coefficients, energy " << e.energy() << ", report "
              << a.get("out") << "\n";
    return kOk;
}

void usage() {
    std::cout << "ballmatch-b200 " << kVersion << ": subtomogram alignment in the ball-harmonics domain (B200)\n"
              << "usage: ballmatch-b200 <align|align-batch|expand> [--flag value ...]\n"
              << "  align        --template T.mrc --subtomo S.mrc [--report R.json] [--truth truth.json]\n"
              << "  align-batch  --template T.mrc (--stack P.mrc | --subtomos a.mrc,b.mrc) [--report R.json]\n"
              << "               [--average avg.mrc] [--chunk 1024]\n"
              << "  expand       --in V.mrc --out report.json [--lmax 42] [--lambda-cut X] [--coeffs-bin F]\n"
              << "  align flags: --bands 7,12,33 --lmax 42 --lambda-cut X --auto-bands --band-thresholds a,b,c\n"
              << "               --prune-after-band --wedge DEG --shift-radius 4 --shift-step 2 --grid-step-deg 22.5\n"
              << "               --max-candidates 20 --newton-max-iter 30 --threads 0 --device -1\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return kUsage;
    }
    const std::string cmd = argv[1];
    if (cmd == "--help" || cmd == "-h") {
        usage();
        return kOk;
    }
    if (cmd == "--version") {
        std::cout << kVersion << "\n";
        return kOk;
    }
    try {
        if (cmd == "align") return cmd_align(parse(argc, argv, 2, kAlignSwitches));
        if (cmd == "align-batch") return cmd_align_batch(parse(argc, argv, 2, kAlignSwitches));
        if (cmd == "expand") return cmd_expand(parse(argc, argv, 2, {}));
        std::cerr << "error: unknown command " << cmd << "\n";
        usage();
        return kUsage;
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kUsage;
    } catch (const bm::io_error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kIo;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kUsage;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
