// solkin_b200_config.hpp -- the reference's run configuration surface
// over the C ABI. Header-only.
//
//   reference                                      here
//   RunConfig (config.hpp:11-59, config.cpp)       solkin_b200::RunConfig
//   cmd_run's preset -> file -> flag layering      solkin_b200::resolve_run_config
//     (tools/solkin_main.cpp:20-28)
//   `solkin matrices` (solkin_main.cpp:43-57)      solkin_b200::matrices_text
//   run(const RunConfig&) (run.hpp, run.cpp:60)    solkin_b200::run(ctx, RunConfig)
//
// Same keys, defaults, presets, error messages and echo format as the
// reference; the key list is one table (visit_keys) shared by apply_kv and
// echo, so the two cannot drift apart. Parsing uses std::stod / std::stoi
// with a full-consumption check, like config.cpp:23-45.
#pragma once

#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include <sys/stat.h>

#include "solkin_b200.hpp"

namespace solkin_b200 {

struct RunConfig {
    std::string scenario = "blob";  // blob | injection
    double L = 200.0;
    double dt = 0.1;
    int k = 3;
    double mu = 400.0;
    double t_final = 400.0;
    double sigma = -1.0;  // <0: resolved to 0.1*L
    double t0 = 2000.0;   // injection source window
    double vmax_e = 12.0;
    double vmax_i = 12.0;
    int fine_block_cells = 50;
    int coarse_block_cells = 50;
    int refinement_ratio = 1;
    int v_cells = 40;
    std::string limiter = "none";
    double limiter_threshold = 0.5;
    bool v_adjust = true;
    double adapt_p = 0.05;
    double adapt_gamma = 0.05;
    double adapt_tol = 1e-14;
    double penalty_scale = 10.0;
    std::string out_dir = "out";
    int cadence = 10;          // flux row every N steps
    int snapshot_cadence = 0;  // 0 = off
    int profile_cadence = 0;   // 0 = off
    int threads = 1;           // accepted for parity; the device ignores it

    // blob-paper, injection-paper, blob-desk, injection-desk (config.cpp:58-86)
    static RunConfig preset(const std::string& name) {
        RunConfig c;
        struct Preset {
            const char* name;
            bool injection;
            int fine, coarse, m, nv;  // 0: keep the default
            double t_final;
        };
        static const Preset table[] = {
            {"blob-desk", false, 0, 0, 0, 0, 400.0},
            {"injection-desk", true, 0, 0, 0, 0, 400.0},
            {"blob-paper", false, 100, 100, 1, 150, 4000.0},
            {"injection-paper", true, 100, 100, 8, 150, 8000.0},
        };
        for (const Preset& p : table) {
            if (name != p.name) continue;
            if (p.injection) c.scenario = "injection";
            if (p.fine) {
                c.fine_block_cells = p.fine;
                c.coarse_block_cells = p.coarse;
                c.refinement_ratio = p.m;
                c.v_cells = p.nv;
            }
            c.t_final = p.t_final;
            return c;
        }
        throw std::runtime_error("unknown preset '" + name +
                                 "' (expected blob-paper, injection-paper, blob-desk, "
                                 "injection-desk)");
    }

    static RunConfig from_file(const std::string& path) {
        RunConfig c;
        c.apply_file(path);
        return c;
    }

    // flat key = value lines, '#' comments (config.cpp:93-109)
    void apply_file(const std::string& path) {
        std::ifstream in(path);
        if (!in.good()) throw std::runtime_error("cannot read config file '" + path + "'");
        std::string line;
        for (int lineno = 1; std::getline(in, line); ++lineno) {
            line = trim(line.substr(0, line.find('#')));
            if (line.empty()) continue;
            const size_t eq = line.find('=');
            if (eq == std::string::npos)
                throw std::runtime_error(path + ":" + std::to_string(lineno) + ": expected key = value");
            apply_kv(trim(line.substr(0, eq)), trim(line.substr(eq + 1)));
        }
    }

    void apply_kv(const std::string& key, const std::string& value) {
        bool found = false;
        visit_keys(*this, [&](const char* name, auto& field) {
            if (found || key != name) return;
            parse_into(key, value, field);
            found = true;
        });
        if (!found) throw std::runtime_error("unknown config key '" + key + "'");
    }

    void resolve() {
        if (sigma < 0) sigma = 0.1 * L;
    }

    // "key: message" per violation, in the reference's order (config.cpp:152-185)
    std::vector<std::string> violations() const {
        std::vector<std::string> out;
        auto need = [&](bool ok, const char* key, const char* msg) {
            if (!ok) out.push_back(std::string(key) + ": " + msg);
        };
        need(scenario == "blob" || scenario == "injection", "scenario", "must be blob or injection");
        need(L > 0, "L", "must be positive");
        need(dt > 0, "dt", "must be positive");
        need(k >= 0 && k <= 6, "k", "must be in 0..6");
        need(mu > 0, "mu", "must be positive");
        need(!(t_final < 0), "t_final", "must be >= 0");
        need(sigma > 0, "sigma", "must be positive (call resolve() to default to 0.1*L)");
        need(t0 > 0, "t0", "must be positive");
        need(vmax_e > 0, "vmax_e", "must be positive");
        need(vmax_i > 0, "vmax_i", "must be positive");
        need(fine_block_cells >= 1, "mesh.fine_block_cells", "must be >= 1");
        need(coarse_block_cells >= 1, "mesh.coarse_block_cells", "must be >= 1");
        need(refinement_ratio >= 1, "mesh.refinement_ratio", "must be >= 1");
        need(v_cells >= 1, "v_cells", "must be >= 1");
        bool limiter_ok = true;
        try {
            LimiterConfig::parse(limiter);
        } catch (const std::exception&) {
            limiter_ok = false;
        }
        need(limiter_ok, "limiter",
             "must be one of none, minmod+simple, minmod+line, meanerr+simple, meanerr+line, sldg");
        need(limiter_threshold > 0, "limiter.threshold", "must be positive");
        need(adapt_p > 0 && !(adapt_gamma < 0) && !(adapt_p + adapt_gamma >= 1), "adaptivity.p/gamma",
             "need 0 < p, 0 <= gamma, p + gamma < 1");
        need(adapt_tol > 0, "adaptivity.tol", "must be positive");
        need(penalty_scale > 0, "poisson.penalty_scale", "must be positive");
        need(cadence >= 1, "output.cadence", "must be >= 1");
        need(snapshot_cadence >= 0, "output.snapshot_cadence", "must be >= 0");
        need(profile_cadence >= 0, "output.profile_cadence", "must be >= 0");
        need(threads >= 1, "threads", "must be >= 1");
        return out;
    }

    void validate() const {
        const auto v = violations();
        if (v.empty()) return;
        std::string msg = "invalid configuration:";
        for (const auto& s : v) msg += "\n  " + s;
        throw std::runtime_error(msg);
    }

    // re-ingestible key = value echo (config.cpp:196-224)
    std::string echo() const {
        std::string out;
        visit_keys(*this, [&](const char* name, const auto& field) {
            out += name;
            out += " = ";
            out += format(field);
            out += "\n";
        });
        return out;
    }

    long nsteps() const { return std::lround(t_final / dt); }

    // the step-shaping subset the C ABI takes
    sk_run_config to_c() const {
        sk_run_config c{};
        c.L = L;
        c.dt = dt;
        c.mu = mu;
        c.sigma = sigma;
        c.vmax_e = vmax_e;
        c.vmax_i = vmax_i;
        c.k = k;
        c.fine_block_cells = fine_block_cells;
        c.coarse_block_cells = coarse_block_cells;
        c.refinement_ratio = refinement_ratio;
        c.v_cells = v_cells;
        c.limiter = LimiterConfig::parse(limiter).c;
        c.limiter.threshold = limiter_threshold;
        c.v_adjust = v_adjust ? 1 : 0;
        c.policy = sk_vadjust{adapt_p, adapt_gamma, adapt_tol};
        c.penalty_scale = penalty_scale;
        c.scenario = scenario == "injection" ? 1 : 0;
        c.t0 = t0;
        return c;
    }

  private:
    // every key, in echo order (config.cpp:111-137 / 196-224)
    template <class Self, class F>
    static void visit_keys(Self& c, F&& f) {
        f("scenario", c.scenario);
        f("L", c.L);
        f("dt", c.dt);
        f("k", c.k);
        f("mu", c.mu);
        f("t_final", c.t_final);
        f("sigma", c.sigma);
        f("t0", c.t0);
        f("vmax_e", c.vmax_e);
        f("vmax_i", c.vmax_i);
        f("mesh.fine_block_cells", c.fine_block_cells);
        f("mesh.coarse_block_cells", c.coarse_block_cells);
        f("mesh.refinement_ratio", c.refinement_ratio);
        f("v_cells", c.v_cells);
        f("limiter", c.limiter);
        f("limiter.threshold", c.limiter_threshold);
        f("adaptivity.v_adjust", c.v_adjust);
        f("adaptivity.p", c.adapt_p);
        f("adaptivity.gamma", c.adapt_gamma);
        f("adaptivity.tol", c.adapt_tol);
        f("poisson.penalty_scale", c.penalty_scale);
        f("output.dir", c.out_dir);
        f("output.cadence", c.cadence);
        f("output.snapshot_cadence", c.snapshot_cadence);
        f("output.profile_cadence", c.profile_cadence);
        f("threads", c.threads);
    }

    static std::string trim(const std::string& s) {
        const char* ws = " \t\r\n";
        const size_t a = s.find_first_not_of(ws);
        if (a == std::string::npos) return "";
        return s.substr(a, s.find_last_not_of(ws) - a + 1);
    }

    static void parse_into(const std::string&, const std::string& v, std::string& out) { out = v; }
    static void parse_into(const std::string& key, const std::string& v, double& out) {
        size_t used = 0;
        double d = 0.0;
        bool ok = true;
        try {
            d = std::stod(v, &used);
        } catch (...) {
            ok = false;
        }
        if (!ok || used != v.size()) throw std::runtime_error(key + ": not a number: '" + v + "'");
        out = d;
    }
    static void parse_into(const std::string& key, const std::string& v, int& out) {
        size_t used = 0;
        int i = 0;
        bool ok = true;
        try {
            i = std::stoi(v, &used);
        } catch (...) {
            ok = false;
        }
        if (!ok || used != v.size()) throw std::runtime_error(key + ": not an integer: '" + v + "'");
        out = i;
    }
    static void parse_into(const std::string& key, const std::string& v, bool& out) {
        if (v == "on" || v == "true" || v == "1")
            out = true;
        else if (v == "off" || v == "false" || v == "0")
            out = false;
        else
            throw std::runtime_error(key + ": expected on|off, got '" + v + "'");
    }

    static std::string format(const std::string& v) { return v; }
    static std::string format(int v) { return std::to_string(v); }
    static std::string format(bool v) { return v ? "on" : "off"; }
    static std::string format(double v) {
        char buf[32];
        std::snprintf(buf, sizeof(buf), "%.17g", v);
        return buf;
    }
};

// cmd_run's layering (tools/solkin_main.cpp:20-28): preset, then the file,
// then the flag overrides (empty / <= 0: not given); resolved and validated.
inline RunConfig resolve_run_config(const std::string& config_path, const std::string& preset,
                                    const std::string& limiter = "", const std::string& out_dir = "",
                                    int threads = 0) {
    RunConfig cfg;
    if (!preset.empty()) cfg = RunConfig::preset(preset);
    if (!config_path.empty()) cfg.apply_file(config_path);
    if (!limiter.empty()) cfg.limiter = limiter;
    if (!out_dir.empty()) cfg.out_dir = out_dir;
    if (threads > 0) cfg.threads = threads;
    cfg.resolve();
    cfg.validate();
    return cfg;
}

// the device context run() builds for a config: Grid1D::three_block over
// [-L, L] (run.cpp:31), degree k, the SIPG penalty
inline Context make_context(const RunConfig& cfg, int device = 0) {
    return Context(GridBlocks::three_block(-cfg.L, cfg.L, cfg.fine_block_cells, cfg.coarse_block_cells,
                                           cfg.refinement_ratio),
                   cfg.k, cfg.penalty_scale, device);
}

// run(cfg) (run.cpp:60-169): nsteps, cadences and out_dir from the config,
// resolved and validated first (run.cpp:61-63), its echo written to
// <out_dir>/config_resolved.cfg (run.cpp:70-73)
inline sk_run_result run(const Context& ctx, const RunConfig& cfg_in) {
    RunConfig cfg = cfg_in;
    cfg.resolve();
    cfg.validate();
    if (!cfg.out_dir.empty()) {
        const std::string& dir = cfg.out_dir;
        ::mkdir(dir.c_str(), 0755);  // OutputWriter's directory (diagnostics.cpp:118-126)
        std::ofstream out(dir + "/config_resolved.cfg", std::ios::trunc);
        if (!out.good()) throw std::runtime_error("cannot open '" + dir + "/config_resolved.cfg' for writing");
        out << cfg.echo();
    }
    return run(ctx, cfg.to_c(), cfg.nsteps(), cfg.cadence, cfg.snapshot_cadence, cfg.profile_cadence,
               cfg.out_dir);
}
// run(const RunConfig&) (run.hpp) with the context built here
inline sk_run_result run(const RunConfig& cfg, int device = 0) { return run(make_context(cfg, device), cfg); }

// build_shift_matrices (advection.cpp:27-66) from the library's constants
struct ShiftMatrices {
    int p = 0;
    double alpha = 0.0;
    std::vector<double> A, B;  // p x p, row-major
};
inline ShiftMatrices build_shift_matrices(int k, double alpha) {
    ShiftMatrices M;
    M.p = k + 1;
    M.alpha = alpha;
    M.A.assign(static_cast<size_t>(M.p) * M.p, 0.0);
    M.B.assign(static_cast<size_t>(M.p) * M.p, 0.0);
    check(sk_shift_matrices(k, alpha, M.A.data(), M.B.data()));
    return M;
}

// the `solkin matrices --alpha a --order k` table (solkin_main.cpp:43-57)
inline std::string matrices_text(double alpha, int order) {
    const ShiftMatrices M = build_shift_matrices(order, alpha);
    std::string out;
    char buf[64];
    auto table = [&](const char* name, const std::vector<double>& mat) {
        std::snprintf(buf, sizeof(buf), "%s(alpha=%.17g), order %d:\n", name, alpha, order);
        out += buf;
        for (int m = 0; m < M.p; ++m) {
            for (int n = 0; n < M.p; ++n) {
                std::snprintf(buf, sizeof(buf), " % .17e", mat[m * M.p + n]);
                out += buf;
            }
            out += "\n";
        }
    };
    table("A", M.A);
    table("B", M.B);
    return out;
}

}  // namespace solkin_b200
