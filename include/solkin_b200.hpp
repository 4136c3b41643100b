// solkin_b200.hpp -- C++ mirror of the reference solver interface over the C ABI.
//
// Header-only. Keeps the reference's names, argument meaning and exception
// types (core/include/solkin/*.hpp) so a caller of proj/core switches by
// changing the namespace and the field type:
//
//   reference                                   here
//   NodalField (field.hpp:21-80)                solkin_b200::NodalField (device resident)
//   advect_x / advect_v (advection.hpp:83-88)   solkin_b200::advect_x / advect_v
//   apply_post_limiter (limiters.hpp:107-108)   solkin_b200::apply_post_limiter
//   charge_density (poisson.hpp:61)             solkin_b200::charge_density
//   PoissonOperator::solve (poisson.hpp:28)     solkin_b200::Context::poisson_solve
//   check_velocity_shrink / shrink_velocity_domain (adaptivity.hpp:21,33)
//   SimulationState + strang_step (stepper.hpp:44-63), run() loop body (run.cpp:124-131)
//   std::runtime_error / SimulationError (common.hpp:9-20)
#pragma once

#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sk_b200.h"

namespace solkin_b200 {

struct SimulationError : std::runtime_error {
    long step;
    SimulationError(long step_, const std::string& msg) : std::runtime_error(msg), step(step_) {}
};

inline void check(sk_status rc) {
    if (rc == SK_OK) return;
    std::string msg = sk_last_error();
    if (rc == SK_ERR_SIMULATION) throw SimulationError(sk_last_error_step(), msg);
    throw std::runtime_error(msg);
}

enum class BoundaryRule { ZeroInflow = SK_BC_ZERO_INFLOW, Periodic = SK_BC_PERIODIC };
enum class SweepDirection { X = SK_DIR_X, V = SK_DIR_V };
enum class Species { Electron = SK_SPECIES_ELECTRON, Ion = SK_SPECIES_ION };

struct LimiterConfig {
    sk_limiter c{0, 0, 0, 0.5, {0.001, 0.998, 0.001}, {0.45, 0.1, 0.45}, 1e-6};
    // limiters.cpp:14-37
    static LimiterConfig parse(const std::string& mode) {
        LimiterConfig cfg;
        if (mode == "none") return cfg;
        if (mode == "sldg") {
            cfg.c.inline_sldg = 1;
            return cfg;
        }
        auto plus = mode.find('+');
        if (plus == std::string::npos) throw std::runtime_error("unknown limiter mode: " + mode);
        std::string ind = mode.substr(0, plus), mod = mode.substr(plus + 1);
        if (ind == "minmod")
            cfg.c.indicator = 1;
        else if (ind == "meanerr")
            cfg.c.indicator = 2;
        else
            throw std::runtime_error("unknown limiter indicator: " + ind);
        if (mod == "simple")
            cfg.c.modifier = 1;
        else if (mod == "line")
            cfg.c.modifier = 2;
        else
            throw std::runtime_error("unknown limiter modifier: " + mod);
        return cfg;
    }
    bool post_enabled() const { return c.indicator != 0; }
};

struct SpeciesParams {  // advection.hpp:64-70
    double charge_sign = -1.0;
    double sqrt_mu = 1.0;
    static SpeciesParams electron() { return {-1.0, 1.0}; }
    static SpeciesParams ion(double mu) {
        if (!(mu > 0)) throw std::runtime_error("SpeciesParams::ion: mass ratio must be positive");
        return {+1.0, std::sqrt(mu)};
    }
};

struct SweepOptions {  // advection.hpp:72-79
    BoundaryRule bc = BoundaryRule::ZeroInflow;
    LimiterConfig limiter{};
    int max_ghost = -1;
    long step_index = 0;
};

struct VAdjustPolicy {  // adaptivity.hpp:13-19
    double p = 0.05, gamma = 0.05, tol = 1e-14;
    sk_vadjust c() const { return {p, gamma, tol}; }
};

struct GridBlocks {
    std::vector<double> left, dx;
    std::vector<int> cells;
    // Grid1D::three_block (grid.cpp:36-46)
    static GridBlocks three_block(double l, double r, int nf, int nc, int m) {
        GridBlocks g;
        g.left.resize(3);
        g.dx.resize(3);
        g.cells.resize(3);
        check(sk_grid_three_block(l, r, nf, nc, m, g.left.data(), g.cells.data(), g.dx.data()));
        return g;
    }
    static GridBlocks uniform(double l, double r, int cells) {
        if (!(r > l && cells >= 1)) throw std::runtime_error("Grid1D::uniform: invalid extent or cell count");
        return GridBlocks{{l}, {(r - l) / cells}, {cells}};
    }
};

// One GPU: x grid, degree k, Poisson operator (assembled + reduced once).
class Context {
  public:
    Context(const GridBlocks& x, int k, double penalty_scale = 10.0, int device = 0) {
        sk_ctx* h = nullptr;
        check(sk_ctx_create(device, k, (int)x.cells.size(), x.left.data(), x.cells.data(),
                            x.dx.data(), penalty_scale, &h));
        h_.reset(h);
    }
    sk_ctx* get() const { return h_.get(); }
    void synchronize() const { check(sk_ctx_synchronize(h_.get())); }
    sk_stats stats() const {
        sk_stats s;
        check(sk_stats_get(h_.get(), &s));
        return s;
    }
    // PoissonOperator::solve (poisson.cpp:166-192) on device buffers
    void poisson_solve(const double* rho_dev, double* E_dev, double* phi_dev = nullptr) const {
        check(sk_poisson_solve(h_.get(), rho_dev, E_dev, phi_dev));
    }

  private:
    struct Del {
        void operator()(sk_ctx* c) const { sk_ctx_destroy(c); }
    };
    std::unique_ptr<sk_ctx, Del> h_;
};

// NodalField on the device, reference layout ((vc*p+vn)*nx+xc)*p+xn.
class NodalField {
  public:
    NodalField(const Context& ctx, Species s, double v_left, double v_right, int v_cells) {
        sk_field* f = nullptr;
        check(sk_field_create(ctx.get(), (int)s, v_left, v_right, v_cells, &f));
        h_.reset(f);
        owner_ = true;
    }
    explicit NodalField(sk_field* borrowed) : raw_(borrowed) {}
    sk_field* get() const { return owner_ ? h_.get() : raw_; }
    size_t size() const { return sk_field_size(get()); }
    double* device_data() const { return sk_field_data_dev(get()); }
    void upload(const std::vector<double>& host) const { check(sk_field_upload(get(), host.data(), host.size())); }
    std::vector<double> download() const {
        std::vector<double> out(size());
        check(sk_field_download(get(), out.data(), out.size()));
        return out;
    }
    double vmax() const {
        double l, d;
        int c;
        check(sk_field_v_grid(get(), &l, &d, &c));
        return l + c * d;  // Grid1D::right (grid.cpp:48-51)
    }
    void fill_blob(double sigma) const { check(sk_field_fill_blob(get(), sigma)); }
    double mass() const { return moments()[0]; }
    double l2_norm() const { return moments()[1]; }
    std::vector<double> moments() const {
        std::vector<double> m(4);
        check(sk_field_moments(get(), m.data()));
        return m;
    }

  private:
    struct Del {
        void operator()(sk_field* f) const { sk_field_destroy(f); }
    };
    std::unique_ptr<sk_field, Del> h_;
    sk_field* raw_ = nullptr;
    bool owner_ = false;
};

inline void advect_x(NodalField& f, double tau, const SpeciesParams& sp, const SweepOptions& opt) {
    check(sk_advect_x(f.get(), tau, sp.sqrt_mu, (int)opt.bc, &opt.limiter.c, opt.max_ghost,
                      opt.step_index));
}
inline void advect_v(NodalField& f, double tau, const double* E_nodes_dev, const SpeciesParams& sp,
                     const SweepOptions& opt) {
    check(sk_advect_v(f.get(), tau, E_nodes_dev, sp.charge_sign, sp.sqrt_mu, (int)opt.bc,
                      &opt.limiter.c));
}
inline void apply_post_limiter(NodalField& f, SweepDirection dir, const LimiterConfig& cfg,
                               BoundaryRule bc) {
    check(sk_post_limit(f.get(), (int)dir, &cfg.c, (int)bc));
}
inline void charge_density(const NodalField& fe, const NodalField& fi, double* rho_dev) {
    check(sk_charge_density(fe.get(), fi.get(), rho_dev));
}
inline bool check_velocity_shrink(const NodalField& f, const VAdjustPolicy& p) {
    sk_vadjust c = p.c();
    int out = 0;
    check(sk_check_velocity_shrink(f.get(), &c, &out));
    return out != 0;
}
inline sk_shrink_result shrink_velocity_domain(NodalField& f, const VAdjustPolicy& p) {
    sk_vadjust c = p.c();
    sk_shrink_result r;
    check(sk_shrink_velocity_domain(f.get(), &c, &r));
    return r;
}

// SimulationState (stepper.hpp:44-54) built by build_initial_state (run.cpp:26-58)
class SimulationState {
  public:
    SimulationState(const Context& ctx, const sk_run_config& cfg) {
        sk_state* s = nullptr;
        check(sk_state_create(ctx.get(), &cfg, &s));
        h_.reset(s);
    }
    sk_state* get() const { return h_.get(); }
    NodalField f_e() const { return NodalField(sk_state_field(h_.get(), 0)); }
    NodalField f_i() const { return NodalField(sk_state_field(h_.get(), 1)); }
    const double* E_dev() const { return sk_state_E_dev(h_.get()); }
    long step() const {
        long s;
        check(sk_state_step_index(h_.get(), &s));
        return s;
    }

  private:
    struct Del {
        void operator()(sk_state* s) const { sk_state_destroy(s); }
    };
    std::unique_ptr<sk_state, Del> h_;
};

// strang_step (stepper.cpp:44-103) and the run() loop body (run.cpp:124-131)
inline void strang_step(SimulationState& s) { check(sk_strang_step(s.get())); }
inline void run_step(SimulationState& s) { check(sk_run_step(s.get())); }

// diagnostics.cpp: WallFlux (diagnostics.hpp:17-21), sample_fluxes, summarize
enum class WallSide { Left = 0, Right = 1 };
struct WallFlux {
    double outflow = 0.0, naive = 0.0;
};
inline WallFlux wall_flux(SimulationState& s, Species sp, WallSide side) {
    WallFlux w;
    check(sk_state_wall_flux(s.get(), static_cast<int>(sp), static_cast<int>(side), &w.outflow, &w.naive));
    return w;
}
inline sk_flux_sample sample_fluxes(SimulationState& s) {
    sk_flux_sample out;
    check(sk_state_sample_fluxes(s.get(), &out));
    return out;
}
inline sk_summary summarize(SimulationState& s) {
    sk_summary out;
    check(sk_state_summarize(s.get(), &out));
    return out;
}
// OutputWriter::write_snapshot / write_profiles (diagnostics.cpp:161-220)
inline void write_snapshot(SimulationState& s, const std::string& dir) {
    check(sk_state_write_snapshot(s.get(), dir.c_str()));
}
inline void write_profiles(SimulationState& s, const std::string& dir) {
    check(sk_state_write_profiles(s.get(), dir.c_str()));
}
// run() (run.cpp:60-169); out_dir empty: no files. SimulationError ends the
// run with exit_code 1 (the reference's contract), other failures throw.
inline sk_run_result run(const Context& ctx, const sk_run_config& cfg, long nsteps, int cadence = 10,
                         int snapshot_cadence = 0, int profile_cadence = 0, const std::string& out_dir = "out") {
    sk_run_result r;
    check(sk_run(ctx.get(), &cfg, nsteps, cadence, snapshot_cadence, profile_cadence,
                 out_dir.empty() ? nullptr : out_dir.c_str(), &r));
    return r;
}

}  // namespace solkin_b200
