// ref_driver.cpp -- CPU ORACLE harness (test / baseline infrastructure only).
//
// Compiled together with the UNMODIFIED reference sources under
// /root/reference/proj/core/src into oracle/_ref/libsolkin_ref.so by
// oracle/Makefile (never copied into this repo). Exposes a flat extern "C"
// surface so tests and bench.py's reference arm can drive the reference's own
// public API through ctypes:
//   * ref_state_* replicate the run() loop body (core/src/run.cpp:124-131):
//     ghost width -> strang_step -> shrink checks with the 10-step cooldown;
//   * ref_* unit entry points wrap advect_x/advect_v/apply_post_limiter/
//     charge_density/check_velocity_shrink/shrink_velocity_domain and the
//     basis/limiter helpers for golden-vector generation.
// LAPACK dpbtrf_/dpbtrs_ are provided by oracle/lapack_band.c (restated
// reference-LAPACK algorithm; the image has no LAPACK development package).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>

#include "sk_oracle.h"
#include "solkin/adaptivity.hpp"
#include "solkin/advection.hpp"
#include "solkin/basis.hpp"
#include "solkin/check.hpp"
#include "solkin/common.hpp"
#include "solkin/config.hpp"
#include "solkin/diagnostics.hpp"
#include "solkin/limiters.hpp"
#include "solkin/poisson.hpp"
#include "solkin/run.hpp"
#include "solkin/stepper.hpp"

using namespace solkin;

extern "C" {
void dpbtrf_(const char* uplo, const int* n, const int* kd, double* ab, const int* ldab, int* info) {
    if (uplo[0] != 'L') {
        *info = -1;
        return;
    }
    *info = sko_dpbtrf_lower(*n, *kd, ab, *ldab);
}
void dpbtrs_(const char* uplo, const int* n, const int* kd, const int* nrhs, const double* ab,
             const int* ldab, double* b, const int* ldb, int* info) {
    if (uplo[0] != 'L') {
        *info = -1;
        return;
    }
    for (int r = 0; r < *nrhs; ++r) sko_dpbtrs_lower(*n, *kd, ab, *ldab, b + (long)r * *ldb);
    *info = 0;
}
}

namespace {

thread_local std::string g_error;

struct RefHandle {
    RunConfig cfg;
    SimulationState state;
    StepOptions opt;
    SweepStats stats;
    StepTimers timers;
    VAdjustPolicy policy;
    long last_shrink_e = -10;
    long last_shrink_i = -10;
    int shrinks_e = 0, shrinks_i = 0;
};

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const SimulationError& e) {
        g_error = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_error = e.what();
        return 1;
    }
}

NodalField& field_of(RefHandle* h, int species) {
    return species == 0 ? h->state.f_e : h->state.f_i;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

void* ref_state_create(double L, double dt, int k, double mu, double sigma, double vmax_e,
                       double vmax_i, int nf, int nc, int m, int nv, const char* limiter,
                       double limiter_threshold, int v_adjust, double adapt_p, double adapt_gamma,
                       double adapt_tol, double penalty_scale, int threads) {
    auto* h = new RefHandle;
    int rc = guarded([&] {
        RunConfig& c = h->cfg;
        c.L = L;
        c.dt = dt;
        c.k = k;
        c.mu = mu;
        c.sigma = sigma;
        c.vmax_e = vmax_e;
        c.vmax_i = vmax_i;
        c.fine_block_cells = nf;
        c.coarse_block_cells = nc;
        c.refinement_ratio = m;
        c.v_cells = nv;
        c.limiter = limiter;
        c.limiter_threshold = limiter_threshold;
        c.v_adjust = v_adjust != 0;
        c.adapt_p = adapt_p;
        c.adapt_gamma = adapt_gamma;
        c.adapt_tol = adapt_tol;
        c.penalty_scale = penalty_scale;
        c.threads = threads;
        c.resolve();
        c.validate();
        h->state = build_initial_state(c);
        h->opt.limiter = LimiterConfig::parse(c.limiter);
        h->opt.limiter.threshold = c.limiter_threshold;
        h->opt.threads = c.threads;
        h->opt.stats = &h->stats;
        h->opt.timers = &h->timers;
        h->policy = VAdjustPolicy{c.adapt_p, c.adapt_gamma, c.adapt_tol};
    });
    if (rc) {
        delete h;
        return nullptr;
    }
    return h;
}

void ref_state_free(void* hp) { delete static_cast<RefHandle*>(hp); }

// diagnostics of the live state (diagnostics.cpp)
int ref_state_wall_flux(void* hp, int species, int side, double* out2) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        WallFlux w = wall_flux(field_of(h, species), side == 1 ? WallSide::Right : WallSide::Left);
        out2[0] = w.outflow;
        out2[1] = w.naive;
    });
}
double ref_state_time(void* hp) { return static_cast<RefHandle*>(hp)->state.time; }
int ref_state_write_snapshot(void* hp, const char* dir) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        OutputWriter w(dir);
        w.write_snapshot(h->state.step, h->state.time, h->state.f_e, h->state.f_i);
    });
}
// run() with files (run.cpp:60-169) for this handle's configuration
int ref_run_files(void* hp, double t_final, int cadence, int snapshot_cadence, int profile_cadence,
                  const char* dir) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        RunConfig c = h->cfg;
        c.t_final = t_final;
        c.cadence = cadence;
        c.snapshot_cadence = snapshot_cadence;
        c.profile_cadence = profile_cadence;
        c.out_dir = dir;
        RunResult r = run(c, true);
        if (r.exit_code) throw std::runtime_error(r.error);
    });
}

// scenario "injection" (config.hpp:11,18; run.cpp:47-53): rebuild the state
int ref_state_set_injection(void* hp, double t0) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        h->cfg.scenario = "injection";
        h->cfg.t0 = t0;
        h->cfg.validate();
        h->state = build_initial_state(h->cfg);
        h->last_shrink_e = h->last_shrink_i = -10;
        h->shrinks_e = h->shrinks_i = 0;
    });
}

// run.cpp:124-131 loop body, including the shrink cadence of run.cpp:98-114.
int ref_state_step(void* hp) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        auto& st = h->state;
        double sqrt_mu_min = std::min(st.electron.sqrt_mu, st.ion.sqrt_mu);
        double vmax_now = std::max(st.f_e.v().right(), st.f_i.v().right());
        double dx_fine = st.f_e.x().blocks()[0].dx;
        h->opt.max_ghost =
            BlockLayout::required_ghost_width(vmax_now, h->cfg.dt, sqrt_mu_min, dx_fine);
        strang_step(st, h->cfg.dt, h->opt);
        auto check = [&](NodalField& f, long& last, int& count) {
            if (!h->cfg.v_adjust) return;
            if (st.step - last < 10) return;
            if (!check_velocity_shrink(f, h->policy)) return;
            shrink_velocity_domain(f, h->policy);
            last = st.step;
            ++count;
        };
        check(st.f_e, h->last_shrink_e, h->shrinks_e);
        check(st.f_i, h->last_shrink_i, h->shrinks_i);
    });
}

// Timed loop for the bench reference arm: returns wall seconds for n steps.
double ref_state_run(void* hp, int n) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i)
        if (ref_state_step(hp)) return -1.0;
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

long ref_state_field_size(void* hp, int species) {
    return (long)field_of(static_cast<RefHandle*>(hp), species).size();
}
void ref_state_get_field(void* hp, int species, double* out) {
    auto& f = field_of(static_cast<RefHandle*>(hp), species);
    std::memcpy(out, f.raw().data(), f.size() * sizeof(double));
}
void ref_state_set_field(void* hp, int species, const double* in) {
    auto& f = field_of(static_cast<RefHandle*>(hp), species);
    std::memcpy(f.raw().data(), in, f.size() * sizeof(double));
}
double ref_state_vmax(void* hp, int species) {
    return field_of(static_cast<RefHandle*>(hp), species).v().right();
}
long ref_state_step_index(void* hp) { return static_cast<RefHandle*>(hp)->state.step; }
int ref_state_shrinks(void* hp, int species) {
    auto* h = static_cast<RefHandle*>(hp);
    return species == 0 ? h->shrinks_e : h->shrinks_i;
}
long ref_state_last_shrink(void* hp, int species) {
    auto* h = static_cast<RefHandle*>(hp);
    return species == 0 ? h->last_shrink_e : h->last_shrink_i;
}
void ref_state_get_E(void* hp, double* out) {
    auto& E = static_cast<RefHandle*>(hp)->state.field.E;
    std::memcpy(out, E.data(), E.size() * sizeof(double));
}
void ref_state_get_phi(void* hp, double* out) {
    auto& phi = static_cast<RefHandle*>(hp)->state.field.phi;
    std::memcpy(out, phi.data(), phi.size() * sizeof(double));
}
void ref_state_get_stats(void* hp, long* out) {
    auto& s = static_cast<RefHandle*>(hp)->stats;
    out[0] = s.outputs;
    out[1] = s.inline_troubled;
    out[2] = s.inline_clamped;
    out[3] = s.inline_mean_outside;
    out[4] = s.post_checked;
    out[5] = s.post_troubled;
}
void ref_state_get_timers(void* hp, double* out) {
    auto& t = static_cast<RefHandle*>(hp)->timers;
    out[0] = t.source;
    out[1] = t.advect_x;
    out[2] = t.advect_v;
    out[3] = t.poisson;
    out[4] = t.post_limiter;
}
// diagnostics: mass, l2 per species + electric energy (field.cpp:52-88, diagnostics.cpp:71-83)
void ref_state_summary(void* hp, double* out) {
    auto* h = static_cast<RefHandle*>(hp);
    auto s = summarize(h->state.f_e, h->state.f_i, h->state.field);
    out[0] = s.mass_e;
    out[1] = s.mass_i;
    out[2] = s.l2_e;
    out[3] = s.l2_i;
    out[4] = s.e_energy;
    out[5] = s.vmax_e;
    out[6] = s.vmax_i;
}

// ---- unit-level operators on a state's fields ----
int ref_state_advect_x(void* hp, int species, double tau, int limited, int max_ghost) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        SweepOptions so;
        so.limiter = h->opt.limiter;
        if (!limited) so.limiter = LimiterConfig{};
        so.threads = h->opt.threads;
        so.max_ghost = max_ghost;
        so.stats = &h->stats;
        so.step_index = h->state.step;
        advect_x(field_of(h, species), tau, species == 0 ? h->state.electron : h->state.ion, so);
    });
}
int ref_state_advect_v(void* hp, int species, double tau, const double* E, int limited) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        SweepOptions so;
        so.limiter = h->opt.limiter;
        if (!limited) so.limiter = LimiterConfig{};
        so.threads = h->opt.threads;
        so.stats = &h->stats;
        auto& f = field_of(h, species);
        std::span<const double> Es(E, size_t(f.nx()) * f.nodes_per_cell());
        advect_v(f, tau, Es, species == 0 ? h->state.electron : h->state.ion, so);
    });
}
int ref_state_post_limit(void* hp, int species, int dir, const char* mode) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        auto cfg = LimiterConfig::parse(mode);
        apply_post_limiter(field_of(h, species), dir == 0 ? SweepDirection::X : SweepDirection::V,
                           cfg, BoundaryRule::ZeroInflow, h->opt.threads, &h->stats);
    });
}
int ref_state_charge_density(void* hp, double* rho) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        auto r = charge_density(h->state.f_e, h->state.f_i);
        std::memcpy(rho, r.data(), r.size() * sizeof(double));
    });
}
int ref_state_poisson_solve(void* hp, const double* rho, double* E, double* phi) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        size_t n = size_t(h->state.f_e.nx()) * h->state.f_e.nodes_per_cell();
        auto fp = h->state.poisson->solve(std::span<const double>(rho, n));
        std::memcpy(E, fp.E.data(), fp.E.size() * sizeof(double));
        if (phi) std::memcpy(phi, fp.phi.data(), fp.phi.size() * sizeof(double));
    });
}
int ref_state_check_shrink(void* hp, int species) {
    auto* h = static_cast<RefHandle*>(hp);
    int out = -1;
    int rc = guarded([&] { out = check_velocity_shrink(field_of(h, species), h->policy) ? 1 : 0; });
    return rc ? -1 : out;
}
int ref_state_shrink(void* hp, int species, double* result) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        auto r = shrink_velocity_domain(field_of(h, species), h->policy);
        result[0] = r.vmax_before;
        result[1] = r.vmax_after;
        result[2] = r.mass_before;
        result[3] = r.mass_after;
    });
}

// ---- basis / limiter helpers ----
int ref_gauss_legendre(int k, double* nodes, double* weights) {
    return guarded([&] {
        auto [n, w] = gauss_legendre(k);
        std::memcpy(nodes, n.data(), n.size() * sizeof(double));
        std::memcpy(weights, w.data(), w.size() * sizeof(double));
    });
}
void ref_decompose_shift(double speed, double dt, double dx, int* istar, double* alpha) {
    auto s = decompose_shift(speed, dt, dx);
    *istar = s.istar;
    *alpha = s.alpha;
}
int ref_shift_matrices(int k, double alpha, double* A, double* B) {
    return guarded([&] {
        auto M = build_shift_matrices(ReferenceBasis::get(k), alpha);
        std::memcpy(A, M.A.data(), M.A.size() * sizeof(double));
        std::memcpy(B, M.B.data(), M.B.size() * sizeof(double));
    });
}
double ref_max_on(int k, const double* u, double a, double b) {
    auto& bs = ReferenceBasis::get(k);
    return bs.max_on(std::span<const double>(u, k + 1), a, b);
}
double ref_min_on(int k, const double* u, double a, double b) {
    auto& bs = ReferenceBasis::get(k);
    return bs.min_on(std::span<const double>(u, k + 1), a, b);
}
// flags: bit0 troubled, bit1 clamped, bit2 mean_outside
int ref_inline_apply(int k, double alpha, double thr, const double* ul, const double* ur,
                     double* up) {
    auto& bs = ReferenceBasis::get(k);
    InlineLimiter lim(bs, alpha, thr);
    const size_t p = k + 1;
    auto r = lim.apply({ul, p}, {ur, p}, {up, p});
    return (r.troubled ? 1 : 0) | (r.clamped ? 2 : 0) | (r.mean_outside ? 4 : 0);
}
int ref_post_indicator(int k, int kind, double thr, const double* um, const double* u0,
                       const double* up) {
    auto& bs = ReferenceBasis::get(k);
    const size_t p = k + 1;
    StencilTriplet t{{um, p}, {u0, p}, {up, p}};
    return kind == 1 ? indicator_minmod(bs, t) : indicator_meanerr(bs, t, thr);
}
void ref_post_modify(int k, int kind, const double* um, const double* u0, const double* up,
                     double* out) {
    auto& bs = ReferenceBasis::get(k);
    const size_t p = k + 1;
    StencilTriplet t{{um, p}, {u0, p}, {up, p}};
    LimiterConfig cfg;
    if (kind == 1)
        modify_simple_weno(bs, t, cfg, {out, p});
    else
        modify_line_weno(bs, t, cfg, {out, p});
}
double ref_smoothness_beta(int k, const double* u) {
    return smoothness_beta(ReferenceBasis::get(k), std::span<const double>(u, k + 1));
}
void ref_fine_to_coarse(int k, const double* fine, int m, double* coarse) {
    const size_t p = k + 1;
    fine_to_coarse(ReferenceBasis::get(k), {fine, m * p}, m, {coarse, p});
}
void ref_coarse_to_fine(int k, const double* coarse, int m, double* fine) {
    const size_t p = k + 1;
    coarse_to_fine(ReferenceBasis::get(k), {coarse, p}, m, {fine, m * p});
}
// check.cpp:29-151 -- the reference's built-in invariant suite; returns failures
int ref_self_checks() {
    std::ostringstream out;
    int failures = run_self_checks(out);
    g_error = out.str();
    return failures;
}

// config.cpp:58-218 -- RunConfig as cmd_run layers it (solkin_main.cpp:20-28):
// preset (empty: defaults) -> file (empty: none) -> kv overrides ("key\tvalue"
// lines, applied verbatim through apply_kv) -> resolve() when asked. Writes
// echo() and violations() (one per line); 1 + ref_last_error() on a throw.
int ref_config_eval(const char* preset, const char* file, const char* kv, int resolve, char* echo,
                    long echo_cap, char* viol, long viol_cap, long* nsteps) {
    return guarded([&] {
        RunConfig c;
        if (preset && *preset) c = RunConfig::preset(preset);
        if (file && *file) c.apply_file(file);
        std::istringstream lines(kv ? kv : "");
        std::string line;
        while (std::getline(lines, line)) {
            if (line.empty()) continue;
            const size_t tab = line.find('\t');
            c.apply_kv(line.substr(0, tab), tab == std::string::npos ? "" : line.substr(tab + 1));
        }
        if (resolve) c.resolve();
        std::string v;
        for (const auto& s : c.violations()) v += s + "\n";
        std::snprintf(echo, echo_cap, "%s", c.echo().c_str());
        std::snprintf(viol, viol_cap, "%s", v.c_str());
        *nsteps = c.nsteps();
    });
}
// tools/solkin_main.cpp:43-57 -- the `solkin matrices` table, from the reference basis
int ref_matrices_text(double alpha, int order, char* out, long cap) {
    return guarded([&] {
        const auto& basis = ReferenceBasis::get(order);
        auto M = build_shift_matrices(basis, alpha);
        std::string s;
        char buf[64];
        auto table = [&](const char* name, const std::vector<double>& mat) {
            std::snprintf(buf, sizeof(buf), "%s(alpha=%.17g), order %d:\n", name, alpha, order);
            s += buf;
            for (int m = 0; m < M.p; ++m) {
                for (int n = 0; n < M.p; ++n) {
                    std::snprintf(buf, sizeof(buf), " % .17e", mat[m * M.p + n]);
                    s += buf;
                }
                s += "\n";
            }
        };
        table("A", M.A);
        table("B", M.B);
        std::snprintf(out, cap, "%s", s.c_str());
    });
}

}  // extern "C"
