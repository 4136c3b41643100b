// C++ drop-in check (test infrastructure): drives the B200 step through the
// reference-shaped C++ API (include/solkin_b200.hpp) and compares it with the
// C oracle (oracle/sk_oracle.h) -- the way a proj/core caller would switch.
// Exit code 0 on parity; prints max relative differences.
#include <cmath>
#include <cstdio>
#include <vector>

#include "../../include/solkin_b200.hpp"
#include "../../oracle/sk_oracle.h"

namespace sb = solkin_b200;

static double rel(const std::vector<double>& a, const double* b, size_t n) {
    double d = 0, m = 0;
    for (size_t i = 0; i < n; ++i) {
        d = std::fmax(d, std::fabs(a[i] - b[i]));
        m = std::fmax(m, std::fabs(b[i]));
    }
    return m > 0 ? d / m : d;
}

int main() {
    const double L = 200.0, dt = 0.1, mu = 1836.0;
    const int k = 3, nf = 8, nc = 16, m = 2, nv = 24;
    sk_run_config cfg{};
    cfg.L = L;
    cfg.dt = dt;
    cfg.mu = mu;
    cfg.sigma = -1.0;
    cfg.vmax_e = cfg.vmax_i = 12.0;
    cfg.k = k;
    cfg.fine_block_cells = nf;
    cfg.coarse_block_cells = nc;
    cfg.refinement_ratio = m;
    cfg.v_cells = nv;
    cfg.limiter = sb::LimiterConfig::parse("sldg").c;
    cfg.v_adjust = 1;
    cfg.policy = {0.05, 0.05, 1e-14};
    cfg.penalty_scale = 10.0;

    sb::Context ctx(sb::GridBlocks::three_block(-L, L, nf, nc, m), k);
    sb::SimulationState st(ctx, cfg);
    sko_state ora;
    if (sko_state_init(&ora, L, dt, k, mu, -1.0, 12.0, 12.0, nf, nc, m, nv, "sldg", 0.5, 1, 0.05,
                       0.05, 1e-14, 10.0)) {
        std::printf("oracle init failed: %s\n", sko_last_error());
        return 2;
    }
    double worst = 0;
    for (int s = 0; s < 12; ++s) {
        sb::run_step(st);
        if (sko_run_step(&ora)) return 3;
    }
    auto fe = st.f_e().download(), fi = st.f_i().download();
    const size_t n = fe.size();
    worst = std::fmax(rel(fe, ora.fe.data, n), rel(fi, ora.fi.data, n));
    bool vmax_ok = st.f_e().vmax() == sko_grid_right(&ora.fe.v) &&
                   st.f_i().vmax() == sko_grid_right(&ora.fi.v);
    std::printf("steps=%ld rel=%.3e vmax_equal=%d\n", st.step(), worst, (int)vmax_ok);
    // the reference's exception mapping: periodic x sweep on a 3-block grid
    try {
        sb::SweepOptions o;
        o.bc = sb::BoundaryRule::Periodic;
        auto f = st.f_e();
        sb::advect_x(f, 0.05, sb::SpeciesParams::electron(), o);
        std::printf("missing runtime_error\n");
        return 4;
    } catch (const std::runtime_error&) {
    }
    sko_state_free(&ora);
    return (worst <= 1e-12 && vmax_ok) ? 0 : 1;
}
