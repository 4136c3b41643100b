/*
 * sk_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference sLdG time step
 * (/root/reference/proj/core, arXiv 2408.11235), written to reproduce the
 * reference's floating-point operation order so that its results can be
 * compared bit for bit against the reference itself (oracle/_ref) and against
 * the CUDA product path built with -fmad=false.
 *
 * ONLY tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library, and only as a checker or a timed CPU baseline.
 * The product path (paper_2408_11235_b200) never links or calls it.
 *
 * Parity pin: tests/test_oracle_pin.py checks every function here against the
 * compiled reference (oracle/_ref/libsolkin_ref.so) and the committed golden
 * vectors in tests/golden/.
 */
#ifndef SK_ORACLE_H
#define SK_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

#define SKO_MAXP 8      /* k <= 6  ->  p = k+1 <= 7 (poisson uses k+2 <= 8) */
#define SKO_MAXB 8      /* x-grid blocks */

/* status codes (mirror solkin/common.hpp:9-20) */
#define SKO_OK 0
#define SKO_ERR_RUNTIME 1     /* std::runtime_error via require()        */
#define SKO_ERR_SIMULATION 2  /* solkin::SimulationError                  */
const char* sko_last_error(void);
long sko_last_error_step(void);

/* ---- basis (basis.cpp) ---- */
typedef struct {
    int k, p;
    double nodes[SKO_MAXP + 1], weights[SKO_MAXP + 1], bary[SKO_MAXP + 1];
    double diff[(SKO_MAXP + 1) * (SKO_MAXP + 1)];
    double mono[(SKO_MAXP + 1) * (SKO_MAXP + 1)];
} sko_basis;

int sko_gauss_legendre(int k, double* nodes, double* weights);
int sko_basis_init(sko_basis* b, int k);
double sko_lagrange(const sko_basis* b, int n, double xi);
double sko_lagrange_derivative(const sko_basis* b, int n, double xi);
double sko_evaluate(const sko_basis* b, const double* u, double xi);
double sko_mean(const sko_basis* b, const double* u);
double sko_integrate(const sko_basis* b, const double* u, double a, double bb);
void sko_interval_moments(const sko_basis* b, double a, double bb, double* m);
void sko_to_monomial(const sko_basis* b, const double* u, double* c);
double sko_max_on(const sko_basis* b, const double* u, double a, double bb);
double sko_min_on(const sko_basis* b, const double* u, double a, double bb);

/* ---- shift (advection.cpp:14-66) ---- */
void sko_decompose_shift(double speed, double dt, double dx, int* istar, double* alpha);
int sko_shift_matrices(const sko_basis* b, double alpha, double* A, double* B);

/* ---- stats (advection.hpp:37-53) ---- */
typedef struct {
    long outputs, inline_troubled, inline_clamped, inline_mean_outside, post_checked, post_troubled;
} sko_stats;

/* ---- limiter config (limiters.hpp:19-34) ---- */
#define SKO_IND_NONE 0
#define SKO_IND_MINMOD 1
#define SKO_IND_MEANERR 2
#define SKO_MOD_NONE 0
#define SKO_MOD_SIMPLE 1
#define SKO_MOD_LINE 2
typedef struct {
    int indicator, modifier, inline_sldg;
    double threshold;
    double gamma_simple[3], gamma_line[3], epsilon;
} sko_limiter;
int sko_limiter_parse(const char* mode, sko_limiter* out);

/* ---- inline sLdG limiter (limiters.cpp:167-222) ---- */
typedef struct {
    double alpha, threshold;
    double ext_l[SKO_MAXP], ext_r[SKO_MAXP];
} sko_inline;
void sko_inline_init(sko_inline* L, const sko_basis* b, double alpha, double threshold);
int sko_inline_indicator(const sko_inline* L, const sko_basis* b, const double* ul,
                         const double* ur, const double* up);
/* returns flags: bit0 troubled, bit1 clamped, bit2 mean_outside */
int sko_inline_clamp(const sko_inline* L, const sko_basis* b, const double* ul, const double* ur,
                     double* up);
int sko_inline_apply(const sko_inline* L, const sko_basis* b, const double* ul, const double* ur,
                     double* up);

/* ---- post limiters (limiters.cpp:47-165) ---- */
double sko_minmod(double a, double b, double c);
int sko_indicator_minmod(const sko_basis* b, const double* um, const double* u0, const double* up);
int sko_indicator_meanerr(const sko_basis* b, const double* um, const double* u0, const double* up,
                          double threshold);
double sko_smoothness_beta(const sko_basis* b, const double* u);
void sko_modify_simple_weno(const sko_basis* b, const double* um, const double* u0,
                            const double* up, const sko_limiter* cfg, double* out);
void sko_modify_line_weno(const sko_basis* b, const double* um, const double* u0, const double* up,
                          const sko_limiter* cfg, double* out);

/* ---- grid (grid.cpp) ---- */
typedef struct {
    int nblocks;
    double left[SKO_MAXB];
    int cells[SKO_MAXB];
    double dx[SKO_MAXB];
    int start[SKO_MAXB + 1];
    int ncells;
} sko_grid;
int sko_grid_init(sko_grid* g, int nblocks, const double* left, const int* cells, const double* dx);
int sko_grid_uniform(sko_grid* g, double left, double right, int cells);
int sko_grid_three_block(sko_grid* g, double left, double right, int nf, int nc, int m);
double sko_grid_right(const sko_grid* g);
int sko_grid_block_of(const sko_grid* g, int cell);
double sko_grid_cell_left(const sko_grid* g, int cell);
double sko_grid_cell_width(const sko_grid* g, int cell);

/* ---- field (field.hpp/.cpp); data layout ((vc*p+vn)*nx+xc)*p+xn ---- */
typedef struct {
    int species; /* 0 electron, 1 ion */
    int k;
    sko_grid x, v;
    double* data; /* caller-owned, nx*nv*p*p doubles */
} sko_field;
double sko_x_node(const sko_field* f, int xc, int xn);
double sko_v_node(const sko_field* f, int vc, int vn);
double sko_mass(const sko_field* f);
double sko_l2_norm(const sko_field* f);
double sko_momentum(const sko_field* f);       /* harness: int v f, mass() loop order */
double sko_kinetic_energy(const sko_field* f); /* harness: int v^2/2 f              */
int sko_all_finite(const sko_field* f);

/* ---- sweeps (advection.cpp:68-238) ---- */
#define SKO_BC_ZERO 0
#define SKO_BC_PERIODIC 1
int sko_advect_line(const sko_basis* b, const double* A, const double* B, int istar, int bc,
                    const double* in, int gl, int n, int gr, double* out, const sko_inline* lim,
                    sko_stats* stats);
int sko_advect_x(sko_field* f, double tau, double sqrt_mu, const sko_limiter* lim, int bc,
                 int max_ghost, long step_index, sko_stats* stats);
int sko_advect_v(sko_field* f, double tau, const double* E, double charge_sign, double sqrt_mu,
                 const sko_limiter* lim, int bc, sko_stats* stats);
/* v sweep of a v-shard: lines hold gl+n+gr cells (halo included), out n cells */
int sko_advect_v_lines(const sko_basis* b, int nlines, int line_stride, const double* in, int gl,
                       int n, int gr, double* out, const double* E, double charge_sign,
                       double sqrt_mu, double tau, double dv, const sko_limiter* lim,
                       sko_stats* stats);
int sko_post_limiter(sko_field* f, int dir, const sko_limiter* cfg, int bc, sko_stats* stats);
/* one x line of advect_x for a given speed (multi-block ghosts included) */
int sko_advect_x_line(int k, int nblocks, const double* left, const int* cells, const double* dx,
                      double speed, double tau, int inline_sldg, double threshold, int max_ghost,
                      const double* line, double* out);

/* ---- adaptivity (adaptivity.cpp) ---- */
void sko_fine_to_coarse(const sko_basis* b, const double* fine, int m, double* coarse);
void sko_coarse_to_fine(const sko_basis* b, const double* coarse, int m, double* fine);
int sko_required_ghost_width(double vmax, double dt, double sqrt_mu_min, double dx_local);
int sko_exchange_block_ghosts(const sko_basis* b, const sko_grid* g, int block, const double* line,
                              int gl, int gr, double* ext);
int sko_check_velocity_shrink(const sko_field* f, double p, double gamma, double tol);
/* result: vmax_before, vmax_after, mass_before, mass_after */
int sko_shrink_velocity_domain(sko_field* f, double p, double gamma, double tol, double* result);

/* ---- poisson (poisson.cpp) ---- */
typedef void (*sko_dpbtrf_fn)(const char*, const int*, const int*, double*, const int*, int*);
typedef void (*sko_dpbtrs_fn)(const char*, const int*, const int*, const int*, const double*,
                              const int*, double*, const int*, int*);
typedef struct {
    sko_grid grid;
    int k, p, n, kd;
    sko_dpbtrs_fn lapack_trs; /* envelope knob, NULL = restatement */
    double penalty_scale, symmetry_defect;
    double* band;   /* (kd+1) x n, column-major lower band */
    double* factor; /* banded Cholesky factor */
    double interp[SKO_MAXP * SKO_MAXP];
    double deriv_at_k[SKO_MAXP * (SKO_MAXP + 1)];
} sko_poisson;
int sko_poisson_init(sko_poisson* P, const sko_grid* g, int k, double penalty_scale);
void sko_poisson_free(sko_poisson* P);
int sko_poisson_build_load(const sko_poisson* P, const double* rho, double* load);
int sko_poisson_solve(const sko_poisson* P, const double* rho, double* phi, double* E);
void sko_charge_density(const sko_field* fe, const sko_field* fi, double* rho);
/* tests only: 0 = reference order, 1 = electrons first (noise envelope) */
void sko_set_rho_order(int mode);
/* tests only: NULL, NULL = the restatement (reference-LAPACK order) */
void sko_set_lapack(sko_dpbtrf_fn trf, sko_dpbtrs_fn trs);
double sko_electric_energy(const sko_grid* g, int k, const double* E);

/* LAPACK restatement (lapack_band.c): reference-LAPACK dpbtf2 + dtbsv order */
int sko_dpbtrf_lower(int n, int kd, double* ab, int ldab);
void sko_dpbtrs_lower(int n, int kd, const double* ab, int ldab, double* b);

/* ---- step + run loop body (stepper.cpp, run.cpp) ---- */
typedef struct {
    sko_field fe, fi;
    sko_poisson poisson;
    double* E;
    double* phi;
    double sqrt_mu_e, sqrt_mu_i, charge_e, charge_i;
    double time, dt;
    long step;
    sko_limiter limiter;
    int bc;
    int v_adjust;
    double adapt_p, adapt_gamma, adapt_tol;
    long last_shrink_e, last_shrink_i;
    int shrinks_e, shrinks_i;
    sko_stats stats;
    int injection;        /* scenario "injection": neutral source (run.cpp:47-53) */
    double t0, sigma;     /* source window and width */
} sko_state;
/* blob initial state (run.cpp:26-58). Allocates field/E storage. */
int sko_state_init(sko_state* S, double L, double dt, int k, double mu, double sigma, double vmax_e,
                   double vmax_i, int nf, int nc, int m, int nv, const char* limiter,
                   double limiter_threshold, int v_adjust, double adapt_p, double adapt_gamma,
                   double adapt_tol, double penalty_scale);
void sko_state_free(sko_state* S);
/* switch to the injection scenario (run.cpp:47-53): zero initial fields, the
 * source S = blob(x, v)/t0 for t <= t0, applied as source_half_step
 * (stepper.cpp:29-42) before and after the sweeps */
int sko_state_set_injection(sko_state* S, double t0);
/* stepper.cpp:29-42 Heun half step of df/dt = S */
void sko_source_half_step(sko_field* f, double t, double half_dt, double t0, double sigma);
int sko_strang_step(sko_state* S, int max_ghost);
/* one run() loop body: ghost width, strang_step, shrink checks (run.cpp:124-131) */
int sko_run_step(sko_state* S);

#ifdef __cplusplus
}
#endif
#endif
