/*
 * sk_b200.h -- C ABI of the B200-native sLdG time step (libsk_b200.so).
 *
 * Drop-in boundary for the reference solver interface in
 * /root/reference/proj/core (arXiv 2408.11235). The reference has no FFI: its
 * "operator API" is a set of free C++ functions over NodalField&. Each entry
 * point below names the reference function it replaces (file:line); the C++
 * mirror with the reference's signatures and exception types is
 * include/solkin_b200.hpp, the ctypes binding is
 * paper_2408_11235_b200/_native.py, and INTEGRATION.md shows how a maintainer
 * binds the reference's callers to it.
 *
 * Conventions
 *  - Plain pointers and sizes only; device pointers are marked `_dev`.
 *  - All work is enqueued asynchronously on the context's CUDA stream
 *    (sk_ctx_set_stream). Functions that return host values synchronise.
 *  - Every function returns an sk_status; on failure sk_last_error() holds
 *    the message (thread-local). SK_ERR_RUNTIME mirrors std::runtime_error
 *    from solkin::require (common.hpp:9-11); SK_ERR_SIMULATION mirrors
 *    solkin::SimulationError{step} (common.hpp:16-20) and
 *    sk_last_error_step() gives its step.
 *  - Errors detected on the device (ghost width, nonfinite values) surface at
 *    the next synchronising call, or immediately when eager errors are on
 *    (the default; sk_ctx_set_eager_errors).
 *  - Field storage is the reference layout ((vc*p+vn)*nx+xc)*p+xn
 *    (field.hpp:71-73), fp64, double-buffered on the device.
 */
#ifndef SK_B200_H
#define SK_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int sk_status;
#define SK_OK 0
#define SK_ERR_RUNTIME 1    /* std::runtime_error (solkin::require)  */
#define SK_ERR_SIMULATION 2 /* solkin::SimulationError               */
#define SK_ERR_CUDA 3       /* CUDA runtime failure / no device       */

#define SK_BC_ZERO_INFLOW 0 /* BoundaryRule::ZeroInflow (advection.hpp:35) */
#define SK_BC_PERIODIC 1    /* BoundaryRule::Periodic (test rule)          */

#define SK_DIR_X 0 /* SweepDirection::X (limiters.hpp:101) */
#define SK_DIR_V 1

#define SK_SPECIES_ELECTRON 0
#define SK_SPECIES_ION 1

typedef struct sk_ctx sk_ctx;     /* one GPU: x grid, degree k, Poisson plan, stream */
typedef struct sk_field sk_field; /* NodalField on the device (field.hpp:21-80)      */
typedef struct sk_state sk_state; /* SimulationState (stepper.hpp:44-54)             */

/* LimiterConfig (limiters.hpp:19-34). indicator: 0 none, 1 minmod, 2 meanerr;
 * modifier: 0 none, 1 simple WENO, 2 line WENO. */
typedef struct {
    int indicator;
    int modifier;
    int inline_sldg;
    double threshold;
    double gamma_simple[3];
    double gamma_line[3];
    double epsilon;
} sk_limiter;

/* SweepStats (advection.hpp:37-53) */
typedef struct {
    long long outputs;
    long long inline_troubled;
    long long inline_clamped;
    long long inline_mean_outside;
    long long post_checked;
    long long post_troubled;
} sk_stats;

/* VAdjustPolicy (adaptivity.hpp:13-19) */
typedef struct {
    double p;
    double gamma;
    double tol;
} sk_vadjust;

/* ShrinkResult (adaptivity.hpp:23-28) */
typedef struct {
    double vmax_before;
    double vmax_after;
    double mass_before;
    double mass_after;
} sk_shrink_result;

/* RunConfig subset that shapes the step (config.hpp:11-41) */
typedef struct {
    double L, dt, mu, sigma, vmax_e, vmax_i;
    int k, fine_block_cells, coarse_block_cells, refinement_ratio, v_cells;
    sk_limiter limiter;
    int v_adjust;
    sk_vadjust policy;
    double penalty_scale;
    /* scenario (config.hpp:11,18): 0 blob (run.cpp:41-46 initial data), 1
     * injection (zero initial data, neutral source blob(x,v)/t0 for t <= t0
     * applied as source_half_step before and after the sweeps, stepper.cpp:29-42) */
    int scenario;
    double t0;
} sk_run_config;

/* ---- errors ---- */
const char* sk_last_error(void);
long sk_last_error_step(void);
const char* sk_version(void);

/* ---- context: Grid1D x (grid.hpp:18-49), degree k, PoissonOperator
 *      (poisson.hpp:24-57, assembled + reduced once) ---- */
sk_status sk_ctx_create(int device, int k, int nblocks, const double* block_left,
                        const int* block_cells, const double* block_dx, double penalty_scale,
                        sk_ctx** out);
sk_status sk_ctx_destroy(sk_ctx* ctx);
sk_status sk_ctx_set_stream(sk_ctx* ctx, void* cuda_stream);
sk_status sk_ctx_set_eager_errors(sk_ctx* ctx, int on);
/* Exact (parity) mode: every sweep uses the reference's rounding sequence
 * (no FMA contraction), the charge density is summed in the reference's serial
 * order and the Poisson solve is replayed as dpbtrs in reference-BLAS order
 * (poisson.cpp:166-216), so whole trajectories are bitwise the reference's.
 * Off (default, fast mode): DFMA-contracted sweeps (k <= 3), charge density
 * fused into the first x sweep, block-cyclic-reduction solve; results agree
 * with the reference to the 1e-12 relative tolerance. */
sk_status sk_ctx_set_exact_reductions(sk_ctx* ctx, int on);
/* Exact mode per part, for attributing a fast-mode deviation: any OR of
 * SK_EXACT_ARITH (unfused sweep/limiter arithmetic), SK_EXACT_RHO (charge
 * density in the reference's serial order, poisson.cpp:194-216) and
 * SK_EXACT_POISSON (dpbtrs order, poisson.cpp:166-174). SK_EXACT_ALL is
 * sk_ctx_set_exact_reductions(ctx, 1); 0 is fast mode. */
#define SK_EXACT_ARITH 1
#define SK_EXACT_RHO 2
#define SK_EXACT_POISSON 4
#define SK_EXACT_ALL 7
sk_status sk_ctx_set_exact_parts(sk_ctx* ctx, int mask);
/* Fusion of step n's second and step n+1's first x half sweep inside
 * sk_run_steps: one pass over f instead of two (32 instead of 48 B/DoF per
 * step). on: 1 always, 0 never, -1 auto (the default; SK_STEP_FUSION=0/1 in
 * the environment forces it): fused for states of at least 2^32 DoF, whose
 * long steps run under the board power cap, where the lower traffic lifts the
 * clock (C5 -1.5 %, C5 at k = 2 -10 %); not below, where the fused pass is
 * compute-bound at full clock (C3 +8 %). Fast mode, blob scenario, no post
 * limiter, uniform x mesh, one rank (sk_state_step_fusion tells). */
sk_status sk_ctx_set_step_fusion(sk_ctx* ctx, int on);
/* Post limiter V flags fused into the v sweep (default on; SK_POST_FUSION=0 in
 * the environment turns it off at context creation): in the step, on walls
 * without a v halo, the v sweep decides each cell's minmod / mean-error flag
 * from the registers it stores (the stencil limiters.cpp's v pass reads back),
 * so the post limiter V runs only its fixes -- one read of f less per step.
 * The flags are bitwise those of the separate pass. */
sk_status sk_ctx_set_post_fusion(sk_ctx* ctx, int on);
/* Out-of-bounds write check: with SK_GUARD=1 in the environment when the
 * context is created, fields, tables, E, rho and phi are allocated with
 * sentinel guard zones; *bad = guard words overwritten since (0 = clean). */
sk_status sk_ctx_check_guards(sk_ctx* ctx, long long* bad);
/* Capacity of the deferred limiter-clamp list (troubled cells queued by the
 * sweeps, clamped by a fixup kernel); above it the fixup rescans the sweep.
 * Sized when a state is created: at least 4 Mi entries, cells/32 of a pass
 * for the inline limiter, cells/6 for the literature post limiters (cells/3 where the
 * device memory allows: rough data flag 15-25 % of a pass); cap may
 * only lower it (for testing the rescan path). */
sk_status sk_ctx_set_fix_capacity(sk_ctx* ctx, unsigned int cap);
sk_status sk_ctx_synchronize(sk_ctx* ctx); /* also reports device-side errors */
sk_status sk_stats_get(sk_ctx* ctx, sk_stats* out);
sk_status sk_stats_reset(sk_ctx* ctx);
/* Grid1D::three_block (grid.cpp:36-46) with the reference's arithmetic */
sk_status sk_grid_three_block(double left, double right, int fine_cells, int coarse_cells, int m,
                              double* block_left, int* block_cells, double* block_dx);
/* build_shift_matrices(ReferenceBasis::get(k), alpha) (advection.cpp:27-66):
 * the p x p shift matrices A, B (row-major, p = k+1) the sweeps apply, from the
 * host copy of the same constants (bitwise the reference's). k in 0..6, alpha in
 * [0,1). Host only -- no context or GPU needed (the `solkin matrices` table,
 * tools/solkin_main.cpp:43-57). */
sk_status sk_shift_matrices(int k, double alpha, double* A, double* B);

/* ---- fields: NodalField(species, x, v, k) (field.cpp:9-16) ---- */
sk_status sk_field_create(sk_ctx* ctx, int species, double v_left, double v_right, int v_cells,
                          sk_field** out);
sk_status sk_field_destroy(sk_field* f);
size_t sk_field_size(const sk_field* f);
double* sk_field_data_dev(sk_field* f); /* current buffer (device) */
sk_status sk_field_upload(sk_field* f, const double* host, size_t count);
sk_status sk_field_download(sk_field* f, double* host, size_t count);
/* Benchmark stress variant: f *= 1 + amp * xi, xi uniform in
 * [-1, 1) from a counter-based hash of (seed, element index), on the device.
 * Replaces the reference self-check's f * (1 + 0.01 xi) perturbation (not its
 * mt19937_64 sequence). */
sk_status sk_field_perturb(sk_field* f, unsigned long long seed, double amp);
/* `height` runs of `width` doubles, `pitch` doubles apart, from element
 * `offset` of the field (layout field.hpp:71-73) into a packed host array:
 * one x line (offset = row * nx*p, width = nx*p, height = 1) or one v line
 * (offset = x dof, width = 1, height = nv*p, pitch = nx*p) -- gather_v_line
 * (field.cpp:18-24) without a full download. */
sk_status sk_field_download_2d(sk_field* f, double* host, size_t offset, size_t width, size_t height,
                               size_t pitch);
sk_status sk_field_upload_async(sk_field* f, const double* host_pinned, size_t count);
sk_status sk_field_download_async(sk_field* f, double* host_pinned, size_t count);
/* v-shard of a NodalField for a multi-GPU run sharded along v: this rank holds
 * global v cells [cell0, cell0+ncell) plus `halo` cells below and above for
 * the v sweep. Storage rows are contiguous, so each halo is one contiguous
 * device block: sk_field_halo(side 0 lower / 1 upper, send 1: interior edge
 * rows to send, 0: halo rows to receive into). */
sk_status sk_field_create_shard(sk_ctx* ctx, int species, double v_left, double v_right,
                                int v_cells_global, int cell0, int ncell, int halo, sk_field** out);
sk_status sk_field_halo(sk_field* f, int side, int send, double** ptr_dev, size_t* count);
/* the same for an explicit width of `cells` halo cells (<= the allocated halo);
 * a sharded velocity shrink exchanges sk_state_shrink_halo cells */
sk_status sk_field_halo_n(sk_field* f, int side, int send, int cells, double** ptr_dev, size_t* count);
/* v grid: left, dx, cells (synchronises: the cut-off updates it on device) */
sk_status sk_field_v_grid(sk_field* f, double* left, double* dx, int* cells);
/* run.cpp:41-46 blob f = (2 pi)^-1/2 exp(-x^2/(2 sigma^2)) exp(-v^2/2) */
sk_status sk_field_fill_blob(sk_field* f, double sigma);

/* ---- operators ---- */
/* advect_x (advection.hpp:83; advection.cpp:144-207). max_ghost < 0: unchecked. */
sk_status sk_advect_x(sk_field* f, double tau, double sqrt_mu, int bc, const sk_limiter* lim,
                      int max_ghost, long step_index);
/* advect_v (advection.hpp:87-88; advection.cpp:209-238). E_dev: nx*(k+1) doubles. */
sk_status sk_advect_v(sk_field* f, double tau, const double* E_dev, double charge_sign,
                      double sqrt_mu, int bc, const sk_limiter* lim);
/* apply_post_limiter (limiters.hpp:107-108; limiters.cpp:280-345) */
sk_status sk_post_limit(sk_field* f, int dir, const sk_limiter* lim, int bc);
/* charge_density (poisson.hpp:61; poisson.cpp:194-216) -> rho_dev[nx*(k+1)] */
sk_status sk_charge_density(sk_field* fe, sk_field* fi, double* rho_dev);
/* PoissonOperator::solve (poisson.cpp:166-192); phi_dev may be NULL */
sk_status sk_poisson_solve(sk_ctx* ctx, const double* rho_dev, double* E_dev, double* phi_dev);
/* check_velocity_shrink (adaptivity.hpp:21; adaptivity.cpp:16-38); synchronises */
sk_status sk_check_velocity_shrink(sk_field* f, const sk_vadjust* policy, int* out_shrink);
/* shrink_velocity_domain (adaptivity.hpp:33; adaptivity.cpp:94-130); synchronises */
sk_status sk_shrink_velocity_domain(sk_field* f, const sk_vadjust* policy, sk_shrink_result* out);
/* mass, l2_norm (field.cpp:52-88), momentum, kinetic energy; synchronises */
sk_status sk_field_moments(sk_field* f, double* out4);
/* electric_energy (diagnostics.cpp:71-83) of E_dev; synchronises */
sk_status sk_electric_energy(sk_ctx* ctx, const double* E_dev, double* out);

/* FluxSample (diagnostics.hpp:24-32) */
typedef struct {
    double t;
    double je_plus, je_minus, ji_plus, ji_minus, je_naive, ji_naive;
    double mass_e, mass_i, e_energy, vmax_e, vmax_i;
} sk_flux_sample;

/* Summary (diagnostics.hpp:34-40) */
typedef struct {
    double mass_e, mass_i, charge, l2_e, l2_i, e_energy, vmax_e, vmax_i;
} sk_summary;

/* RunResult subset (run.hpp:20-33) */
typedef struct {
    int exit_code;          /* 0 ok, 1 SimulationError (message in sk_last_error) */
    long steps_done;
    long shrinks_e, shrinks_i;
    double wall_seconds;
    sk_stats stats;
} sk_run_result;

/* ---- state + step: build_initial_state (run.cpp:26-58), strang_step
 *      (stepper.cpp:44-103), run() loop body (run.cpp:124-131) ---- */
sk_status sk_state_create(sk_ctx* ctx, const sk_run_config* cfg, sk_state** out);
sk_status sk_state_destroy(sk_state* s);
sk_field* sk_state_field(sk_state* s, int species);
double* sk_state_E_dev(sk_state* s);
sk_status sk_state_download_E(sk_state* s, double* host, size_t count);
/* the charge density of the state's last step (poisson.cpp:194-216 output,
 * the Poisson right-hand side), nx*(k+1) values */
sk_status sk_state_download_rho(sk_state* s, double* host, size_t count);
/* v-sharded state: rank `rank` of `nranks` holds v_cells/nranks cells of each
 * species plus `halo` cells; the step runs as phase 2 (x half sweep + local
 * rho) -> caller all-reduces rho (sk_state_rho_dev) and exchanges the halos
 * -> phase 3 (Poisson, v sweep, x half sweep, step end; with the velocity
 * cut-off also the local shrink check: the ranks holding the probe cells
 * clear sk_state_shrink_flags_dev) -> caller all-reduces the two int flags
 * (MIN) and, for a species whose flag is set, exchanges
 * sk_state_shrink_halo cells with sk_field_halo_n -> phase 4 (shrink).
 * With a post limiter (apply_post_limiter), phase 3 stops after
 * the v sweep: the caller exchanges one-cell halos (sk_field_halo_n, cells 1)
 * and phase 5 runs post V, the second x half sweep, post X, the step end and
 * the local cut-off check.
 * Phases 0/1: local initial rho and the Poisson solve of the all-reduced rho
 * (initial field). */
sk_status sk_state_create_shard(sk_ctx* ctx, const sk_run_config* cfg, int rank, int nranks,
                                int halo, sk_state** out);
double* sk_state_rho_dev(sk_state* s);
int* sk_state_shrink_flags_dev(sk_state* s); /* int[2], device: 1 = shrink this step */
int sk_state_shrink_halo(sk_state* s);        /* halo cells a sharded shrink reads */
/* Adaptive v-halo exchange of a shard (phases 6-9 of sk_state_phase): phase 6
 * (Poisson + v tables) records the cells this step's v sweep reads beyond the
 * shard -- max over x dofs of |i*|+1 (advection.cpp:14-25, :226) -- into a
 * pinned word read by sk_state_vhalo_need once phase 6 has completed; the
 * caller exchanges that many cells (sk_state_set_vhalo, then sk_field_halo)
 * while phase 7 sweeps the v chunks that read no halo cell for shifts up to
 * `bound`, and phase 8 sweeps the rest (phase 9: all chunks, when the shift
 * exceeded `bound`). Width and bound are at most sk_state_vhalo_capacity. */
sk_status sk_state_vhalo_need(sk_state* s, int* need);
sk_status sk_state_set_vhalo(sk_state* s, int width, int bound);
int sk_state_vhalo_capacity(sk_state* s);
sk_status sk_state_phase(sk_state* s, int phase);
/* ---- diagnostics and output (diagnostics.cpp, run.cpp:60-169).
 * Single-GPU states; all synchronise. */
/* state.time (stepper.cpp:98) */
sk_status sk_state_time(sk_state* s, double* t);
/* wall_flux (diagnostics.cpp:24-69): side 0 left, 1 right; bitwise the
 * reference's (boundary cells downloaded, the reference's loop on the host) */
sk_status sk_state_wall_flux(sk_state* s, int species, int side, double* outflow, double* naive);
/* sample_fluxes (diagnostics.cpp:98-116); masses from the device reduction */
sk_status sk_state_sample_fluxes(sk_state* s, sk_flux_sample* out);
/* summarize (diagnostics.cpp:85-96) */
sk_status sk_state_summarize(sk_state* s, sk_summary* out);
/* OutputWriter::write_snapshot (diagnostics.cpp:161-194): dir/snapshot_<step>.bin
 * (SOLKSNP1 layout) + .meta, byte-compatible with the reference's files */
sk_status sk_state_write_snapshot(sk_state* s, const char* dir);
/* OutputWriter::write_profiles (diagnostics.cpp:196-220): dir/profiles_<step>.csv */
sk_status sk_state_write_profiles(sk_state* s, const char* dir);
/* run() (run.cpp:60-169): nsteps run() loop bodies with a flux.csv row every
 * `cadence` steps (and at step 0), snapshots / profiles at their cadences (0:
 * off), run.log, into out_dir (NULL: no files). The steps between samples run
 * as CUDA-graph replays. */
sk_status sk_run(sk_ctx* ctx, const sk_run_config* cfg, long nsteps, int cadence, int snapshot_cadence,
                 int profile_cadence, const char* out_dir, sk_run_result* out);

/* one strang_step (no shrink); max_ghost < 0: run()'s rule */
sk_status sk_strang_step(sk_state* s);
/* one run() loop body: strang_step + shrink checks with the 10-step cooldown */
sk_status sk_run_step(sk_state* s);
/* n loop bodies, replayed as CUDA graphs of up to 10 bodies (SK_GRAPH_STEPS).
 * With step fusion on (sk_ctx_set_step_fusion, fast mode) each step boundary
 * inside a graph runs step n's second and step n+1's first x half sweep as one
 * pass over f, unless the velocity cut-off may check at the end of step n
 * (then both sweeps run separately, decided on the device). */
sk_status sk_run_steps(sk_state* s, int n);
/* *on = 1 when sk_run_steps fuses this state's step boundaries (see
 * sk_ctx_set_step_fusion). */
sk_status sk_state_step_fusion(sk_state* s, int* on);
/* Capture (without running) the CUDA graphs sk_run_steps(state, n) will
 * replay from the current state, so a later sk_run_steps(n) does no capture
 * inside a timed region. */
sk_status sk_state_prepare_steps(sk_state* state, int n);
sk_status sk_state_step_index(sk_state* s, long* step);
sk_status sk_state_shrinks(sk_state* s, int species, int* count, long* last_step);
/* per-phase CUDA-event timing of the step (disables graph replay while on).
 * Phases: 0 x tables, 1 x sweep 1, 2 post X 1, 3 charge density, 4 Poisson,
 * 5 v tables, 6 v sweep, 7 post V, 8 x sweep 2, 9 post X 2, 10 step end +
 * cut-off, 11/12/13 the launches after the main kernel of x sweep 1 / v sweep /
 * x sweep 2 (limiter fixup, fused-moment reduction). Phases 1, 6, 8 then time
 * the sweep kernel alone. sk_state_phase_times returns and clears the
 * accumulated ms. */
sk_status sk_state_set_phase_timing(sk_state* s, int on);
sk_status sk_state_phase_times(sk_state* s, double* ms, long* count, int n);
/* kernels this context has enqueued (graph replays included) */
long long sk_ctx_launch_count(sk_ctx* ctx);
/* drop-in strang_step over HOST NodalFields: upload, step, download */
sk_status sk_run_step_host(sk_state* s, double* fe_host, double* fi_host, size_t count);
/* n such steps with the host copies pipelined across steps (each step still
 * uploads both species from and downloads both results into the host arrays;
 * the next step's electron upload overlaps this step's ion download). */
sk_status sk_run_steps_host(sk_state* s, int n, double* fe_host, double* fi_host, size_t count);

#ifdef __cplusplus
}
#endif
#endif
