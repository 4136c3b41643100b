// sk_kernels.cuh -- kernel parameter blocks and launchers (sk_kernels.cu).
#pragma once

#include "sk_internal.hpp"

namespace sk {

constexpr int kXThreads = 256;  // x sweep CTA
constexpr int kVThreads = 128;  // v sweep CTA (one thread per x dof)
constexpr int kVChunk = 32;     // v cells per v-sweep thread
constexpr int kRhoCorrCopies = 64;  // fused-moment clamp corrections: copies keyed by v row

inline int xtab_nf(int P) { return ((2 + 2 * P * P + 2 * P) + 1) & ~1; }  // AoS row, 16B aligned
inline int vtab_nf(int P) { return 2 + 2 * P * P + 2 * P; }

// Per-line shift tables (make_plan, advection.cpp:132-140) for the x sweep.
struct XTabArgs {
    Basis basis;
    Grid grid;
    const DevVGrid* vg[2];  // per species
    DevStatus* st;
    double* tab[2];      // [nclass][nlines][nf]
    double sqrt_mu[2];
    double tau;
    int nlines;          // nv * P
    int nspecies;
    int species0;        // first species index handled
    int inline_sldg;
    double threshold;
    int max_ghost;       // >=0 explicit, -1 no check, -2 run() rule from dt_auto
    double dt_auto;
    long long step_index;  // <0: use st->step
};

// A field's two buffers exchange roles after a velocity cut-off event (the
// projection lands in the other buffer; finalize toggles the field's flag
// instead of copying it back). Every kernel resolves its buffers through it.
__device__ __forceinline__ bool field_flipped(const int* flip) { return flip != nullptr && *flip != 0; }

struct XSweepArgs {
    Basis basis;
    Grid grid;
    DevStatus* st;
    const double* src[2];
    double* dst[2];
    const int* flip[2];   // per-field buffer flip (shrink events): swap src and dst
    const double* tab[2];
    int nlines;
    int nspecies;
    int species0;
    int tile_start[kMaxBlocks + 1];  // tiles per block (prefix)
    int inline_sldg;
    int periodic;
    int check_finite;
    int fma;  // fast-mode DFMA arithmetic (0: reference rounding sequence)
    double threshold;
    double thr_hi, thr_lo;  // make_thr_cut(threshold), precomputed on the host
    // deferred limiter clamp: troubled cells are queued here and clamped by
    // the fixup kernel so one slow cell never stalls a whole CTA
    unsigned long long* fix_list;
    unsigned int* fix_count;
    unsigned int fix_cap;
    // fused charge-density moment (first x sweep, no post limiter): per-CTA
    // partial sums [G/ntl][nx*P] + int64 fixed-point corrections of clamped cells
    int rho_fuse;
    double* rho_partial;
    unsigned long long* rho_corr;
    const DevVGrid* vg[2];
    double charge_w[2];   // +1 ions, -1 electrons (poisson.cpp:202-214)
    // 3-block ghost cells across a dx jump, precomputed by xghost_kernel:
    // [(sp * nlines + line) * nblocks + b][j - 1][P], j = 1..ghost_cap cells
    // outward on the side the line's shift reaches (null: computed in-kernel)
    double* ghost;
    int ghost_cap;
    // post-limiter flag pass (xsweep_kernel MODE 1): the literature indicator
    // of every cell from its window, in place; flagged cells are queued
    PostCfg post;
    // sweep + post-limiter x flags of its outputs (1 minmod, 2 mean error;
    // xsweep_kernel MODE 4 / 5; 0: plain sweep)
    int post_x;
    // device-decided alternatives (fused / unfused step boundary): the kernel
    // runs only if (*gate != 0) == gate_on; gate == nullptr: always
    const int* gate;
    int gate_on;
    // injection source half step (stepper.cpp:29-42) fused into
    // the sweep: 1 = added to the source cells as they are read (the half step
    // at state.time before the first x sweep, stepper.cpp:68-72), 2 = added to
    // the outputs (at state.time + half after the second, stepper.cpp:93-97);
    // the fixup kernel applies it the same way to the cells it reloads / clamps
    int src_mode;
    const double* src_gx;      // [nxd] x factor of the source blob
    const double* src_gv[2];   // [kSourceLevels][nlines] v factor per v-grid level
    double src_half, src_t0;
};

struct VTabArgs {
    Basis basis;
    const DevVGrid* vg[2];
    double* tab[2];      // SoA [nf][nxd]
    const double* E;
    double charge[2];
    double sqrt_mu[2];
    double tau;
    int nxd;
    int nspecies;
    int species0;
    int inline_sldg;
    double threshold;
    DevStatus* st;
    int halo_lo, halo_hi;  // v-shard: max readable cells below/above (-1: wall)
    int* halo_need;        // v-shard: max over x dofs of the cells read beyond the shard (atomicMax)
};

struct VSweepArgs {
    Basis basis;
    DevStatus* st;
    const double* src[2];  // points at local cell 0 (halo rows before/after)
    double* dst[2];
    const int* flip[2];
    const double* tab[2];
    long long ld;          // row stride (nx * P)
    int nxd;
    int n;                 // local v cells written
    int gl, gr;            // halo cells readable below / above
    int nspecies;
    int species0;
    int inline_sldg;
    int periodic;
    int check_finite;
    int chunk_major;  // grid order: v chunks fastest (large tables, see vsweep_kernel)
    int fma;  // fast-mode DFMA arithmetic (0: reference rounding sequence)
    double threshold;
    double thr_hi, thr_lo;  // make_thr_cut(threshold), precomputed on the host
    unsigned long long* fix_list;
    unsigned int* fix_count;
    unsigned int fix_cap;
    int chunk0, nchunks;  // v chunks [chunk0, chunk0 + nchunks) of kVChunk cells (nchunks 0: all)
    // post limiter V flags fused into the sweep (1 minmod, 2 mean error; 0 off):
    // flagged cells go to fix_list in the post pass's format (walls, no halo)
    int post_v;
    PostCfg post;
};

struct RhoArgs {
    Basis basis;
    const DevStatus* st;
    const DevVGrid* vg[2];
    const double* f[2];
    const double* alt[2];  // the fields' other buffers (used when flipped)
    const int* flip[2];
    double* partial;       // [2][nchunks][nxd]
    double* rho;
    long long ld;
    int nxd;
    int nrows;             // local v rows (cells*P)
    int nchunks;
    int rows_per_chunk;
};

struct PoissonDev {
    int k, ps, ncells, nlevels;
    int kd;
    const double* chol;    // banded Cholesky factor (ldab = kd+1), exact mode
    int level_n[32];
    long long level_off[32], keep_off[32], odd_off[32];
    const double *AlphaT, *GammaT, *LoT, *UpT, *DinvT, *DinvTop;  // see PoissonPlan
    const double *interp, *deriv, *h, *ws;
    double *bws, *xws;     // per level SoA [ps][rows]
    // one step of iterative refinement on the block-cyclic-reduction solve:
    // stage 1 solves from rho into ir_x (phi, AoS); stage 2 solves A d = b - A x
    // (residual from the SIPG band, computed in its load phase) and writes
    // phi = x + d and E. band = the assembled matrix, (kd+1) x n lower.
    const double* band;
    double* ir_x;
    double* exws;          // exact mode: 3n doubles (poisson_exact_kernel)
    const DevStatus* st;   // halts on a raised error
};

struct ShrinkArgs {
    Basis basis;
    DevStatus* st;
    DevVGrid* vg[2];
    double* f[2];
    double* out[2];
    const int* flip[2];    // f/out exchange roles when set; finalize toggles it
    int* flip_w[2];
    double* ttab[2];       // [nv][4 pieces][P*P]
    int* tcell[2];         // [nv][4]
    long long ld;
    int nxd;
    int nv;                // v cells held by this field (a v shard: nv < nv_global)
    int nv_global;
    int cell0;             // first global v cell held
    int halo;              // allocated halo cells below/above (old cells a shard may read)
    int species_mask;      // which species to consider
    int v_adjust;
    // 0: run() cadence (check + shrink), 1: shrink unchecked (standalone),
    // -1: forced check only (standalone), -2: cadence check only (v shards,
    // before the decision is all-reduced), 2: shrink only (decision taken)
    int force;
    double p, gamma, tol;
    long long cooldown;
};

struct DiagArgs {
    Basis basis;
    Grid grid;
    const DevVGrid* vg;
    const double* f;
    const double* alt;
    const int* flip;
    double* partial;       // [nblk][4]
    long long ld;
    int nxd;
    int nrows;
};

struct PostArgs {
    Basis basis;
    Grid grid;
    DevStatus* st;
    const double* src[2];
    double* dst[2];
    const int* flip[2];
    int gl, gr;            // readable v halo cells below/above (v shards; 0 at walls)
    PostCfg cfg;
    long long ld;
    int nxd;
    int nrows;             // v rows
    int nv;
    int nspecies;
    int species0;
    int periodic;
    int tile_start[kMaxBlocks + 1];
    int fma;               // fast-mode indicators (0: the reference's operation order)
    // flagged cells are queued for the modifier kernel (overflow: it rescans)
    unsigned long long* fix_list;
    unsigned int* fix_count;
    unsigned int fix_cap;
    double* fix_vals;      // [fix_cap][P] modified values, scattered after all are computed
    int flags_queued;      // the sweep already queued the flags (VSweepArgs::post_v, XSweepArgs::post_x)
    // x, after a sweep that fused the charge density: corrections of the
    // modified cells (null: none)
    unsigned long long* rho_corr;
    double charge_w[2];
    const DevVGrid* vg[2];
};

// launchers (P = k+1 dispatch inside)
cudaError_t launch_init_device();
cudaError_t launch_xtab(const XTabArgs& a, cudaStream_t s);
cudaError_t launch_xsweep(const XSweepArgs& a, int ntiles, cudaStream_t s);
// 3-block ghost pre-pass (a.ghost, a.ghost_cap set); needed only when adjacent
// blocks differ in dx and the boundary is not periodic
cudaError_t launch_xghost(const XSweepArgs& a, cudaStream_t s);
inline bool xghost_grid(const Grid& g) {
    for (int b = 0; b + 1 < g.nblocks; ++b)
        if (g.dx[b] != g.dx[b + 1]) return true;
    return false;
}
cudaError_t launch_vtab(const VTabArgs& a, cudaStream_t s);
cudaError_t launch_vsweep(const VSweepArgs& a, cudaStream_t s);
cudaError_t launch_xfix(const XSweepArgs& a, cudaStream_t s);
// rho = sum of the fused partials + fixed-point corrections; returns #partials
// fused = 1: the partials of the MODE 3 (two fused half sweeps) launch
cudaError_t launch_rho_fused_reduce(const XSweepArgs& a, double* rho, cudaStream_t s, int fused = 0);
int xsweep_rho_groups(const XSweepArgs& a, int fused = 0);
// two consecutive x half sweeps in one pass (step n's last, step n+1's first
// with the fused charge density), fast mode, single-dx-class non-periodic grids
bool xsweep_fused_supported(int P);
cudaError_t launch_xsweep_fused(const XSweepArgs& a, cudaStream_t s);
// its fixup: the queued output cells recomputed with both clamps (inline sLdG)
cudaError_t launch_xfix2(const XSweepArgs& a, cudaStream_t s);
// device decision for a fusable step boundary (DevStatus::fuse_ok) and the
// flip-flag toggle of its unfused alternative
cudaError_t launch_fuse_decide(DevStatus* st, int v_adjust, long long cooldown, cudaStream_t s);
cudaError_t launch_flip_toggle(const DevStatus* st, int* f0, int* f1, cudaStream_t s);
cudaError_t launch_vfix(const VSweepArgs& a, cudaStream_t s);
cudaError_t launch_rho(const RhoArgs& a, int nspecies_mask, cudaStream_t s);
cudaError_t launch_poisson(const PoissonDev& pd, int stage, const double* rho, double* E, double* phi,
                           cudaStream_t s);
// exact-reduction mode: reference summation order / sequential dpbtrs
cudaError_t launch_rho_exact(const RhoArgs& a, cudaStream_t s);
cudaError_t launch_poisson_exact(const PoissonDev& pd, const double* rho, double* E, double* phi,
                                 cudaStream_t s);
// injection source half step (stepper.cpp:29-42), both species
constexpr int kSourceLevels = 48;  // v-grid levels (velocity shrinks) with host-built exp tables
struct SourceArgs {
    double* f[2];
    double* alt[2];
    const int* flip[2];
    const double* gx;     // [nxd]: (2 pi)^-1/2 exp(-x^2 / (2 sigma^2)) at the x nodes
    const double* gv[2];  // [kSourceLevels][nrows]: exp(-v^2/2) at the v nodes of each v-grid level
    int nrows, nxd;
    long long ld;
    DevStatus* st;
    double half, t0;
    int second;           // 0: source at state.time, 1: at state.time + half
};
cudaError_t launch_source(const SourceArgs& a, cudaStream_t s);

cudaError_t launch_step_end(DevStatus* st, double dt, int v_adjust, long long cooldown, int species_mask,
                            cudaStream_t s);
cudaError_t launch_shrink(const ShrinkArgs& a, cudaStream_t s);
cudaError_t launch_diag(const DiagArgs& a, double* out4, double* partial, cudaStream_t s);
cudaError_t launch_fill_separable(double* f, const double* gx, const double* gv, long long ld,
                                  int nrows, cudaStream_t s);
cudaError_t launch_post_x(const PostArgs& a, int ntiles, cudaStream_t s);
cudaError_t launch_post_v(const PostArgs& a, cudaStream_t s);
cudaError_t launch_scale_copy(double* dst, const double* src, size_t n, cudaStream_t s);
cudaError_t launch_perturb(double* f, size_t n, unsigned long long seed, double amp, cudaStream_t s);

}  // namespace sk
