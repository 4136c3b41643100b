// sk_internal.hpp -- shared host/device types of the B200 sLdG library.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "sk_numerics.cuh"

namespace sk {

constexpr int kMaxBlocks = 8;

// Block-structured 1D x mesh (core/include/solkin/grid.hpp:18-49) plus the
// dx classes a sweep needs one shift plan for (advection.cpp:172-180 keys
// plans by dx).
struct Grid {
    int nblocks = 0;
    double left[kMaxBlocks] = {};
    int cells[kMaxBlocks] = {};
    double dx[kMaxBlocks] = {};
    int start[kMaxBlocks + 1] = {};
    int ncells = 0;
    int cls[kMaxBlocks] = {};       // block -> dx class
    int nclass = 0;
    double class_dx[kMaxBlocks] = {};
};

// Mutable per-species device state: the v grid shrinks on device
// (adaptivity.cpp:94-130) so kernels read it from here, never from the host.
struct DevVGrid {
    double left;
    double dx;
    int cells;   // global v cell count (Grid1D::right = left + cells*dx)
    int cell0;   // first global v cell held by this field (v-shard offset)
};

// Device-resident step / error / counter block (one per context).
struct DevStatus {
    unsigned long long stats[2][4];  // [species][troubled, clamped, mean_outside, post_troubled]
    unsigned long long post_checked[2];
    int err_code;       // 0 ok, 1 runtime_error, 2 SimulationError
    int err_kind;       // 1 ghost width, 2 neighbour capacity, 3 nonfinite, 4 shrink table
    int err_need;       // required ghost width
    int err_have;       // provided ghost width
    long long err_step;
    long long step;               // state.step (stepper.hpp:53)
    long long last_shrink[2];     // run.cpp:81-82
    int shrink_flag[2];           // decision of the current check
    int shrink_count[2];
    double vmax_before[2];        // of the last shrink
    int nonfinite;
    int fuse_ok;                  // this step boundary runs the fused x half sweeps (no cut-off check can fire)
    double time;                  // state.time (stepper.cpp:98), advanced at each step end
};

// Host-side reference-cell constants (bitwise equal to basis.cpp).
Basis make_basis(int k);
double host_lagrange(const Basis& b, int n, double xi);
double host_lagrange_derivative(const Basis& b, int n, double xi);

int grid_block_of(const Grid& g, int cell);
double grid_cell_left(const Grid& g, int cell);
double grid_cell_width(const Grid& g, int cell);
double grid_right(const Grid& g);
std::string grid_init(Grid& g, int nblocks, const double* left, const int* cells, const double* dx);

// Block cyclic reduction plan for the SIPG Poisson band (poisson.cpp:59-133):
// assembled exactly like the reference, reduced on the host once, solved on the
// device every step (sk_poisson.cu).
struct PoissonPlan {
    int k = 0, ps = 0, ncells = 0, nlevels = 0;
    std::vector<int> level_n;        // block rows per level
    std::vector<long> level_off;     // offset (in blocks) of each level (vectors)
    std::vector<long> keep_off;      // offset of the level's even rows (alpha/gamma)
    std::vector<long> odd_off;       // offset of the level's odd rows (Lo/Up/Dinv)
    // transposed + compacted for coalesced device reads: entry (m,n) of all
    // rows of a level is contiguous, [level block][ps*ps][rows]
    std::vector<double> AlphaT, GammaT, LoT, UpT, DinvT, DinvTop;
    std::vector<double> interp;      // (k+2)x(k+1)
    std::vector<double> deriv;       // (k+1)x(k+2)
    std::vector<double> h;           // cell widths
    std::vector<double> ws;          // weights of degree k+1
    std::vector<double> band;        // reference band (for residual checks)
    std::vector<double> chol;        // dpbtf2 factor of band (exact-reduction mode)
    int kd = 0;
    double symmetry_defect = 0.0;
};
std::string poisson_plan_build(PoissonPlan& P, const Grid& g, int k, double penalty_scale);

}  // namespace sk
