// sk_kernels.cu -- sm_100a kernels of the sLdG time step.
//
// Data layout in HBM is the reference's NodalField layout
// ((vc*P+vn)*nx+xc)*P+xn (core/include/solkin/field.hpp:71-73): an x line is a
// contiguous row of nx*P doubles, a v line is a column with row stride nx*P.
//
//   xtab_kernel     per (species, dx class, v row): i*, alpha, A, B, limiter
//                   moments (make_plan, advection.cpp:132-140) + ghost checks
//   xsweep_kernel   K1: one CTA per (x-row, tile of a block): coalesced window
//                   load (with 3-block ghost transfer, adaptivity.cpp:169-207)
//                   -> SoA smem -> per-cell projection + inline limiter in
//                   registers -> SoA smem -> coalesced store
//   vtab_kernel     per (species, x dof): tables from E (advect_v, :209-238)
//   vsweep_kernel   K2: one thread per x dof over a chunk of v cells, sliding
//                   2-cell register window; loads/stores coalesced across x
//   rho_*           K4: deterministic two-pass charge-density moment
//   poisson_kernel  block-cyclic-reduction replay of the SIPG solve + E=-phi'
//   shrink_*        K5/K6: velocity cut-off check, transfer tables, projection
//   diag_*          K8: mass / L2 / momentum / kinetic-energy reductions
//   post_*          K3: minmod / mean-error indicators + simple / line WENO
// All arithmetic is fp64 with -fmad=false so per-cell results are bitwise the
// reference's.
#include <algorithm>
#include <type_traits>
#include <utility>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "sk_kernels.cuh"

#include <cstdlib>

namespace sk {

namespace {

template <int P>
__host__ __device__ constexpr int xs_pad() {
    return P == 2 ? 8 : P == 3 ? 5 : P == 4 ? 4 : P >= 5 ? 3 : 0;
}
template <int P, int T>
__host__ __device__ constexpr int xs_stride() {
    return ((T + 2 + 15) / 16) * 16 + xs_pad<P>();
}
template <int P>
__host__ __device__ constexpr int xnf() {
    return ((2 + 2 * P * P + 2 * P) + 1) & ~1;
}
template <int P>
__host__ __device__ constexpr int vnf() {
    return 2 + 2 * P * P + 2 * P;
}

__device__ __forceinline__ void raise_error(DevStatus* st, int code, int kind, int need, int have,
                                            long long step) {
    if (atomicCAS(&st->err_code, 0, code) == 0) {
        st->err_kind = kind;
        st->err_need = need;
        st->err_have = have;
        st->err_step = step;
    }
}

// A raised error halts the run: every later kernel of the step sequence
// returns at entry, so the state stays as the failing step left it (the
// reference's exception unwinds out of run(): run.cpp:147-155) until the host
// collects and clears the error.
__device__ __forceinline__ bool halted(const DevStatus* st) {
    return st && *reinterpret_cast<const volatile int*>(&st->err_code) != 0;
}

// Programmatic dependent launch: every kernel of the step is launched with
// programmatic stream serialisation (pdl_launch), waits here for the previous
// grid's completion and memory before touching anything, and at once lets the
// next kernel's CTAs be scheduled as its own last wave retires -- the launch
// and block-scheduling gaps between the ~15 kernels of a step overlap the
// previous kernel's tail. (A no-op for kernels launched without the attribute.)
__constant__ int c_pdl_trigger;  // 1: trigger at entry, 0: implicit trigger at CTA exit (SK_PDL)
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (c_pdl_trigger) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

__device__ __forceinline__ void count_flags(unsigned long long* dst, unsigned t, unsigned c,
                                            unsigned o) {
    const unsigned full = 0xffffffffu;
    t = __reduce_add_sync(full, t);
    c = __reduce_add_sync(full, c);
    o = __reduce_add_sync(full, o);
    if ((threadIdx.x & 31) == 0) {
        if (t) atomicAdd(&dst[0], (unsigned long long)t);
        if (c) atomicAdd(&dst[1], (unsigned long long)c);
        if (o) atomicAdd(&dst[2], (unsigned long long)o);
    }
}

// Warp-aggregated append of troubled cells to the deferred-clamp list. The
// counter keeps counting past the capacity so the fixup kernel can tell that
// the list overflowed (it then rescans the whole sweep). Called by the whole
// (converged) warp; the common no-troubled-cell case is one vote.
template <int N>
__device__ __forceinline__ void defer_push_n(unsigned int* count, unsigned int cap,
                                             unsigned long long* list, const bool (&want)[N],
                                             const unsigned long long (&entry)[N],
                                             unsigned members = 0xffffffffu) {
    bool any = false;
#pragma unroll
    for (int i = 0; i < N; ++i) any |= want[i];
    if (!__any_sync(members, any)) return;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const unsigned m = __ballot_sync(members, want[i]);
        if (!m) continue;
        const int leader = __ffs(m) - 1;
        unsigned base = 0;
        if (lane == leader) base = atomicAdd(count, (unsigned)__popc(m));
        base = __shfl_sync(members, base, leader);
        const unsigned slot = base + __popc(m & ((1u << lane) - 1u));
        if (want[i] && slot < cap) list[slot] = entry[i];
    }
}

// the same queue staged per warp in shared memory: flagged entries collect in
// the warp's kQCap-slot slice and reach the global list in one atomic + one
// coalesced copy per flush, so a warp stalls on the contended counter once per
// kQCap entries instead of once per flagged tile. n is warp-uniform.
constexpr int kQCap = 64;
// post-limiter list entries (sp << 63 | row << 32 | col): bit 62 marks a
// candidate whose flag the fix kernel decides from the field (rows < 2^30)
constexpr unsigned long long kPostCandidate = 1ull << 62;
__device__ __forceinline__ void wq_flush(unsigned long long* q, int& n, unsigned int* count,
                                         unsigned int cap, unsigned long long* list,
                                         unsigned members = 0xffffffffu) {
    if (n == 0) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(members) - 1;
    __syncwarp(members);
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(count, (unsigned)n);
    base = __shfl_sync(members, base, leader);
    const int step = __popc(members);  // members' ranks cover the entries
    for (int i = __popc(members & ((1u << lane) - 1u)); i < n; i += step)
        if (base + i < cap) list[base + i] = q[i];
    __syncwarp(members);
    n = 0;
}
template <int N>
__device__ __forceinline__ void wq_push(unsigned long long* q, int& n, unsigned int* count, unsigned int cap,
                                        unsigned long long* list, const bool (&want)[N],
                                        const unsigned long long (&entry)[N],
                                        unsigned members = 0xffffffffu) {
    bool any = false;
#pragma unroll
    for (int i = 0; i < N; ++i) any |= want[i];
    if (!__any_sync(members, any)) return;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const unsigned m = __ballot_sync(members, want[i]);
        if (!m) continue;
        if (n + __popc(m) > kQCap) wq_flush(q, n, count, cap, list, members);
        if (want[i]) q[n + __popc(m & ((1u << lane) - 1u))] = entry[i];
        n += __popc(m);
    }
}

// per-species limiter counters of a whole block: warp reduce -> shared ->
// one global atomic per nonzero counter per block (the fixup kernels' per-warp
// atomics all hit the same six words)
__device__ __forceinline__ void block_count_flags(DevStatus* st, const unsigned (&ct)[2],
                                                  const unsigned (&cc)[2], const unsigned (&co)[2]) {
    __shared__ unsigned acc[6];
    if (threadIdx.x < 6) acc[threadIdx.x] = 0;
    __syncthreads();
    const unsigned full = 0xffffffffu;
    unsigned v[6] = {ct[0], cc[0], co[0], ct[1], cc[1], co[1]};
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        v[i] = __reduce_add_sync(full, v[i]);
        if ((threadIdx.x & 31) == 0 && v[i]) atomicAdd(&acc[i], v[i]);
    }
    __syncthreads();
    if (threadIdx.x < 6 && acc[threadIdx.x])
        atomicAdd(&st->stats[threadIdx.x / 3][threadIdx.x % 3], (unsigned long long)acc[threadIdx.x]);
}

template <int P>
constexpr bool kHasFmaDev = P <= 4;  // fast-mode DFMA kernels exist for k <= 3

// true when none of the P values is inf/NaN: one test on the OR of the
// exponent fields' all-ones patterns instead of P separate isfinite()
template <int P>
__device__ __forceinline__ bool all_finite(const double* o) {
    unsigned nf = 0;
#pragma unroll
    for (int m = 0; m < P; ++m) nf |= (unsigned)((((unsigned)__double2hiint(o[m]) & 0x7ff00000u) == 0x7ff00000u));
    return nf == 0;
}

// ---------------------------------------------------------------------------
// x tables
// ---------------------------------------------------------------------------
template <int P>
__global__ void xtab_kernel(const __grid_constant__ XTabArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    const int line = blockIdx.x * blockDim.x + threadIdx.x;
    if (line >= a.nlines) return;
    const int sp = a.species0 + blockIdx.y;
    const Grid& g = a.grid;
    const DevVGrid vg = *a.vg[sp];
    const int vc = line / P, vn = line - (line / P) * P;
    // field.cpp:37-40 v_node = cell_left + cell_width * node
    // global cell index so a v-shard reproduces the single-GPU v_node bitwise
    const double vnode = (vg.left + (vc + vg.cell0) * vg.dx) + vg.dx * a.basis.nodes[vn];
    const double speed = vnode / a.sqrt_mu[sp];  // advection.cpp:164
    constexpr int NF = xnf<P>();
    int istar_c[kMaxBlocks];
    for (int c = 0; c < g.nclass; ++c) {
        int istar;
        double alpha;
        decompose_shift(speed, a.tau, g.class_dx[c], istar, alpha);
        istar_c[c] = istar;
        double A[P * P], B[P * P];
        shift_matrices<P>(a.basis, alpha, A, B);
        double* row = a.tab[sp] + ((long long)c * a.nlines + line) * NF;
        row[0] = (double)istar;
        row[1] = alpha;
#pragma unroll
        for (int i = 0; i < P * P; ++i) {
            row[2 + i] = A[i];
            row[2 + P * P + i] = B[i];
        }
        if (a.inline_sldg) {  // limiters.cpp:167-173
            double el[P], er[P];
            interval_moments<P>(a.basis, -alpha, 1.0 - alpha, el);
            interval_moments<P>(a.basis, 1.0 - alpha, 2.0 - alpha, er);
#pragma unroll
            for (int i = 0; i < P; ++i) {
                row[2 + 2 * P * P + i] = el[i];
                row[2 + 2 * P * P + P + i] = er[i];
            }
        }
    }
    if (g.nblocks == 1) return;
    // ghost-width checks (advection.cpp:181-190) and neighbour capacity
    // (adaptivity.cpp:179-183)
    int max_ghost = a.max_ghost;
    if (max_ghost == -2) {  // run.cpp:125-128
        const DevVGrid v0 = *a.vg[0], v1 = *a.vg[1];
        double r0 = v0.left + v0.cells * v0.dx, r1 = v1.left + v1.cells * v1.dx;
        double vmax_now = dmax2(r0, r1);
        double smm = dmin2(a.sqrt_mu[0], a.sqrt_mu[1]);
        max_ghost = (int)ceil(vmax_now * a.dt_auto / (smm * g.dx[0])) + 1;
    }
    const DevStatus* stc = a.st;
    long long step = a.step_index >= 0 ? a.step_index : stc->step;
    for (int b = 0; b < g.nblocks; ++b) {
        int istar = istar_c[g.cls[b]];
        int gl = b > 0 ? max(0, -istar) : 0;
        int gr = b + 1 < g.nblocks ? max(0, istar + 1) : 0;
        int need = max(gl, gr);
        if (max_ghost >= 0 && need > max_ghost) {
            raise_error(a.st, 2, 1, need, max_ghost, step);
            return;
        }
        for (int side = 0; side < 2; ++side) {
            int j = side == 0 ? gl : gr;
            if (j == 0) continue;
            bool left = side == 0;
            int nb = left ? b - 1 : b + 1;
            int iface = left ? g.start[b] : g.start[b] + g.cells[b];
            int lo, hi;
            if (g.dx[nb] == g.dx[b]) {
                lo = left ? iface - j : iface + (j - 1);
                hi = lo + 1;
            } else if (g.dx[nb] > g.dx[b]) {
                int m = (int)llround(g.dx[nb] / g.dx[b]);
                lo = left ? iface - 1 - (j - 1) / m : iface + (j - 1) / m;
                hi = lo + 1;
            } else {
                int m = (int)llround(g.dx[b] / g.dx[nb]);
                lo = left ? iface - j * m : iface + (j - 1) * m;
                hi = lo + m;
            }
            if (!(lo >= g.start[nb] && hi <= g.start[nb] + g.cells[nb])) {
                raise_error(a.st, 1, 2, j, 0, step);
                return;
            }
        }
    }
}

// Injection source half step of one x line (stepper.cpp:29-42, run.cpp:47-53):
// f += 0.5 half (S(t) + S(t + half)), S = H(t0 - t) blob(x, v) / t0, with the
// blob's x and v factors from host libm tables (source_kernel's arithmetic).
// t: the half step's start (state.time, or state.time + half for the second)
struct LineSource {
    bool on;
    double gv, w, t, t2, t0;
    const double* gx;
};
__device__ __forceinline__ LineSource line_source(const XSweepArgs& a, int sp, int line, int mode) {
    LineSource s{};
    if (a.src_mode != mode) return s;
    const double t = mode == 2 ? a.st->time + a.src_half : a.st->time;
    if (!(t <= a.src_t0)) return s;  // SourceTerm::active (stepper.hpp:19-21)
    const int lev = a.st->shrink_count[sp];
    if (lev >= kSourceLevels) {  // (as source_kernel)
        raise_error(a.st, 1, 7, lev, kSourceLevels, a.st->step);
        return s;
    }
    s.on = true;
    s.gv = a.src_gv[sp][(long long)lev * a.nlines + line];
    s.w = 0.5 * a.src_half;
    s.t = t;
    s.t2 = t + a.src_half;
    s.t0 = a.src_t0;
    s.gx = a.src_gx;
    return s;
}
// u (the P nodes of global x cell xc) += the source increment, bitwise source_kernel
template <int P>
__device__ __forceinline__ void add_source(const LineSource& s, int xc, double* u) {
#pragma unroll
    for (int n = 0; n < P; ++n) {
        const double blob = s.gx[xc * P + n] * s.gv;
        const double s1 = s.t > s.t0 ? 0.0 : blob / s.t0;
        const double s2 = s.t2 > s.t0 ? 0.0 : blob / s.t0;
        u[n] = u[n] + s.w * (s1 + s2);
    }
}

// ghost cell value for block-local cell s outside [0, cells_b) (fill_ghost,
// adaptivity.cpp:169-207): copy / coarse_to_fine piece / fine_to_coarse.
// src (the first injection source half step, if on): the reference adds it
// to every cell before the ghosts are transferred -- added to each
// neighbour cell value read, in the same rounding
template <int P, int MC = 0>
__device__ double x_fetch_outside(const Basis& basis, const Grid& g, const double* line, int b,
                                  int s, int n, const LineSource* src = nullptr) {
    const bool left = s < 0;
    int nb, j;
    if (left) {
        if (b == 0) return 0.0;
        nb = b - 1;
        j = -s;
    } else {
        if (b == g.nblocks - 1) return 0.0;
        nb = b + 1;
        j = s - g.cells[b] + 1;
    }
    const int iface = left ? g.start[b] : g.start[b] + g.cells[b];
    const int nb_begin = g.start[nb], nb_end = nb_begin + g.cells[nb];
    const bool ws = src != nullptr && src->on;
    if (g.dx[nb] == g.dx[b]) {
        int sc = left ? iface - j : iface + (j - 1);
        if (sc < nb_begin || sc >= nb_end) return 0.0;
        if (ws) {
            double u[P];
#pragma unroll
            for (int q = 0; q < P; ++q) u[q] = line[(long long)sc * P + q];
            add_source<P>(*src, sc, u);
            return u[n];
        }
        return line[(long long)sc * P + n];
    }
    if (g.dx[nb] > g.dx[b]) {
        const int m = MC > 0 ? MC : (int)llround(g.dx[nb] / g.dx[b]);
        int coarse = left ? iface - 1 - (j - 1) / m : iface + (j - 1) / m;
        if (coarse < nb_begin || coarse >= nb_end) return 0.0;
        int piece = left ? m - 1 - (j - 1) % m : (j - 1) % m;
        double u[P];
#pragma unroll
        for (int q = 0; q < P; ++q) u[q] = line[(long long)coarse * P + q];
        if (ws) add_source<P>(*src, coarse, u);
        return coarse_to_fine_node<P, MC>(basis, u, m, piece, n);
    }
    const int m = MC > 0 ? MC : (int)llround(g.dx[b] / g.dx[nb]);
    int lo = left ? iface - j * m : iface + (j - 1) * m;
    if (lo < nb_begin || lo + m > nb_end) return 0.0;
    if (ws) {  // fine_to_coarse_node's arithmetic on the cells with the source added
        double acc = 0.0;
#pragma unroll (MC > 0 ? MC : 1)
        for (int jj = 0; jj < m; ++jj) {
            double u[P];
#pragma unroll
            for (int q = 0; q < P; ++q) u[q] = line[(long long)(lo + jj) * P + q];
            add_source<P>(*src, lo + jj, u);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                double xi_c = (jj + basis.nodes[q]) / m;
                acc += basis.weights[q] / m * u[q] * lagrange<P>(basis, n, xi_c);
            }
        }
        return acc / basis.weights[n];
    }
    return fine_to_coarse_node<P, MC>(basis, line + (long long)lo * P, m, n);
}

// ---------------------------------------------------------------------------
// cp.async helpers (LDGSTS: global -> shared without a register round trip)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
// 8-byte async copy; valid == false zero-fills the destination (no global read)
__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(sdst)),
                 "l"(gsrc), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// fp64 tensor-core MMA (SASS DMMA): D(8x8) = A(8x4, row) * B(4x8, col) + C.
// Lane l holds A[l/4][l%4], B[l%4][l/4] and D[l/4][2(l%4) + {0,1}].
// ---------------------------------------------------------------------------
constexpr bool kXsweepDmma = false;  // see xsweep_kernel
constexpr bool kSeamAsync = true;  // MODE 3, k = 3: the producer computes each tile's seam cell one tile later
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// TMA bulk copy / mbarrier helpers (sm_90+; SASS UBLKCP / SYNCS)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    // the suspend-time hint lets a waiting warp sleep until the phase flips
    // instead of spinning on try_wait (a spinning producer warp stole ~8 % of
    // the x sweep's issue slots)
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "SK_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra SK_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(1000000)
        : "memory");
}
// the barrier's current phase also waits for this thread's prior cp.async
// copies (pending count +1 now, -1 when they land)
__device__ __forceinline__ void mbar_cp_async_arrive(unsigned long long* bar) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* sdst, const void* gsrc, unsigned bytes,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_1d(void* gdst, const void* ssrc, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void consumer_sync(int nthreads) {
    asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
}

// does block b's side (0 left, 1 right) border a block of another dx? Those
// ghost cells are projections (fill_ghost) and come from the xghost buffer
__device__ __forceinline__ bool xghost_side(const Grid& g, int b, int side) {
    const int nb = side == 0 ? b - 1 : b + 1;
    return nb >= 0 && nb < g.nblocks && g.dx[nb] != g.dx[b];
}

// K1a: 3-block ghost pre-pass, one warp per (species, line). A line's windows
// in block b span cells [istar_b, cells_b + istar_b + 1), so they reach
// -istar_b cells past the left edge (istar_b < 0) or istar_b + 1 past the
// right one. Those across a dx jump are evaluated here with x_fetch_outside's
// arithmetic (adaptivity.cpp:169-207), off the sweep producer's critical path:
// its fill is then an asynchronous copy, not a chain of dependent loads. The
// lanes load the blocks' shifts together and share the line's ghost values.
template <int P>
__global__ void __launch_bounds__(256, 4) xghost_kernel(const __grid_constant__ XSweepArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    const Grid& g = a.grid;
    const int w = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    const int nb = g.nblocks;
    if (w >= a.nspecies * a.nlines) return;
    const int line = w % a.nlines;
    const int sp = a.species0 + w / a.nlines;
    int ist = 0, cnt = 0, ratio = 0;
    if (lane < nb) {
        ist = (int)__ldg(a.tab[sp] + ((long long)g.cls[lane] * a.nlines + line) * xnf<P>());
        const int side = ist < 0 ? 0 : 1;
        if (xghost_side(g, lane, side)) {
            cnt = min(side == 0 ? -ist : ist + 1, a.ghost_cap) * P;
            const double d0 = g.dx[lane], d1 = g.dx[side == 0 ? lane - 1 : lane + 1];
            ratio = (int)llround(d1 > d0 ? d1 / d0 : d0 / d1);
        }
    }
    int pre[kMaxBlocks + 1], sgn[kMaxBlocks];
    pre[0] = 0;
#pragma unroll
    for (int b = 0; b < kMaxBlocks; ++b) {
        pre[b + 1] = pre[b] + __shfl_sync(0xffffffffu, cnt, b);
        sgn[b] = __shfl_sync(0xffffffffu, ist, b) < 0 ? 0 : 1;
    }
    const int total = pre[kMaxBlocks];
    if (total == 0) return;
    // one refinement ratio for all jumps (the 3-block mesh): unrolled loops
    const int rmax = __reduce_max_sync(0xffffffffu, ratio);
    const int rmin = (int)__reduce_min_sync(0xffffffffu, (unsigned)(ratio > 0 ? ratio : 0x7fffffff));
    const int m = rmax == rmin ? rmax : 0;
    const double* src = (field_flipped(a.flip[sp]) ? a.dst[sp] : a.src[sp]) + (long long)line * g.ncells * P;
    double* out = a.ghost + (long long)(sp * a.nlines + line) * nb * a.ghost_cap * P;
    const LineSource lsrc = line_source(a, sp, line, 1);  // (first injection half step, if fused)
    auto fill = [&](auto mc) {
        constexpr int MC = decltype(mc)::value;
        for (int e = lane; e < total; e += 32) {
            int b = 0, base = 0, sg = 0;  // last block starting at or before e (register selects)
#pragma unroll
            for (int k = 0; k < kMaxBlocks; ++k)
                if (e >= pre[k]) {
                    b = k;
                    base = pre[k];
                    sg = sgn[k];
                }
            const int l = e - base;
            const int j = l / P + 1, n = l - (l / P) * P;
            out[(long long)b * a.ghost_cap * P + l] =
                x_fetch_outside<P, MC>(a.basis, g, src, b, sg == 0 ? -j : g.cells[b] - 1 + j, n, &lsrc);
        }
    };
    switch (m) {  // the usual refinement ratios unrolled; others at run time
        case 2: fill(std::integral_constant<int, 2>{}); break;
        case 4: fill(std::integral_constant<int, 4>{}); break;
        case 8: fill(std::integral_constant<int, 8>{}); break;
        default: fill(std::integral_constant<int, 0>{}); break;
    }
}

// literature post-limiter indicator of one cell from its x or v stencil
// (post_summary / post_decide: one arithmetic for the stencil passes and the
// flags fused into the v sweep)
template <int P, bool FAST = false>
__device__ __forceinline__ bool post_flag(const PostCfg& cfg, const Basis& b, const double* um,
                                          const double* u0, const double* up) {
    return cfg.indicator == 1 ? post_flag_sum<P, FAST, 1>(b, cfg, um, u0, up)
                              : post_flag_sum<P, FAST, 2>(b, cfg, um, u0, up);
}

// the same with the indicator fixed at compile time (flag passes: straight-line
// code, so a thread's cells interleave)
template <int P, bool FAST, int IND>
__device__ __forceinline__ bool post_flag_t(const PostCfg& cfg, const Basis& b, const double* um,
                                            const double* u0, const double* up) {
    return post_flag_sum<P, FAST, IND>(b, cfg, um, u0, up);
}

// ---------------------------------------------------------------------------
// K1: x sweep -- warp-specialised TMA pipeline over tiles
//   tile = (species, x row, block, T cells); its source window is T+1 cells
//   that are contiguous in HBM. One producer warp streams windows (and the
//   tile's table row) into an S-stage smem ring with cp.async.bulk + mbarrier
//   transaction counts, and its lanes fill the window cells outside the
//   contiguous valid range (walls, 3-block ghosts, periodic wrap) before the
//   stage is armed; NC consumer warps compute two cells each (projection +
//   inline indicator in registers, matrices as smem broadcasts), hand the stage
//   back, queue troubled cells for the fixup and store each cell with one
//   256-bit store straight to HBM.
// ---------------------------------------------------------------------------
#ifndef SK_X_CPT4
#define SK_X_CPT4 2   // k = 3 x sweep: cells per consumer thread
#endif
#ifndef SK_X_STAGES
#define SK_X_STAGES 5  // x sweep input ring depth
#endif
#ifndef SK_X_MINB4
#define SK_X_MINB4 2  // k = 3 x sweep: resident CTAs per SM
#endif
template <int P>
struct XCfg {
    static constexpr int NC = 8;                    // consumer warps
    static constexpr int NT = NC * 32;
    static constexpr int CPT = P < 4 ? 2 : P == 4 ? SK_X_CPT4 : 1;
    static constexpr int MINB = P == 4 ? SK_X_MINB4 : 2;  // CTAs per SM the registers must allow
    static constexpr int T = CPT * NT;              // output cells per tile
    static constexpr int WIN = (((T + 1) * P + 4) + 1) / 2 * 2;  // window doubles (+ slack), even
    static constexpr int NF = xnf<P>();
    static constexpr int HDR = 6;                   // tile header (8 ints + weight) from the producer
    static constexpr int STAGE = ((WIN + NF + HDR + 1) / 2) * 2;
    static constexpr int S = SK_X_STAGES;           // input stages (outputs go straight to HBM)
    static constexpr int RACC = 0;                  // (fused-moment accumulators live in registers)
    static constexpr size_t SMEM = sizeof(double) * (size_t)(S * STAGE + RACC) + 8 * 2 * S + 8 * NC * kQCap;
    // MODE 3 (two half sweeps fused): 4 input stages, the intermediate line
    // segment, the clamped second-pass cells and two troubled-cell lists
    static constexpr int S3 = 4;
    static constexpr int WIN3 = (((T + 2) * P + 4) + 1) / 2 * 2;
    static constexpr int STAGE3 = ((WIN3 + NF + HDR + 1) / 2) * 2;
    static constexpr int SR = S3 + 1;  // MODE 3: seam-cell ring (producer -> consumers), slots
    static constexpr size_t SMEM3 = sizeof(double) * (size_t)(S3 * STAGE3 + 2 * (T + 1) * P + 2 * (NF + 2)) +
                                    8 * 2 * S3 + 8 * NC * kQCap + sizeof(int) * (2 * (T + 1) + 4) +
                                    sizeof(double) * SR * (P + 1) + 8 * SR;
    // MODE 1/2 (post-limiter flag passes): full T-cell tiles with a T + 2 cell window
    static constexpr size_t SMEM12 = sizeof(double) * (size_t)(S * STAGE3) + 8 * 2 * S + 8 * NC * kQCap;
    // MODE 4 / 5 (sweep + post-limiter flags): the tile's output summaries
    // [2 tile parities][m, a, b][T] after the queues
    static constexpr size_t SMEM45 = SMEM + sizeof(double) * 2 * 3 * T;
    template <int MODE>
    static constexpr size_t smem() {
        return MODE == 3 ? SMEM3 : (MODE == 1 || MODE == 2) ? SMEM12 : MODE >= 4 ? SMEM45 : SMEM;
    }
};

struct XTile {
    int sp, line, b, c0, nt;
};

__device__ __forceinline__ XTile decode_xtile(const XSweepArgs& a, int t, int T) {
    const int ntl = a.tile_start[a.grid.nblocks];
    XTile x;
    const int tl = t % ntl;
    const int rest = t / ntl;
    x.line = rest % a.nlines;
    x.sp = a.species0 + rest / a.nlines;
    int b = 0;
    while (tl >= a.tile_start[b + 1]) ++b;
    x.b = b;
    x.c0 = (tl - a.tile_start[b]) * T;
    x.nt = min(T, a.grid.cells[b] - x.c0);
    return x;
}

// valid contiguous block-local cell range that a bulk copy may fetch
__device__ __forceinline__ void xvalid_range(const XSweepArgs& a, int b, int& vlo, int& vhi) {
    const Grid& g = a.grid;
    vlo = 0;
    vhi = g.cells[b];
    if (a.periodic) return;
    if (b > 0 && g.dx[b - 1] == g.dx[b]) vlo = -g.cells[b - 1];
    if (b + 1 < g.nblocks && g.dx[b + 1] == g.dx[b]) vhi = g.cells[b] + g.cells[b + 1];
}

// P doubles of one cell from shared memory (16-byte vector loads for even P;
// the window origin is 16B-aligned whenever P is even)
template <int P>
__device__ __forceinline__ void lds_cell(const double* p, double* u) {
    if constexpr (P % 2 == 0) {
#pragma unroll
        for (int i = 0; i < P / 2; ++i) {
            const double2 v = reinterpret_cast<const double2*>(p)[i];
            u[2 * i] = v.x;
            u[2 * i + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int n = 0; n < P; ++n) u[n] = p[n];
    }
}
// the same for a warp reading 32 consecutive cells (lane L: cell base + L):
// for P = 4 lanes 4..7 of every 8 fetch their two 16-byte halves in swapped
// order, so each 128-bit load instruction hits all 32 banks once per 8 lanes
// (4 wavefronts instead of 8)
template <int P>
__device__ __forceinline__ void lds_cell_w(const double* p, double* u) {
    if constexpr (P == 4) {
        const int h = (threadIdx.x >> 2) & 1;
        const double2* q = reinterpret_cast<const double2*>(p);
        const double2 a = q[h], b = q[h ^ 1];
        u[0] = h ? b.x : a.x;
        u[1] = h ? b.y : a.y;
        u[2] = h ? a.x : b.x;
        u[3] = h ? a.y : b.y;
    } else {
        lds_cell<P>(p, u);
    }
}
template <int P>
__device__ __forceinline__ void sts_cell(double* p, const double* u) {
    if constexpr (P % 2 == 0) {
#pragma unroll
        for (int i = 0; i < P / 2; ++i)
            reinterpret_cast<double2*>(p)[i] = make_double2(u[2 * i], u[2 * i + 1]);
    } else {
#pragma unroll
        for (int n = 0; n < P; ++n) p[n] = u[n];
    }
}

// one output cell to global memory. k = 3: one 256-bit store per cell, so a
// warp writes 32 whole sectors per instruction (two 128-bit stores would each
// touch every sector half-full and double the L1 traffic)
template <int P>
__device__ __forceinline__ void stg_cell(double* dp, const double* o) {
    if constexpr (P == 4) {
        if ((((unsigned long long)dp) & 31) == 0) {
            asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dp), "d"(o[0]), "d"(o[1]), "d"(o[2]),
                         "d"(o[3])
                         : "memory");
            return;
        }
    } else if constexpr (P % 2 == 0) {
        if ((((unsigned long long)dp) & 15) == 0) {
#pragma unroll
            for (int i = 0; i < P / 2; ++i) reinterpret_cast<double2*>(dp)[i] = make_double2(o[2 * i], o[2 * i + 1]);
            return;
        }
    }
#pragma unroll
    for (int m = 0; m < P; ++m) dp[m] = o[m];
}

// MODE 0: the x sweep. MODE 1 / 2: the post-limiter flag pass in x with the
// minmod / mean-error indicator (limiters.cpp:254-345) on the same pipeline --
// window = the tile's cells and one neighbour on each side (tiles of T-1
// cells), no table row, the indicator per cell, flagged cells queued; in place
// (nothing stored). MODE 3: two consecutive x half sweeps fused (fused_tile).
// SRC (MODE 0): the injection source half step fused into this sweep, 1 on the
// cells read, 2 on the outputs (XSweepArgs::src_mode); a template argument so
// the plain sweeps carry none of its registers
template <int P, bool INLINE, bool RHO, bool FMA, int MODE = 0, int SRC = 0>
__global__ void __launch_bounds__((XCfg<P>::NC + 1) * 32, XCfg<P>::MINB)
    xsweep_kernel(const __grid_constant__ XSweepArgs a) {
    pdl_enter();
    using C = XCfg<P>;
    constexpr int S = MODE == 3 ? C::S3 : C::S;  // input stages
    // fast mode at k = 3: the projection and indicator on the fp64 tensor cores
    // (DMMA m8n8k4, two per 8 cells). Measured on B200 (C3): x sweeps 0.80 ->
    // 2.0 ms / 0.75 -> 1.44 ms, ~1.5 TFLOP/s effective -- the fp64 MMA path is
    // far slower than the DFMA pipe here, so it stays compiled out
    // (profiles/r02_dmma_xsweep.txt).
    constexpr bool kDmma = kXsweepDmma && P == 4 && FMA && MODE == 0 && C::T % (C::NC * 8) == 0;
    if (halted(a.st)) return;
    static_assert(MODE == 0 || MODE >= 3 || (!INLINE && !RHO), "the flag pass has no sweep limiter or moment");
    static_assert(MODE < 4 || (SRC == 0 && !INLINE), "fused post flags: no fused source, no inline limiter");
    // MODE 4 / 5: the x sweep deciding the post limiter's x flags (minmod /
    // mean error) of its own outputs -- summaries of the tile's cells in
    // shared memory, one consumer barrier, each cell's decision from its
    // neighbours' summaries; a tile's first and last cell (neighbour in
    // another tile or block) go to the list as candidates the fix kernel
    // re-decides from the field
    constexpr int PX = MODE >= 4 ? MODE - 3 : 0;
    // MODE 3: the seam cell from the producer (measured: k = 3 C5 -1.7 %, k = 2 +1.4 %)
    constexpr bool SA = kSeamAsync && MODE == 3 && P == 4;
    static_assert(MODE != 3 || C::T <= 2 * C::NT, "MODE 3: T + 1 intermediate cells over 3 passes of the consumers");
    if (a.gate && ((*a.gate != 0) != (a.gate_on != 0))) return;  // device-decided alternative
    // cells per tile: T in every mode -- the flag passes (one neighbour cell
    // each side) and MODE 3 (two shifts) stage a T + 2 cell window instead of
    // shortening the tile, so power-of-two blocks split into full tiles (511-
    // cell tiles left 1-2 cell remainder tiles in most lines)
    constexpr int TT = C::T;
    constexpr bool SWEEP = MODE == 0 || MODE >= 4;   // one plain half sweep per tile
    constexpr int WIN = SWEEP ? C::WIN : C::WIN3;
    constexpr int STAGE = SWEEP ? C::STAGE : C::STAGE3;
    constexpr int WX = SWEEP ? 1 : 2;                // window cells beyond the tile
    extern __shared__ __align__(128) double smem[];
    double* stages = smem;                                   // S x STAGE
    double* racc = smem + S * STAGE;                         // [T][P] this CTA's column (RHO)
    unsigned long long* full = reinterpret_cast<unsigned long long*>(racc + C::RACC);
    unsigned long long* empty = full + S;
    unsigned long long* wqueue = empty + S;  // [NC][kQCap] deferred entries per consumer warp
    // MODE 3, by tile parity: intermediate cells [2][T][P], the tile's table
    // row + moment weight [2][NF + 2] (read after the stage is handed back),
    // pass-1 troubled flags as tile epochs [2][T]
    [[maybe_unused]] double* mid = reinterpret_cast<double*>(wqueue + C::NC * kQCap);
    [[maybe_unused]] double* rowc = mid + 2 * (C::T + 1) * P;
    [[maybe_unused]] int* tl1 = reinterpret_cast<int*>(rowc + 2 * (C::NF + 2));
    [[maybe_unused]] double* psum = reinterpret_cast<double*>(wqueue + C::NC * kQCap);  // MODE 4 / 5
    // MODE 3: the seam ring -- each tile's last intermediate cell (the next tile's first), computed by the
    // producer from the landed stage one tile later, [SR][P + 1] (values, troubled flag) + one mbarrier each
    [[maybe_unused]] double* seamv = reinterpret_cast<double*>(tl1 + 2 * (C::T + 1) + 4);
    [[maybe_unused]] unsigned long long* seambar = reinterpret_cast<unsigned long long*>(seamv + C::SR * (P + 1));
    const Grid& g = a.grid;
    const int ntot = a.nspecies * a.nlines * a.tile_start[g.nblocks];
    const int G = gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int vb = blockIdx.x;
    const unsigned fm = (field_flipped(a.flip[0]) ? 1u : 0u) | (field_flipped(a.flip[1]) ? 2u : 0u);
    auto srcp = [&](int sp) -> const double* { return ((fm >> sp) & 1u) ? a.dst[sp] : a.src[sp]; };
    auto dstp = [&](int sp) -> double* { return ((fm >> sp) & 1u) ? const_cast<double*>(a.src[sp]) : a.dst[sp]; };

    if constexpr (MODE == 3)
        for (int i = threadIdx.x; i < 2 * (C::T + 1); i += blockDim.x) tl1[i] = -1;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], C::NC);
        }
        if constexpr (SA)
            for (int i = 0; i < C::SR; ++i) mbar_init(&seambar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (warp == C::NC) {
        // ---------------- producer warp ----------------
        // lane 0 streams windows with TMA (bulk copies cover only the 16-byte
        // aligned interior of the valid cells; lane 0 moves the <= 2 leftover
        // doubles itself), so no copy lands outside the valid cells and all 32
        // lanes can write the window cells outside that range -- walls, 3-block
        // ghosts, periodic wrap -- before the stage is armed: the consumers
        // never wait on each other for edge tiles
        constexpr bool PFILL = true;
        auto row_of = [&](const XTile& x) -> const double* {
            return a.tab[x.sp] + ((long long)g.cls[x.b] * a.nlines + x.line) * C::NF;
        };
        // (sign * w_vn) * dv of a v row: dv per species, loaded once
        [[maybe_unused]] double dvs[2] = {0.0, 0.0};
        if (RHO && lane == 0)
            for (int i = 0; i < 2; ++i)
                if (a.vg[i]) dvs[i] = a.vg[i]->dx;
        static_assert(PFILL, "the istar batches need all producer lanes");
        {
            // table shifts of this CTA's tiles in batches of 32, one per lane,
            // loaded a batch ahead: short tiles (3-block meshes) would otherwise
            // wait out one load latency each
            auto batch_istar = [&](int it0) -> int {
                const long long t = vb + (long long)(it0 + lane) * G;
                if constexpr (MODE == 1 || MODE == 2) return -1;  // window starts one cell left
                // MODE 3: two shifts, the window starts 2 i* cells away
                const int ist = t < ntot ? (int)__ldg(row_of(decode_xtile(a, (int)t, TT))) : 0;
                return MODE == 3 ? 2 * ist : ist;
            };
            int ist_cur = batch_istar(0);
            int ist_nxt = batch_istar(32);
            // MODE 3 (lane 0): the previous tile, whose seam cell is computed once this one is armed
            [[maybe_unused]] int p_it = -1, p_nt = 0, p_c0 = 0, p_b = 0, p_line = 0, p_istar = 0;
            [[maybe_unused]] auto seam_of = [&](int j, int jnt, int jc0, int jb, int jline, int jistar) {
                const int jstg = j % S;
                mbar_wait(&full[jstg], (j / S) & 1);  // (the stage is re-armed only by this warp, later)
                const double* pst = stages + jstg * STAGE;
                const double* prow = pst + WIN;
                const long long jeg = (long long)jline * g.ncells * P + ((long long)g.start[jb] + jc0 + jistar) * P;
                const double* pwin = pst + 2 + (int)(jeg & 1);
                const long long gm = (long long)g.start[jb] + jc0 + jistar / 2 + jnt;
                double o[P];
                bool tr = false;
                if (gm < 0 || gm >= g.ncells) {
#pragma unroll
                    for (int n = 0; n < P; ++n) o[n] = 0.0;
                } else {  // pass 1's arithmetic on the same window values and table row
                    double ul[P], ur[P];
                    lds_cell<P>(pwin + jnt * P, ul);
                    lds_cell<P>(pwin + (jnt + 1) * P, ur);
                    project_cell_f<P, FMA>(prow + 2, prow + 2 + P * P, ul, ur, o);
                    if constexpr (INLINE) {
                        const ThrCut pcut{a.threshold, a.thr_hi, a.thr_lo};
                        tr = inline_indicator_m<P, FMA>(pcut, prow + 2 + 2 * P * P, prow + 2 + 2 * P * P + P,
                                                        mean_f<P, FMA>(a.basis, ul), mean_f<P, FMA>(a.basis, ur), o);
                    }
                }
                double* sv = seamv + (j % C::SR) * (P + 1);
#pragma unroll
                for (int n = 0; n < P; ++n) sv[n] = o[n];
                sv[P] = tr ? 1.0 : 0.0;
                mbar_arrive(&seambar[j % C::SR]);
            };
            int it = 0;
            for (int t = vb; t < ntot; t += G, ++it) {
                const int stg = it % S;
                if ((it & 31) == 0 && it > 0) {
                    ist_cur = ist_nxt;
                    ist_nxt = batch_istar(it + 32);
                }
                const XTile x = decode_xtile(a, t, TT);
                const int istar = __shfl_sync(0xffffffffu, ist_cur, it & 31);
                mbar_wait(&empty[stg], ((it / S) & 1) ^ 1);
                const int s0 = x.c0 + istar;
                int vlo, vhi;
                xvalid_range(a, x.b, vlo, vhi);
                const int clo = max(s0, vlo), chi = min(s0 + x.nt + WX, vhi);
                double* st = stages + stg * STAGE;
                // element parity of window cell s0 in HBM decides the smem origin
                const long long lbase = (long long)x.line * g.ncells * P;
                const long long eg = lbase + ((long long)g.start[x.b] + s0) * P;
                const int woff = (int)(eg & 1);
                if constexpr (PFILL) {
                    if (clo > s0 || chi < s0 + x.nt + WX) {
                        const double* src = srcp(x.sp) + lbase;
                        double* w = st + 2 + woff;
                        const int cells_b = g.cells[x.b];
                        const int nlo = (max(clo, s0) - s0) * P;
                        const int nhi0 = (min(max(chi, s0), s0 + x.nt + WX) - s0) * P;
                        const int nfill = nlo + ((x.nt + WX) * P - nhi0);
                        const double* gh = a.ghost ? a.ghost + ((long long)(x.sp * a.nlines + x.line) * g.nblocks + x.b) *
                                                                   a.ghost_cap * P
                                                   : nullptr;
                        bool anyc = false;  // async fills: tracked by the stage barrier
                        for (int f = lane; f < nfill; f += 32) {
                            const int e = f < nlo ? f : nhi0 + (f - nlo);
                            const int wc = e / P, n = e - (e / P) * P;
                            const int sc = s0 + wc;
                            if (a.periodic) {
                                const int ss = ((sc % cells_b) + cells_b) % cells_b;
                                cp_async8(w + e, src + (long long)(g.start[x.b] + ss) * P + n, true);
                                anyc = true;
                                continue;
                            }
                            const int side = sc < 0 ? 0 : 1;
                            const int j = side == 0 ? -sc : sc - cells_b + 1;
                            if (gh && j <= a.ghost_cap && xghost_side(g, x.b, side)) {
                                cp_async8(w + e, gh + (j - 1) * P + n, true);
                                anyc = true;
                            } else {
                                if constexpr (SRC == 1) {
                                    const LineSource lsrc = line_source(a, x.sp, x.line, 1);
                                    w[e] = x_fetch_outside<P>(a.basis, g, src, x.b, sc, n, &lsrc);
                                } else {
                                    w[e] = x_fetch_outside<P>(a.basis, g, src, x.b, sc, n);
                                }
                            }
                        }
                        if (anyc) mbar_cp_async_arrive(&full[stg]);
                    }
                    __syncwarp();  // fills ordered before lane 0's arrive (release)
                    if (lane != 0) continue;
                }
                // decoded tile for the consumers (released by the arrive below)
                int* hdr = reinterpret_cast<int*>(st + WIN + C::NF);
                hdr[0] = x.sp;
                hdr[1] = x.line;
                hdr[2] = x.b;
                hdr[3] = x.c0;
                hdr[4] = x.nt;
                hdr[5] = s0;
                hdr[6] = clo;
                hdr[7] = chi;
                if (RHO) {  // (sign * w_vn) * dv of this v row (poisson.cpp:207)
                    const int vn = x.line - (x.line / P) * P;
                    reinterpret_cast<double*>(hdr)[4] = a.charge_w[x.sp] * a.basis.weights[vn] * dvs[x.sp];
                }
                unsigned bytes = (MODE == 1 || MODE == 2) ? 0u : C::NF * 8;
                long long ga = 0, gb = 0;
                if (chi > clo) {
                    // element g of the line sits at st + 2 + woff + (g - eg): same
                    // parity in HBM and shared memory
                    const long long g0 = eg + (long long)(clo - s0) * P;
                    const long long g1 = eg + (long long)(chi - s0) * P;
                    ga = (g0 + 1) & ~1LL;
                    gb = g1 & ~1LL;
                    if (gb < ga) gb = ga;
                    double* wbase = st + 2 + woff - eg;
                    const double* gsrc = srcp(x.sp);
                    bool any = false;  // leftovers: async, completion tracked by the stage barrier
                    for (long long g = g0; g < ga && g < g1; ++g, any = true) cp_async8(wbase + g, gsrc + g, true);
                    for (long long g = gb > g0 ? gb : g0; g < g1; ++g, any = true) cp_async8(wbase + g, gsrc + g, true);
                    if (any) mbar_cp_async_arrive(&full[stg]);
                    bytes += (unsigned)(gb - ga) * 8;
                }
                mbar_expect_tx(&full[stg], bytes);
                if constexpr (SWEEP || MODE == 3) tma_load_1d(st + WIN, row_of(x), C::NF * 8, &full[stg]);
                if (gb > ga) {
                    double* dst = st + 2 + woff + (ga - eg);
                    tma_load_1d(dst, srcp(x.sp) + ga, (unsigned)(gb - ga) * 8, &full[stg]);
                }
                if constexpr (SA) {
                    if (p_it >= 0) seam_of(p_it, p_nt, p_c0, p_b, p_line, p_istar);
                    p_it = it;
                    p_nt = x.nt;
                    p_c0 = x.c0;
                    p_b = x.b;
                    p_line = x.line;
                    p_istar = istar;
                }
            }
            if constexpr (SA)
                if (lane == 0 && p_it >= 0) seam_of(p_it, p_nt, p_c0, p_b, p_line, p_istar);
        }
        return;
    }

    // ---------------- consumer warps ----------------
    const int tid = threadIdx.x;
    [[maybe_unused]] const ThrCut cut{a.threshold, a.thr_hi, a.thr_lo};
    unsigned nt_t = 0, nt_c = 0, nt_o = 0;
    bool bad = false;
    unsigned long long* wq = wqueue + warp * kQCap;
    int wq_n = 0;
    [[maybe_unused]] unsigned f3[2][3] = {{0, 0, 0}, {0, 0, 0}};  // MODE 3: in-kernel clamp counters
    // fused moment: the grid is a multiple of the tiles per line, so this CTA
    // always sees the same tile column and each thread the same cells -- the
    // accumulators live in registers
    // (DMMA path: [8-cell group][2 nodes] per lane, see below)
    constexpr int RA = kDmma ? C::T / C::NC / 8 : C::CPT, RB = kDmma ? 1 : P;
    [[maybe_unused]] double rreg[RHO ? RA : 1][RHO ? RB : 1];
    if constexpr (RHO)
#pragma unroll
        for (int cc = 0; cc < RA; ++cc)
#pragma unroll
            for (int m = 0; m < RB; ++m) rreg[cc][m] = 0.0;
    (void)racc;
    int rcol_nt = 0, rcol_base = 0;
    int it = 0;
    for (int t = vb; t < ntot; t += G, ++it) {
        const int stg = it % S;
        mbar_wait(&full[stg], (it / S) & 1);
        double* st = stages + stg * STAGE;
        const double* row = st + WIN;
        const int* hdr = reinterpret_cast<const int*>(st + WIN + C::NF);
        const int sp = hdr[0], line = hdr[1], b = hdr[2], c0 = hdr[3], nt = hdr[4];
        const int s0 = hdr[5], clo = hdr[6], chi = hdr[7];
        const int cells_b = g.cells[b];
        if constexpr (RHO) {
            rcol_nt = nt;
            rcol_base = g.start[b] + c0;
        }
        const long long lbase = (long long)line * g.ncells * P;
        const long long eg = lbase + ((long long)g.start[b] + s0) * P;
        const double* win = st + 2 + (int)(eg & 1);  // window cell w, node n at win[w*P+n]
        // cells per thread this warp has in this tile (warp-uniform): short
        // tiles (3-block meshes) skip the idle slots instead of recomputing
        const int ncc = min(C::CPT, nt > warp * 32 + C::NT ? 2 : (nt > warp * 32 ? 1 : 0));
        // MODE 3: step n's second x half sweep and step n+1's first one in one
        // pass over the tile (stepper.cpp:90 then :74, same tau and v grid, so
        // the same table row): the window holds the 2 i*-shifted sources and
        // the intermediate cells stay in shared memory. No clamp runs here:
        // pass 2 reads the unclamped intermediate, and every output cell a
        // troubled cell can reach (troubled itself, or next to a troubled
        // intermediate cell) is queued; xfix2_kernel recomputes those cells
        // with both clamps from the intact sources (the arithmetic of the
        // unfused sweep + fixup) and corrects the fused moment exactly. One
        // consumer barrier per tile (intermediate, flags and row copy are
        // double-buffered by tile parity).
        [[maybe_unused]] auto fused_tile = [&]() {
            const int istar = (int)row[0];
            const int pb = it & 1;
            double* midb = mid + pb * (C::T + 1) * P;
            int* t1 = tl1 + pb * (C::T + 1);           // pass-1 troubled flags: tile epoch
            double* rc = rowc + pb * (C::NF + 2);
            const int gbase = g.start[b] + c0;  // global cell of the tile's first output
            const int nmid = nt + 1;            // intermediate cells the outputs read
            if (tid < C::NF) rc[tid] = row[tid];
            if (tid == C::NF) rc[C::NF] = RHO ? reinterpret_cast<const double*>(hdr)[4] : 0.0;
            // ---- pass 1: intermediate cells gbase + i* + m, m < nmid (<= T + 1); the last
            // one (m = nt) comes from the producer's seam ring (kSeamAsync) ----
            constexpr int SEAMP = SA ? 1 : 0;
#pragma unroll
            for (int cc = 0; cc < 3 - SEAMP; ++cc) {
                const int m = tid + cc * C::NT;
                if (m < nmid - SEAMP) {
                    const int gm = gbase + istar + m;
                    double o[P];
                    if (gm < 0 || gm >= g.ncells) {
#pragma unroll
                        for (int n = 0; n < P; ++n) o[n] = 0.0;  // zero inflow (advection.cpp:89-93)
                    } else {
                        double ul[P], ur[P];
                        lds_cell_w<P>(win + m * P, ul);
                        lds_cell_w<P>(win + (m + 1) * P, ur);
                        project_cell_f<P, FMA>(row + 2, row + 2 + P * P, ul, ur, o);
                        if constexpr (INLINE)
                            if (inline_indicator_m<P, FMA>(cut, row + 2 + 2 * P * P, row + 2 + 2 * P * P + P,
                                                           mean_f<P, FMA>(a.basis, ul),
                                                           mean_f<P, FMA>(a.basis, ur), o)) {
                                t1[m] = it;
                                if (m < nt) f3[sp & 1][0] += 1;  // seam cell m = nt: the next tile's m = 0
                            }
                    }
                    sts_cell<P>(midb + m * P, o);
                    if (a.check_finite) bad |= !all_finite<P>(o);  // step n's end state (stepper.cpp:99-102)
                }
            }
            if constexpr (SA)
                if (tid == 0) {
                    mbar_wait(&seambar[it % C::SR], (it / C::SR) & 1);
                    const double* sv = seamv + (it % C::SR) * (P + 1);
                    double o[P];
#pragma unroll
                    for (int n = 0; n < P; ++n) o[n] = sv[n];
                    if (sv[P] != 0.0) t1[nt] = it;
                    sts_cell<P>(midb + nt * P, o);
                    if (a.check_finite) bad |= !all_finite<P>(o);
                }
            // the window is consumed
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
            consumer_sync(C::NT);
            // ---- pass 2: output cells c < nt from intermediate cells c, c+1 ----
            const double* Am = rc + 2;
            const double* Bm = rc + 2 + P * P;
            [[maybe_unused]] const double* ext = rc + 2 + 2 * P * P;
            const double wdv = rc[C::NF];
            double* dline = dstp(sp) + lbase + (long long)gbase * P;
            [[maybe_unused]] bool fix[2];
            [[maybe_unused]] unsigned long long entry[2];
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int c = tid + cc * C::NT;
                fix[cc] = false;
                entry[cc] = ((unsigned long long)(sp & 1) << 63) | ((unsigned long long)line << 32) |
                            (unsigned)(gbase + c);
                if (c < nt) {
                    double ul[P], ur[P], o[P];
                    lds_cell_w<P>(midb + c * P, ul);
                    lds_cell_w<P>(midb + (c + 1) * P, ur);
                    project_cell_f<P, FMA>(Am, Bm, ul, ur, o);
                    if constexpr (INLINE)
                        fix[cc] = t1[c] == it || t1[c + 1] == it ||
                                  inline_indicator_m<P, FMA>(cut, ext, ext + P, mean_f<P, FMA>(a.basis, ul),
                                                             mean_f<P, FMA>(a.basis, ur), o);
                    if constexpr (RHO) {  // step n+1's charge density (poisson.cpp:207)
#pragma unroll
                        for (int m = 0; m < P; ++m) rreg[cc][m] = madd<FMA>(rreg[cc][m], wdv, o[m]);
                    }
                    stg_cell<P>(dline + (long long)c * P, o);
                }
            }
            if constexpr (INLINE) wq_push<2>(wq, wq_n, a.fix_count, a.fix_cap, a.fix_list, fix, entry);
        };
        if constexpr (MODE == 3) {
            fused_tile();
            continue;
        }
        if constexpr (MODE == 1 || MODE == 2) {
            // post-limiter flags: cell c's stencil is window cells c, c+1, c+2
            auto flags = [&](auto ncc_c) {
                constexpr int NCC = decltype(ncc_c)::value;
                bool tr[NCC];
                unsigned long long entry[NCC];
#pragma unroll
                for (int cc = 0; cc < NCC; ++cc) {
                    const int c = tid + cc * C::NT;
                    tr[cc] = false;
                    entry[cc] = ((unsigned long long)(sp & 1) << 63) | ((unsigned long long)line << 32) |
                                (unsigned)(g.start[b] + c0 + c);
                    if (c < nt) {
                        double um[P], u0[P], up[P];
                        lds_cell<P>(win + c * P, um);
                        lds_cell<P>(win + (c + 1) * P, u0);
                        lds_cell<P>(win + (c + 2) * P, up);
                        tr[cc] = post_flag_t<P, FMA, MODE>(a.post, a.basis, um, u0, up);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[stg]);
                wq_push<NCC>(wq, wq_n, a.fix_count, a.fix_cap, a.fix_list, tr, entry);
            };
            if (C::CPT == 2 && ncc == 2) {
                flags(std::integral_constant<int, C::CPT>{});
            } else if (ncc >= 1) {
                flags(std::integral_constant<int, 1>{});
            } else {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[stg]);
            }
            continue;
        }
        if constexpr (kDmma) {
            // Fast mode, k = 3: the tile as 8-cell groups on the fp64 tensor
            // cores. Per cell the 8 inputs (left source cell, right source
            // cell) map to 8 outputs with one 8x8 matrix constant along the
            // line: the projection (advection.cpp:95-101) and, for the inline
            // indicator, the two source means and the two extension moments of
            // the projected cell (limiters.cpp:175-188), which are linear in
            // the inputs too. Two m8n8k4 MMAs per 8 cells replace ~80 DFMA and
            // shared loads per cell; quad lanes 0/1 hold nodes 0-1 / 2-3 of a
            // cell, lanes 2/3 its means / extension moments.
            const int kq = lane & 3, nq = lane >> 2;
            const double* Am = row + 2;
            const double* Bm = row + 2 + P * P;
            double b0, b1;  // W[kq][nq], W[4 + kq][nq]
            if (nq < P) {
                b0 = Am[nq * P + kq];
                b1 = Bm[nq * P + kq];
            } else if (nq == P) {
                b0 = a.basis.weights[kq];
                b1 = 0.0;
            } else if (nq == P + 1) {
                b0 = 0.0;
                b1 = a.basis.weights[kq];
            } else {
                const double* e = row + 2 + 2 * P * P + (nq == P + 2 ? 0 : P);
                b0 = 0.0;
                b1 = 0.0;
                if (INLINE)
#pragma unroll
                    for (int m = 0; m < P; ++m) {
                        b0 = fma(e[m], Am[m * P + kq], b0);
                        b1 = fma(e[m], Bm[m * P + kq], b1);
                    }
            }
            constexpr int G = C::T / C::NC / 8;  // 8-cell groups per warp
            const int wbase = warp * (C::T / C::NC);
            double fa[G][2];  // A fragments: this lane's input of the left / right source cell
#pragma unroll
            for (int gi = 0; gi < G; ++gi) {
                const int c = wbase + 8 * gi;
                fa[gi][0] = fa[gi][1] = 0.0;
                if (c < nt) {  // warp-uniform
                    fa[gi][0] = win[(c + nq) * P + kq];
                    fa[gi][1] = win[(c + 1 + nq) * P + kq];
                }
            }
            // the window stage is consumed
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
            double wdv = 0.0;
            if constexpr (RHO) wdv = reinterpret_cast<const double*>(hdr)[4];
            double* dline = dstp(sp) + lbase + (long long)(g.start[b] + c0) * P;
#pragma unroll
            for (int gi = 0; gi < G; ++gi) {
                if (wbase + 8 * gi >= nt) break;  // warp-uniform
                double d0 = 0.0, d1 = 0.0;
                dmma884(d0, d1, fa[gi][0], b0);
                dmma884(d0, d1, fa[gi][1], b1);
                const int cell = wbase + 8 * gi + nq;
                const bool valid = cell < nt;
                if constexpr (INLINE) {
                    // lane kq = 2 takes the extension moments from its neighbour
                    const double ex = __shfl_down_sync(0xffffffffu, d0, 1);
                    const double ey = __shfl_down_sync(0xffffffffu, d1, 1);
                    const bool tr[1] = {kq == 2 && valid &&
                                        over_threshold(fabs(ex - d0) + fabs(ey - d1), dmax2(fabs(d0), fabs(d1)), cut)};
                    const unsigned long long entry[1] = {((unsigned long long)(sp & 1) << 63) |
                                                         ((unsigned long long)line << 32) |
                                                         (unsigned)(g.start[b] + c0 + cell)};
                    wq_push<1>(wq, wq_n, a.fix_count, a.fix_cap, a.fix_list, tr, entry);
                }
                if constexpr (RHO) {
                    // node kq of the cell to lane kq: one accumulator per lane
                    const int src = (lane & ~3) | (kq >> 1);
                    const double x0 = __shfl_sync(0xffffffffu, d0, src), x1 = __shfl_sync(0xffffffffu, d1, src);
                    if (valid) rreg[gi][0] = fma(wdv, (kq & 1) ? x1 : x0, rreg[gi][0]);
                }
                if (kq < 2 && valid) {
                    if (a.check_finite) bad |= !(isfinite(d0) && isfinite(d1));
                    *reinterpret_cast<double2*>(dline + (long long)cell * P + 2 * kq) = make_double2(d0, d1);
                }
            }
            continue;
        }
        if constexpr (!kDmma) {
        auto cells = [&](auto ncc_c) {
            constexpr int NCC = decltype(ncc_c)::value;
            double ul[NCC][P], ur[NCC][P], o[NCC][P];
#pragma unroll
            for (int cc = 0; cc < NCC; ++cc) {
                const int c = min(tid + cc * C::NT, nt - 1);
                lds_cell_w<P>(win + c * P, ul[cc]);
                lds_cell_w<P>(win + (c + 1) * P, ur[cc]);
            }
            if constexpr (SRC == 1) {  // the step's first source half step, on the cells as read
                const LineSource src = line_source(a, sp, line, 1);
                if (src.on) {
                    // raw line cells only (ghosts across a dx jump arrive with it)
                    int vlo, vhi;
                    xvalid_range(a, b, vlo, vhi);
#pragma unroll
                    for (int cc = 0; cc < NCC; ++cc) {
                        const int wl = s0 + min(tid + cc * C::NT, nt - 1);  // block-local window cell c
                        if (wl >= vlo && wl < vhi) add_source<P>(src, g.start[b] + wl, ul[cc]);
                        if (wl + 1 >= vlo && wl + 1 < vhi) add_source<P>(src, g.start[b] + wl + 1, ur[cc]);
                    }
                }
            }
            // advection.cpp:95-101, both cells share each broadcast matrix load
#pragma unroll
            for (int m = 0; m < P; ++m) {
                double acc[NCC];
#pragma unroll
                for (int cc = 0; cc < NCC; ++cc) acc[cc] = 0.0;
                double am[P], bm[P];
                lds_cell<P>(row + 2 + m * P, am);
                lds_cell<P>(row + 2 + P * P + m * P, bm);
#pragma unroll
                for (int j = 0; j < P; ++j) {
#pragma unroll
                    for (int cc = 0; cc < NCC; ++cc) {
                        if constexpr (FMA)
                            acc[cc] = fma(bm[j], ur[cc][j], fma(am[j], ul[cc][j], acc[cc]));
                        else
                            acc[cc] += am[j] * ul[cc][j] + bm[j] * ur[cc][j];
                    }
                }
#pragma unroll
                for (int cc = 0; cc < NCC; ++cc) o[cc][m] = acc[cc];
            }
            double wdv = 0.0;
            if constexpr (RHO) wdv = reinterpret_cast<const double*>(hdr)[4];
            [[maybe_unused]] bool tr[NCC];
            [[maybe_unused]] unsigned long long entry[NCC];
#pragma unroll
            for (int cc = 0; cc < NCC; ++cc) {
                const int c = tid + cc * C::NT;
                if constexpr (INLINE) {
                    const double* ext = row + 2 + 2 * P * P;
                    tr[cc] = c < nt && inline_indicator_m<P, FMA>(cut, ext, ext + P, mean_f<P, FMA>(a.basis, ul[cc]),
                                                                  mean_f<P, FMA>(a.basis, ur[cc]), o[cc]);
                    entry[cc] = ((unsigned long long)(sp & 1) << 63) | ((unsigned long long)line << 32) |
                                (unsigned)(g.start[b] + c0 + c);
                }
                if (c < nt) {
                    if constexpr (RHO) {
#pragma unroll
                        for (int m = 0; m < P; ++m) rreg[cc][m] = madd<FMA>(rreg[cc][m], wdv, o[cc][m]);
                    }
                }
            }
            if (a.check_finite) {  // stepper.cpp:99-102, only on the step's last sweep
#pragma unroll
                for (int cc = 0; cc < NCC; ++cc)
                    if (tid + cc * C::NT < nt) bad |= !all_finite<P>(o[cc]);
            }
            // the window stage is consumed (all that follows is in registers):
            // hand it back before the queue atomics and the stores
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
            // troubled cells are queued for the fixup kernel (on overflow it rescans)
            if constexpr (INLINE) wq_push<NCC>(wq, wq_n, a.fix_count, a.fix_cap, a.fix_list, tr, entry);
            double* dline = dstp(sp) + lbase + (long long)(g.start[b] + c0) * P;
            if constexpr (SRC == 2) {  // the step's second source half step, on the outputs; a troubled
                const LineSource src = line_source(a, sp, line, 2);  // cell gets it after its clamp (xfix)
                if (src.on)
#pragma unroll
                    for (int cc = 0; cc < NCC; ++cc) {
                        const int c = tid + cc * C::NT;
                        bool troubled = false;
                        if constexpr (INLINE) troubled = tr[cc];
                        if (c < nt && !troubled) add_source<P>(src, g.start[b] + c0 + c, o[cc]);
                    }
            }
#pragma unroll
            for (int cc = 0; cc < NCC; ++cc) {
                const int c = tid + cc * C::NT;
                if (c < nt) {
                    // straight to HBM: the warp's lanes cover 32 contiguous cells
                    stg_cell<P>(dline + (long long)c * P, o[cc]);
                }
            }
            if constexpr (PX != 0) {  // the post limiter's summaries of the stored cells
                double* q = psum + (it & 1) * 3 * C::T;
#pragma unroll
                for (int cc = 0; cc < NCC; ++cc) {
                    const int c = tid + cc * C::NT;
                    if (c < nt) {
                        const PostSum ps = post_summary<P, FMA, PX>(a.basis, a.post, o[cc]);
                        q[c] = ps.m;
                        q[C::T + c] = ps.a;
                        q[2 * C::T + c] = ps.b;
                    }
                }
            }
        };
        // (the fused-moment variant keeps one body: its register accumulators
        // leave no room for a second)
        if ((C::CPT == 2 && ncc == 2) || (RHO && ncc >= 1)) {
            cells(std::integral_constant<int, C::CPT>{});
        } else if (!RHO && ncc >= 1) {
            cells(std::integral_constant<int, 1>{});
        } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
        }
        if constexpr (PX != 0) {
            // every summary of the tile is in (double-buffered by tile parity,
            // so one barrier per tile orders both the reads and the next writes)
            consumer_sync(C::NT);
            const double* q = psum + (it & 1) * 3 * C::T;
            auto sum_at = [&](int c) { return PostSum{q[c], q[C::T + c], q[2 * C::T + c]}; };
            bool tr[C::CPT];
            unsigned long long entry[C::CPT];
#pragma unroll
            for (int cc = 0; cc < C::CPT; ++cc) {
                const int c = tid + cc * C::NT;
                tr[cc] = false;
                entry[cc] = ((unsigned long long)(sp & 1) << 63) | ((unsigned long long)line << 32) |
                            (unsigned)(g.start[b] + c0 + c);
                if (c < nt) {
                    if (c == 0 || c == nt - 1) {  // neighbour outside the tile: a candidate
                        tr[cc] = true;
                        entry[cc] |= kPostCandidate;
                    } else {
                        tr[cc] = post_decide<FMA, PX>(a.post, sum_at(c - 1), sum_at(c), sum_at(c + 1));
                    }
                }
            }
            wq_push<C::CPT>(wq, wq_n, a.fix_count, a.fix_cap, a.fix_list, tr, entry);
        }
        }
    }
    if (RHO && rcol_nt > 0) {
        // this CTA always saw the same tile column (grid is a multiple of the
        // tiles per line): one partial row per (column, CTA group)
        const int ntl = a.tile_start[g.nblocks];
        double* prow = a.rho_partial + (long long)(vb / ntl) * g.ncells * P;
        if constexpr (kDmma) {
            const int kq = lane & 3, nq = lane >> 2, wbase = warp * (C::T / C::NC);
#pragma unroll
            for (int gi = 0; gi < RA; ++gi) {
                const int c = wbase + 8 * gi + nq;
                if (c < rcol_nt) prow[(long long)(rcol_base + c) * P + kq] = rreg[gi][0];
            }
        } else {
#pragma unroll
            for (int cc = 0; cc < C::CPT; ++cc) {
                const int c = tid + cc * C::NT;
                if (c < rcol_nt) {
#pragma unroll
                    for (int n = 0; n < P; ++n) prow[(long long)(rcol_base + c) * P + n] = rreg[cc][n];
                }
            }
        }
    }
    if constexpr (INLINE || MODE == 1 || MODE == 2 || PX != 0) wq_flush(wq, wq_n, a.fix_count, a.fix_cap, a.fix_list);
    if constexpr (INLINE && MODE == 3) {
        count_flags(a.st->stats[0], f3[0][0], f3[0][1], f3[0][2]);
        count_flags(a.st->stats[1], f3[1][0], f3[1][1], f3[1][2]);
    } else if constexpr (INLINE) {
        count_flags(a.st->stats[a.nspecies == 1 ? a.species0 : 0], nt_t, nt_c, nt_o);
    }
    if (a.check_finite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&a.st->nonfinite, 1);
}

// ---------------------------------------------------------------------------
// v tables and K2: v sweep
// ---------------------------------------------------------------------------
template <int P>
__global__ void vtab_kernel(const __grid_constant__ VTabArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    const int xd = blockIdx.x * blockDim.x + threadIdx.x;
    if (xd >= a.nxd) return;
    const int sp = a.species0 + blockIdx.y;
    const double speed = a.charge[sp] * a.E[xd] / a.sqrt_mu[sp];  // advection.cpp:226
    const double dv = a.vg[sp]->dx;
    int istar;
    double alpha;
    decompose_shift(speed, a.tau, dv, istar, alpha);
    double A[P * P], B[P * P];
    shift_matrices<P>(a.basis, alpha, A, B);
    if (a.halo_need) {  // the shard's exchange width is sized from this (sk_state_vhalo_need)
        atomicMax(a.halo_need, max(-istar, istar + 1));
    } else if ((a.halo_lo >= 0 && -istar > a.halo_lo) || (a.halo_hi >= 0 && istar + 1 > a.halo_hi)) {
        raise_error(a.st, 2, 5, max(-istar, istar + 1), max(a.halo_lo, a.halo_hi), a.st->step);
    }
    double* t = a.tab[sp];
    const int n = a.nxd;
    t[xd] = (double)istar;
    t[n + xd] = alpha;
#pragma unroll
    for (int i = 0; i < P * P; ++i) {
        t[(long long)(2 + i) * n + xd] = A[i];
        t[(long long)(2 + P * P + i) * n + xd] = B[i];
    }
    if (a.inline_sldg) {
        double el[P], er[P];
        interval_moments<P>(a.basis, -alpha, 1.0 - alpha, el);
        interval_moments<P>(a.basis, 1.0 - alpha, 2.0 - alpha, er);
#pragma unroll
        for (int i = 0; i < P; ++i) {
            t[(long long)(2 + 2 * P * P + i) * n + xd] = el[i];
            t[(long long)(2 + 2 * P * P + P + i) * n + xd] = er[i];
        }
    }
}

template <int P>
__device__ __forceinline__ void vload(const double* f, long long ld, int xd, int s, int lo, int hi,
                                      int periodic, int ncell, double* u) {
    if (periodic) s = ((s % ncell) + ncell) % ncell;
    if (s >= lo && s < hi) {
        const double* p = f + (long long)s * P * ld + xd;
#pragma unroll
        for (int n = 0; n < P; ++n) u[n] = __ldg(p + n * ld);
    } else {
#pragma unroll
        for (int n = 0; n < P; ++n) u[n] = 0.0;
    }
}

// One thread per x dof walks kVChunk v cells. Source cells stream through a
// per-thread R-deep cp.async ring in shared memory ([slot][node][thread], so
// consecutive threads hit consecutive banks), keeping R*P loads in flight per
// thread without spending registers on them.
template <int P>
__host__ __device__ constexpr int vring() { return P <= 4 ? 8 : 4; }

// issue the P node rows of source cell s (pointer gp = its row-0 address) into
// a ring slot; cells outside [lo, hi) are zero-filled without a global read
template <int P>
__device__ __forceinline__ void vissue(const double* gp, long long ld, bool valid, double* slot) {
#pragma unroll
    for (int n = 0; n < P; ++n) cp_async8(slot + n * kVThreads, valid ? gp + n * ld : gp, valid);
}

// PV (post limiter V fused, 1 minmod / 2 mean error): every output cell's
// summary (post_summary) is formed from the registers it is stored from, and
// cell j's flag is decided once cell j + 1's is known -- the stencil the post
// pass would read back. A chunk also computes (without storing) its two
// neighbour cells, so no flag waits for another block; outside [0, n) the
// stencil sees the walls' zero cells like the post pass.
template <int P, bool INLINE, bool PERIODIC, bool FMA, int PV = 0>
__global__ void __launch_bounds__(kVThreads) vsweep_kernel(const __grid_constant__ VSweepArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    constexpr int R = vring<P>();
    static_assert(kVChunk % R == 0, "chunk must be a multiple of the ring depth");
    __shared__ double ring[R * P * kVThreads];
    // PV: flagged cells staged per warp (post limiters flag ~5-10 % of the cells)
    __shared__ unsigned long long wqueue[PV ? kVThreads / 32 : 1][PV ? kQCap : 1];
    [[maybe_unused]] unsigned long long* wq = wqueue[PV ? threadIdx.x >> 5 : 0];
    [[maybe_unused]] int wq_n = 0;
    // chunk_major: v chunks are the fastest grid dimension, so the blocks that
    // share an x range (and its table rows, ~1/3 of the bytes a chunk reads)
    // run back to back -- chosen when the tables would not stay in L2
    const int xb = a.chunk_major ? blockIdx.y : blockIdx.x;
    const int jb = a.chunk0 + (a.chunk_major ? blockIdx.x : blockIdx.y);
    const int xd = xb * blockDim.x + threadIdx.x;
    const int sp = a.species0 + blockIdx.z;
    const int j0 = jb * kVChunk;
    const int j1 = min(j0 + kVChunk, a.n);
    static_assert(PV == 0 || (!INLINE && !PERIODIC), "fused post flags: no inline limiter, walls");
    const int js = PV && j0 > 0 ? j0 - 1 : j0;   // outputs computed: [js, je) (PV: the neighbours too)
    const int je = PV && j1 < a.n ? j1 + 1 : j1;
    bool bad = false;
    double* my = ring + threadIdx.x;
    [[maybe_unused]] const unsigned members = __ballot_sync(0xffffffffu, xd < a.nxd);
    if (xd < a.nxd) {
        const double* t = a.tab[sp];
        const int nx = a.nxd;
        const int istar = (int)t[xd];
        const bool fl = field_flipped(a.flip[sp]);
        const double* f = (fl ? a.dst[sp] : a.src[sp]) + xd;
        const long long ld = a.ld;
        const long long cstride = (long long)P * ld;  // one v cell
        const int lo = -a.gl, hi = a.n + a.gr;
        const int ncells = (je - js) + 1;              // source cells of this run
        // next source cell to issue and its row pointer (non-periodic: linear walk)
        int s_iss = js + istar;
        auto src_of = [&](int s) -> const double* {
            if constexpr (PERIODIC) s = ((s % a.n) + a.n) % a.n;
            return f + (long long)s * cstride;
        };
        auto ok = [&](int s) -> bool {
            if constexpr (PERIODIC) return true;
            return (unsigned)(s - lo) < (unsigned)(hi - lo);
        };
        const double* g_iss = src_of(s_iss);
#pragma unroll
        for (int c = 0; c < R - 1; ++c) {  // prologue: cells 0..R-2
            if (c < ncells) vissue<P>(g_iss, ld, ok(s_iss), my + c * P * kVThreads);
            cp_commit();
            ++s_iss;
            g_iss = PERIODIC ? src_of(s_iss) : g_iss + cstride;
        }
        const double alpha = t[nx + xd];
        double A[P * P], B[P * P], el[INLINE ? P : 1], er[INLINE ? P : 1];
#pragma unroll
        for (int i = 0; i < P * P; ++i) {
            A[i] = t[(long long)(2 + i) * nx + xd];
            B[i] = t[(long long)(2 + P * P + i) * nx + xd];
        }
        if constexpr (INLINE) {
#pragma unroll
            for (int i = 0; i < P; ++i) {
                el[i] = t[(long long)(2 + 2 * P * P + i) * nx + xd];
                er[i] = t[(long long)(2 + 2 * P * P + P + i) * nx + xd];
            }
        }
        (void)alpha;
        double ul[P], ur[P];
        cp_wait<R - 2>();
#pragma unroll
        for (int n = 0; n < P; ++n) ul[n] = my[n * kVThreads];
        [[maybe_unused]] const ThrCut cut{a.threshold, a.thr_hi, a.thr_lo};
        [[maybe_unused]] double mean_l = INLINE ? mean_f<P, FMA>(a.basis, ul) : 0.0;  // carried along the walk
        const bool check = a.check_finite;
        if (R - 1 < ncells) vissue<P>(g_iss, ld, ok(s_iss), my + (R - 1) * P * kVThreads);
        cp_commit();
        ++s_iss;
        g_iss = PERIODIC ? src_of(s_iss) : g_iss + cstride;
        double* op = (fl ? const_cast<double*>(a.src[sp]) : a.dst[sp]) + xd + (long long)js * cstride;
        [[maybe_unused]] PostSum pa{0.0, 0.0, 0.0}, pb{0.0, 0.0, 0.0};  // cells j - 2, j - 1 (walls: zero)
        constexpr int NOUT = kVChunk + (PV ? 2 : 0);
        for (int jb = 0; jb < NOUT; jb += R) {
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const int jj = jb + u;  // output cell js + jj; ur = ring cell jj+1
                if (js + jj < je) {
                    cp_wait<R - 2>();
                    const double* sl = my + ((u + 1) % R) * P * kVThreads;
#pragma unroll
                    for (int n = 0; n < P; ++n) ur[n] = sl[n * kVThreads];
                    if (jj + R < ncells) vissue<P>(g_iss, ld, ok(s_iss), my + u * P * kVThreads);
                    cp_commit();
                    ++s_iss;
                    g_iss = PERIODIC ? src_of(s_iss) : g_iss + cstride;
                    double o[P];
                    project_cell_f<P, FMA>(A, B, ul, ur, o);
                    if constexpr (INLINE) {
                        const double mean_r = mean_f<P, FMA>(a.basis, ur);
                        const bool tr[1] = {inline_indicator_m<P, FMA>(cut, el, er, mean_l, mean_r, o)};
                        const unsigned long long entry[1] = {((unsigned long long)(sp & 1) << 63) |
                                                             ((unsigned long long)(j0 + jj) << 32) |
                                                             (unsigned)xd};
                        defer_push_n<1>(a.fix_count, a.fix_cap, a.fix_list, tr, entry, members);
                        mean_l = mean_r;
                    }
                    bool store = true;
                    if constexpr (PV != 0) {
                        const int j = js + jj;
                        const PostSum sn = post_summary<P, FMA, PV>(a.basis, a.post, o);
                        if (j - 1 >= j0) {  // cell j - 1's stencil is complete
                            const bool tr[1] = {post_decide<FMA, PV>(a.post, pa, pb, sn)};
                            const unsigned long long entry[1] = {((unsigned long long)(sp & 1) << 63) |
                                                                 ((unsigned long long)(j - 1) << 32) |
                                                                 (unsigned)xd};
                            wq_push<1>(wq, wq_n, a.fix_count, a.fix_cap, a.fix_list, tr, entry, members);
                        }
                        pa = pb;
                        pb = sn;
                        store = j >= j0 && j < j1;
                    }
                    if (store) {
                        if (check) bad |= !all_finite<P>(o);
#pragma unroll
                        for (int m = 0; m < P; ++m) op[m * ld] = o[m];
                    }
                    op += cstride;
#pragma unroll
                    for (int n = 0; n < P; ++n) ul[n] = ur[n];
                }
            }
        }
        if constexpr (PV != 0)
            if (je == j1 && j1 - 1 >= j0) {  // the last cell against the upper wall's zero cell
                const bool tr[1] = {post_decide<FMA, PV>(a.post, pa, pb, PostSum{0.0, 0.0, 0.0})};
                const unsigned long long entry[1] = {((unsigned long long)(sp & 1) << 63) |
                                                     ((unsigned long long)(j1 - 1) << 32) | (unsigned)xd};
                wq_push<1>(wq, wq_n, a.fix_count, a.fix_cap, a.fix_list, tr, entry, members);
            }
        if constexpr (PV != 0) wq_flush(wq, wq_n, a.fix_count, a.fix_cap, a.fix_list, members);
        cp_wait<0>();
    }
    if (a.check_finite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
        atomicOr(&a.st->nonfinite, 1);
}

// ---------------------------------------------------------------------------
// deferred theta clamp of troubled cells (limiters.cpp:191-215), one thread per
// queued cell. The sweep's source buffer is intact (ping-pong), so ul/ur are
// re-read exactly as the sweep saw them and the result is bitwise the same.
// ---------------------------------------------------------------------------
// Clamp corrections of the fused charge density as exact integers: d splits
// exactly into hi = RN(d 2^30) 2^-30 and lo = d - hi (|lo| <= 2^-31), summed
// as int64 at scales 2^30 and 2^76. Integer sums do not depend on the order
// of the atomics, so rho is deterministic; the range is |sum| < 2^33 per x
// dof and the dropped part of lo is < 2^-77 per correction.
__device__ __forceinline__ void rho_corr_add(unsigned long long* base, long long lo_off, long long i, double d) {
    const double hi = rint(d * 0x1p30) * 0x1p-30;
    const double lo = d - hi;
    atomicAdd(base + i, (unsigned long long)__double2ll_rn(hi * 0x1p30));
    atomicAdd(base + lo_off + i, (unsigned long long)__double2ll_rn(lo * 0x1p76));
}
__device__ __forceinline__ double rho_corr_value(unsigned long long hi, unsigned long long lo) {
    return (double)(long long)hi * 0x1p-30 + (double)(long long)lo * 0x1p-76;
}

// the sweep's troubled decision, recomputed by a fixup rescan with the same
// arithmetic the sweep used
template <int P>
__device__ __forceinline__ bool rescan_indicator(const Basis& b, double thr, int fma, const double* el,
                                                 const double* er, const double* ul, const double* ur,
                                                 const double* o) {
    const ThrCut cut = make_thr_cut(thr);
    if constexpr (kHasFmaDev<P>)
        if (fma)
            return inline_indicator_m<P, true>(cut, el, er, mean_f<P, true>(b, ul), mean_f<P, true>(b, ur), o);
    return inline_indicator_m<P, false>(cut, el, er, mean<P>(b, ul), mean<P>(b, ur), o);
}

// out-of-line ghost fetch for the fixup kernels (keeps their code small)
template <int P>
__device__ __noinline__ double x_fetch_outside_ool(const Basis& basis, const Grid& g, const double* line,
                                                   int b, int s, int n, const LineSource* src = nullptr) {
    return x_fetch_outside<P>(basis, g, line, b, s, n, src);
}

template <int P, bool FMA>
__device__ __forceinline__ void xfix_cell(const XSweepArgs& a, int sp, int line, int cell, bool rescan,
                                       unsigned* ct, unsigned* cc, unsigned* co) {
    constexpr int NF = xnf<P>();
    const Grid& g = a.grid;
    int b = 0;
    while (cell >= g.start[b + 1]) ++b;
    const int local = cell - g.start[b];
    const double* row = a.tab[sp] + ((long long)g.cls[b] * a.nlines + line) * NF;
    const int istar = (int)row[0];
    const double alpha = row[1];
    const long long lbase = (long long)line * g.ncells * P;
    const bool flipped = field_flipped(a.flip[sp]);
    const double* src = (flipped ? a.dst[sp] : a.src[sp]) + lbase;
    // the sweep read its sources with the first injection half step added (if fused)
    const LineSource src1 = line_source(a, sp, line, 1);
    double uu[2][P];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int s = local + istar + h;
        if (a.periodic || (s >= 0 && s < g.cells[b])) {
            const int ss = a.periodic ? ((s % g.cells[b]) + g.cells[b]) % g.cells[b] : s;
            const double* cp = src + (long long)(g.start[b] + ss) * P;
#pragma unroll
            for (int q = 0; q < P; ++q) uu[h][q] = cp[q];
            if (src1.on) add_source<P>(src1, g.start[b] + ss, uu[h]);
        } else {
#pragma unroll
            for (int q = 0; q < P; ++q) uu[h][q] = x_fetch_outside_ool<P>(a.basis, g, src, b, s, q, &src1);
        }
    }
    const LineSource src2 = line_source(a, sp, line, 2);
    double* up = (flipped ? const_cast<double*>(a.src[sp]) : a.dst[sp]) + lbase + (long long)cell * P;
    double o[P];
#pragma unroll
    for (int q = 0; q < P; ++q) o[q] = up[q];
    if (rescan && src2.on)  // untroubled cells hold projection + source: recompute the projection
        project_cell_f<P, FMA>(row + 2, row + 2 + P * P, uu[0], uu[1], o);  // (the sweep's arithmetic)
    if (rescan && !rescan_indicator<P>(a.basis, a.threshold, a.fma, row + 2 + 2 * P * P,
                                       row + 2 + 2 * P * P + P, uu[0], uu[1], o))
        return;
    double o0[P];
#pragma unroll
    for (int q = 0; q < P; ++q) o0[q] = o[q];
    const int fl = inline_clamp_f<P, FMA>(a.basis, alpha, uu[0], uu[1], o);
    double os[P];  // stored: with the second source half step after the clamp
#pragma unroll
    for (int q = 0; q < P; ++q) os[q] = o[q];
    if (src2.on) add_source<P>(src2, cell, os);
#pragma unroll
    for (int q = 0; q < P; ++q) up[q] = os[q];
    if (a.rho_fuse && (fl & 2)) {  // the fused moment summed the unclamped values
        const int vn = line - (line / P) * P;
        const double wdv = a.charge_w[sp] * a.basis.weights[vn] * a.vg[sp]->dx;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const double d = wdv * o[q] - wdv * o0[q];
            // spread over copies by v row: clamped cells of many rows share an x dof
            rho_corr_add(a.rho_corr + (long long)(line % kRhoCorrCopies) * a.grid.ncells * P,
                         (long long)kRhoCorrCopies * a.grid.ncells * P, (long long)cell * P + q, d);
        }
    }
    ct[sp] += fl & 1;
    cc[sp] += (fl >> 1) & 1;
    co[sp] += (fl >> 2) & 1;
}

template <int P, bool FMA>
__global__ void __launch_bounds__(128, 8) xfix_kernel(const __grid_constant__ XSweepArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    if (a.gate && ((*a.gate != 0) != (a.gate_on != 0))) return;
    const unsigned cnt = *a.fix_count;
    unsigned ct[2] = {0, 0}, cc[2] = {0, 0}, co[2] = {0, 0};
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    // list mode, or (list overflowed) a rescan of every cell of the sweep; one
    // loop so the clamp is inlined once (twice made the kernel fetch-bound)
    const bool rescan = cnt > a.fix_cap;
    const long long n = rescan ? (long long)a.nspecies * a.nlines * a.grid.ncells : (long long)cnt;
    for (long long i = i0; i < n; i += stride) {
        int sp, line, cell;
        if (!rescan) {
            const unsigned long long e = a.fix_list[i];
            sp = (int)(e >> 63);
            line = (int)((e >> 32) & 0x7fffffffu);
            cell = (int)(e & 0xffffffffu);
        } else {
            cell = (int)(i % a.grid.ncells);
            const long long r = i / a.grid.ncells;
            sp = a.species0 + (int)(r / a.nlines);
            line = (int)(r % a.nlines);
        }
        xfix_cell<P, FMA>(a, sp, line, cell, rescan, ct, cc, co);
    }
    block_count_flags(a.st, ct, cc, co);
}

// Fixup of a fused step boundary (xsweep_kernel MODE 3): output cell `cell`
// of line `line` recomputed from the fused sweep's intact sources with both
// half sweeps' clamps -- intermediate cells cell + i* and cell + i* + 1 (each
// clamped when troubled, limiters.cpp:191-215), then the output (clamped when
// troubled) -- i.e. what the unfused x sweep + xfix and x sweep + xfix give.
// The fused moment summed the stored value: the difference goes into the
// exact integer corrections. Counters: the output's flags, and the clamp
// flags of its left intermediate cell (each troubled intermediate cell is the
// left one of exactly one queued output; the fused kernel counted it troubled).
template <int P, bool FMA>
__device__ __forceinline__ void xfix2_cell(const XSweepArgs& a, int sp, int line, int cell, unsigned* ct,
                                           unsigned* cc, unsigned* co) {
    constexpr int NF = xnf<P>();
    const Grid& g = a.grid;
    int b = 0;
    while (cell >= g.start[b + 1]) ++b;
    const double* row = a.tab[sp] + ((long long)g.cls[b] * a.nlines + line) * NF;
    const int istar = (int)row[0];
    const double alpha = row[1];
    const double* A = row + 2;
    const double* B = row + 2 + P * P;
    const double* el = row + 2 + 2 * P * P;
    const double* er = el + P;
    const ThrCut cut{a.threshold, a.thr_hi, a.thr_lo};
    const long long lbase = (long long)line * g.ncells * P;
    const bool flipped = field_flipped(a.flip[sp]);
    const double* src = (flipped ? a.dst[sp] : a.src[sp]) + lbase;
    double* out = (flipped ? const_cast<double*>(a.src[sp]) : a.dst[sp]) + lbase + (long long)cell * P;
    auto load = [&](int k, double* u) {
        if (k >= 0 && k < g.ncells) {
#pragma unroll
            for (int q = 0; q < P; ++q) u[q] = src[(long long)k * P + q];
        } else {
#pragma unroll
            for (int q = 0; q < P; ++q) u[q] = 0.0;  // zero inflow
        }
    };
    double mid[2][P];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int k = cell + istar + j;
        if (k < 0 || k >= g.ncells) {
#pragma unroll
            for (int q = 0; q < P; ++q) mid[j][q] = 0.0;
            continue;
        }
        double ul[P], ur[P];
        load(k + istar, ul);
        load(k + istar + 1, ur);
        project_cell_f<P, FMA>(A, B, ul, ur, mid[j]);
        if (inline_indicator_m<P, FMA>(cut, el, er, mean_f<P, FMA>(a.basis, ul), mean_f<P, FMA>(a.basis, ur),
                                       mid[j])) {
            const int fl = inline_clamp_f<P, FMA>(a.basis, alpha, ul, ur, mid[j]);
            if (j == 0) {
                cc[sp] += (fl >> 1) & 1;
                co[sp] += (fl >> 2) & 1;
            }
        }
    }
    double o[P];
    project_cell_f<P, FMA>(A, B, mid[0], mid[1], o);
    if (inline_indicator_m<P, FMA>(cut, el, er, mean_f<P, FMA>(a.basis, mid[0]), mean_f<P, FMA>(a.basis, mid[1]),
                                   o)) {
        const int fl = inline_clamp_f<P, FMA>(a.basis, alpha, mid[0], mid[1], o);
        ct[sp] += fl & 1;
        cc[sp] += (fl >> 1) & 1;
        co[sp] += (fl >> 2) & 1;
    }
    const int vn = line - (line / P) * P;
    const double wdv = a.charge_w[sp] * a.basis.weights[vn] * a.vg[sp]->dx;
#pragma unroll
    for (int q = 0; q < P; ++q) {
        const double old = out[q];
        out[q] = o[q];
        const double d = wdv * o[q] - wdv * old;
        if (d != 0.0)
            rho_corr_add(a.rho_corr + (long long)(line % kRhoCorrCopies) * a.grid.ncells * P,
                         (long long)kRhoCorrCopies * a.grid.ncells * P, (long long)cell * P + q, d);
    }
}

template <int P, bool FMA>
__global__ void __launch_bounds__(128, 4) xfix2_kernel(const __grid_constant__ XSweepArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    if (a.gate && ((*a.gate != 0) != (a.gate_on != 0))) return;
    const unsigned cnt = *a.fix_count;
    unsigned ct[2] = {0, 0}, cc[2] = {0, 0}, co[2] = {0, 0};
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    // list mode, or (the list overflowed) every output cell
    const bool rescan = cnt > a.fix_cap;
    const long long n = rescan ? (long long)a.nspecies * a.nlines * a.grid.ncells : (long long)cnt;
    for (long long i = i0; i < n; i += stride) {
        int sp, line, cell;
        if (!rescan) {
            const unsigned long long e = a.fix_list[i];
            sp = (int)(e >> 63);
            line = (int)((e >> 32) & 0x7fffffffu);
            cell = (int)(e & 0xffffffffu);
        } else {
            cell = (int)(i % a.grid.ncells);
            const long long r = i / a.grid.ncells;
            sp = a.species0 + (int)(r / a.nlines);
            line = (int)(r % a.nlines);
        }
        xfix2_cell<P, FMA>(a, sp, line, cell, ct, cc, co);
    }
    block_count_flags(a.st, ct, cc, co);
}

template <int P, bool FMA>
__device__ __forceinline__ void vfix_cell(const VSweepArgs& a, int sp, int j, int xd, bool rescan,
                                       unsigned* ct, unsigned* cc, unsigned* co) {
    const double* t = a.tab[sp];
    const int nx = a.nxd;
    const int istar = (int)t[xd];
    const double alpha = t[nx + xd];
    double ul[P], ur[P], o[P];
    const bool flipped = field_flipped(a.flip[sp]);
    const double* src = flipped ? a.dst[sp] : a.src[sp];
    vload<P>(src, a.ld, xd, j + istar, -a.gl, a.n + a.gr, a.periodic, a.n, ul);
    vload<P>(src, a.ld, xd, j + istar + 1, -a.gl, a.n + a.gr, a.periodic, a.n, ur);
    double* op = (flipped ? const_cast<double*>(a.src[sp]) : a.dst[sp]) + (long long)j * P * a.ld + xd;
#pragma unroll
    for (int m = 0; m < P; ++m) o[m] = op[m * a.ld];
    if (rescan) {
        double el[P], er[P];
#pragma unroll
        for (int i = 0; i < P; ++i) {
            el[i] = t[(long long)(2 + 2 * P * P + i) * nx + xd];
            er[i] = t[(long long)(2 + 2 * P * P + P + i) * nx + xd];
        }
        if (!rescan_indicator<P>(a.basis, a.threshold, a.fma, el, er, ul, ur, o)) return;
    }
    const int fl = inline_clamp_f<P, FMA>(a.basis, alpha, ul, ur, o);
#pragma unroll
    for (int m = 0; m < P; ++m) op[m * a.ld] = o[m];
    ct[sp] += fl & 1;
    cc[sp] += (fl >> 1) & 1;
    co[sp] += (fl >> 2) & 1;
}

template <int P, bool FMA>
__global__ void __launch_bounds__(128, 8) vfix_kernel(const __grid_constant__ VSweepArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    const unsigned cnt = *a.fix_count;
    unsigned ct[2] = {0, 0}, cc[2] = {0, 0}, co[2] = {0, 0};
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool rescan = cnt > a.fix_cap;  // see xfix_kernel
    const long long n = rescan ? (long long)a.nspecies * a.n * a.nxd : (long long)cnt;
    for (long long i = i0; i < n; i += stride) {
        int sp, j, xd;
        if (!rescan) {
            const unsigned long long e = a.fix_list[i];
            sp = (int)(e >> 63);
            j = (int)((e >> 32) & 0x7fffffffu);
            xd = (int)(e & 0xffffffffu);
        } else {
            xd = (int)(i % a.nxd);
            const long long r = i / a.nxd;
            sp = a.species0 + (int)(r / a.n);
            j = (int)(r % a.n);
        }
        vfix_cell<P, FMA>(a, sp, j, xd, rescan, ct, cc, co);
    }
    block_count_flags(a.st, ct, cc, co);
}

// ---------------------------------------------------------------------------
// K4: charge density (poisson.cpp:194-216), deterministic two-pass
// ---------------------------------------------------------------------------
template <int P>
__global__ void rho_partial_kernel(const __grid_constant__ RhoArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    const int xd = blockIdx.x * blockDim.x + threadIdx.x;
    if (xd >= a.nxd) return;
    const int sp = blockIdx.z;
    const int chunk = blockIdx.y;
    const double dv = a.vg[sp]->dx;
    const int r0 = chunk * a.rows_per_chunk, r1 = min(r0 + a.rows_per_chunk, a.nrows);
    const double* f = (field_flipped(a.flip[sp]) ? a.alt[sp] : a.f[sp]) + xd;
    double acc = 0.0;
    for (int r = r0; r < r1; ++r) {
        const int vn = r - (r / P) * P;
        acc += a.basis.weights[vn] * dv * __ldg(f + (long long)r * a.ld);
    }
    a.partial[((long long)sp * a.nchunks + chunk) * a.nxd + xd] = acc;
}

__global__ void rho_reduce_kernel(const __grid_constant__ RhoArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    const int xd = blockIdx.x * blockDim.x + threadIdx.x;
    if (xd >= a.nxd) return;
    double acc = 0.0;
    for (int c = 0; c < a.nchunks; ++c) acc += a.partial[((long long)1 * a.nchunks + c) * a.nxd + xd];
    for (int c = 0; c < a.nchunks; ++c) acc -= a.partial[((long long)0 * a.nchunks + c) * a.nxd + xd];
    a.rho[xd] = acc;
}

// ---------------------------------------------------------------------------
// Poisson: replay of the host block-cyclic-reduction plan (single CTA, one
// thread per block row per level, PS = k+2 compile-time)
// ---------------------------------------------------------------------------
// Load value of row i = c*PS + m for the BCR replay: stage 0/1 the SIPG load
// (poisson.cpp:135-149); stage 2 the residual b_i - (A x)_i of the stage-1
// solution x (band rows i-kd .. i+kd, j ascending).
template <int PS>
__device__ __forceinline__ double poisson_load(const PoissonDev& pd, int stage, const double* rho, int c, int m) {
    constexpr int KD = 2 * PS - 1, LD = KD + 1;
    const int k = PS - 2;
    double val = 0.0;
#pragma unroll
    for (int n = 0; n <= k; ++n) val += pd.interp[m * (k + 1) + n] * rho[c * (k + 1) + n];
    double b = pd.ws[m] * pd.h[c] * val;
    if (stage == 2) {
        const int i = c * PS + m, n = pd.ncells * PS;
        double ax = 0.0;
#pragma unroll
        for (int d = -KD; d <= KD; ++d) {
            const int j = i + d;
            if (j < 0 || j >= n) continue;
            const double aij = d < 0 ? pd.band[(long long)j * LD - d] : pd.band[(long long)i * LD + d];
            ax += aij * pd.ir_x[j];
        }
        b -= ax;
    }
    return b;
}

// M is stored transposed over rows: entry (m,n) of row r at M[(m*PS+n)*rows + r]
template <int PS>
__device__ __forceinline__ void matvec_t(const double* __restrict__ M, int rows, int r,
                                         const double* x, double* v, double sign) {
#pragma unroll
    for (int m = 0; m < PS; ++m) {
        double acc = 0.0;
#pragma unroll
        for (int n = 0; n < PS; ++n) acc += M[(long long)(m * PS + n) * rows + r] * x[n];
        v[m] += sign * acc;
    }
}

template <int PS>
__global__ void __launch_bounds__(1024) poisson_kernel(const __grid_constant__ PoissonDev pd, int stage,
                                                       const double* __restrict__ rho,
                                                       double* __restrict__ E,
                                                       double* __restrict__ phi) {
    pdl_enter();
    if (halted(pd.st)) return;
    constexpr int pp = PS * PS;
    const int k = PS - 2, N = pd.ncells;
    const int tid = threadIdx.x, nth = blockDim.x;
    // vectors are SoA per level: b_l[m*Nl + q]
    double* b0 = pd.bws;
    for (int i = tid; i < N * PS; i += nth) {  // load vector (poisson.cpp:135-149) / residual
        const int m = i / N, c = i - (i / N) * N;
        b0[i] = poisson_load<PS>(pd, stage, rho, c, m);
    }
    __syncthreads();
    // reduction: b'_r = b_q + alpha_q b_{q-1} + gamma_q b_{q+1}, q = 2r;
    // one thread per (row, component): coalesced over rows, short chains
    for (int l = 0; l + 1 < pd.nlevels; ++l) {
        const int Nl = pd.level_n[l], Nn = pd.level_n[l + 1];
        const double* bl = pd.bws + pd.level_off[l] * PS;
        double* bn = pd.bws + pd.level_off[l + 1] * PS;
        const double* Al = pd.AlphaT + pd.keep_off[l] * pp;
        const double* Gl = pd.GammaT + pd.keep_off[l] * pp;
        for (int i = tid; i < Nn * PS; i += nth) {
            const int m = i / Nn, r = i - (i / Nn) * Nn, q = 2 * r;
            double v = bl[m * Nl + q];
            if (q - 1 >= 0) {
                double acc = 0.0;
#pragma unroll
                for (int n = 0; n < PS; ++n) acc += Al[(long long)(m * PS + n) * Nn + r] * bl[n * Nl + q - 1];
                v += acc;
            }
            if (q + 1 < Nl) {
                double acc = 0.0;
#pragma unroll
                for (int n = 0; n < PS; ++n) acc += Gl[(long long)(m * PS + n) * Nn + r] * bl[n * Nl + q + 1];
                v += acc;
            }
            bn[m * Nn + r] = v;
        }
        __syncthreads();
    }
    {
        const int L = pd.nlevels - 1;
        const double* bt = pd.bws + pd.level_off[L] * PS;
        double* xt = pd.xws + pd.level_off[L] * PS;
        if (tid < PS) {
            double acc = 0.0;
#pragma unroll
            for (int n = 0; n < PS; ++n) acc += pd.DinvTop[tid * PS + n] * bt[n];
            xt[tid] = acc;
        }
        __syncthreads();
    }
    // back substitution: even rows inherit, odd rows x = Dinv (b - Lo x_{q-1} - Up x_{q+1})
    for (int l = pd.nlevels - 2; l >= 0; --l) {
        const int Nl = pd.level_n[l], Nn = pd.level_n[l + 1], No = Nl / 2;
        double* bl = pd.bws + pd.level_off[l] * PS;
        double* xl = pd.xws + pd.level_off[l] * PS;
        const double* xn = pd.xws + pd.level_off[l + 1] * PS;
        const double* Lo = pd.LoT + pd.odd_off[l] * pp;
        const double* Up = pd.UpT + pd.odd_off[l] * pp;
        const double* Di = pd.DinvT + pd.odd_off[l] * pp;
        // residual t = b - Lo x_{q-1} - Up x_{q+1} of odd rows, in place in b;
        // even rows copy from the coarser level
        for (int i = tid; i < Nl * PS; i += nth) {
            const int m = i / Nl, q = i - (i / Nl) * Nl;
            if ((q & 1) == 0) {
                xl[m * Nl + q] = xn[m * Nn + q / 2];
            } else {
                const int o = q >> 1;
                double t = bl[m * Nl + q];
                double acc = 0.0;
#pragma unroll
                for (int n = 0; n < PS; ++n) acc += Lo[(long long)(m * PS + n) * No + o] * xn[n * Nn + o];
                t -= acc;
                if (q + 1 < Nl) {
                    acc = 0.0;
#pragma unroll
                    for (int n = 0; n < PS; ++n) acc += Up[(long long)(m * PS + n) * No + o] * xn[n * Nn + o + 1];
                    t -= acc;
                }
                bl[m * Nl + q] = t;
            }
        }
        __syncthreads();
        for (int i = tid; i < No * PS; i += nth) {
            const int m = i / No, o = i - (i / No) * No, q = 2 * o + 1;
            double acc = 0.0;
#pragma unroll
            for (int n = 0; n < PS; ++n) acc += Di[(long long)(m * PS + n) * No + o] * bl[n * Nl + q];
            xl[m * Nl + q] = acc;
        }
        __syncthreads();
    }
    const double* x0 = pd.xws;
    if (stage == 1) {  // first solve of the refinement: keep x, no E yet
        for (int i = tid; i < N * PS; i += nth) {
            const int c = i / PS, m = i - (i / PS) * PS;
            pd.ir_x[i] = x0[m * N + c];
        }
        return;
    }
    auto xv = [&](int n, int c) { return stage == 2 ? pd.ir_x[c * PS + n] + x0[n * N + c] : x0[n * N + c]; };
    if (phi)
        for (int i = tid; i < N * PS; i += nth) {
            const int c = i / PS, m = i - (i / PS) * PS;
            phi[i] = xv(m, c);
        }
    // E = -phi' at the degree-k nodes (poisson.cpp:176-192)
    for (int i = tid; i < N * (k + 1); i += nth) {
        const int c = i / (k + 1), m = i - (i / (k + 1)) * (k + 1);
        double dphi = 0.0;
#pragma unroll
        for (int n = 0; n < PS; ++n) dphi += pd.deriv[m * PS + n] * xv(n, c);
        E[i] = -dphi / pd.h[c];
    }
}

// ---------------------------------------------------------------------------
// Poisson on a thread-block cluster, communication-avoiding: the same block-
// cyclic-reduction replay, every row computed with the single-CTA kernel's
// expressions (bitwise the same result). CTA c owns the level-0 rows
// [cB, (c+1)B) (B a multiple of 2^K). Instead of exchanging neighbour rows at
// every level, each CTA recomputes the halo its own rows depend on: the
// K reduction levels and the K back-substitution levels run CTA-locally with
// __syncthreads; only the <= 2C rows of level K go through CTA 0 (two cluster
// barriers around it). Level vectors live in shared memory.
// ---------------------------------------------------------------------------
namespace cg = cooperative_groups;

constexpr int kPMaxLev = 32;

struct PClusterMap {
    int N, C, B, K;
};

// row ranges of CTA c: b_l on [ra, rb) (reduction + back-substitution needs),
// x_l on [xa, xb) (back substitution), own level-l rows [lo, hi)
struct PRanges {
    int ra[kPMaxLev], rb[kPMaxLev], xa[kPMaxLev], xb[kPMaxLev];
};
__host__ __device__ inline int pc_lo(const PClusterMap& m, int c, int l) {
    const long long L = (long long)c * m.B < m.N ? (long long)c * m.B : m.N;
    return (int)((L + (1LL << l) - 1) >> l);
}
__host__ __device__ inline void pc_ranges(const PClusterMap& m, const int* level_n, int c, PRanges& R) {
    const int K = m.K;
    R.xa[0] = pc_lo(m, c, 0);
    R.xb[0] = pc_lo(m, c + 1, 0);
    for (int l = 0; l < K; ++l) {
        R.xa[l + 1] = R.xa[l] >> 1;
        const int e = (R.xb[l] >> 1) + 1;
        R.xb[l + 1] = e < level_n[l + 1] ? e : level_n[l + 1];
        if (R.xb[l] <= R.xa[l]) R.xb[l + 1] = R.xa[l + 1];  // nothing to solve
    }
    R.ra[K] = pc_lo(m, c, K);
    R.rb[K] = pc_lo(m, c + 1, K);
    for (int l = K - 1; l >= 0; --l) {
        int a = 2 * R.ra[l + 1] - 1, b = 2 * R.rb[l + 1];
        if (R.rb[l + 1] <= R.ra[l + 1]) {  // no reduction rows above: back-sub needs only
            a = R.xa[l];
            b = R.xb[l];
        } else {
            if (R.xb[l] > R.xa[l]) {
                a = a < R.xa[l] ? a : R.xa[l];
                b = b > R.xb[l] ? b : R.xb[l];
            }
        }
        R.ra[l] = a > 0 ? a : 0;
        R.rb[l] = b < level_n[l] ? b : level_n[l];
        if (R.rb[l] < R.ra[l]) R.rb[l] = R.ra[l];
    }
}
// doubles of shared memory: b levels 0..K, x levels 0..K, then (CTA 0) the top
__host__ __device__ inline int pc_vec_doubles(const PClusterMap& m, const PRanges& R, int ps) {
    int o = 0;
    for (int l = 0; l <= m.K; ++l) o += (R.rb[l] - R.ra[l]) + (R.xb[l] - R.xa[l]);
    return o * ps;
}

template <int PS>
__global__ void __launch_bounds__(1024) poisson_cluster_kernel(const __grid_constant__ PoissonDev pd,
                                                               const __grid_constant__ PClusterMap cm, int stage,
                                                               const double* __restrict__ rho,
                                                               double* __restrict__ E,
                                                               double* __restrict__ phi) {
    pdl_enter();
    if (halted(pd.st)) return;
    constexpr int pp = PS * PS;
    extern __shared__ double psm[];
    cg::cluster_group cl = cg::this_cluster();
    const int c = (int)cl.block_rank();
    const int k = PS - 2;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int K = cm.K, L = pd.nlevels;
    __shared__ PRanges R;
    __shared__ int bo[kPMaxLev], xo[kPMaxLev];
    if (tid == 0) {
        pc_ranges(cm, pd.level_n, c, R);
        int o = 0;
        for (int l = 0; l <= K; ++l) {
            bo[l] = o;
            o += (R.rb[l] - R.ra[l]) * PS;
        }
        for (int l = 0; l <= K; ++l) {
            xo[l] = o;
            o += (R.xb[l] - R.xa[l]) * PS;
        }
    }
    __syncthreads();
    // ---- load vector (poisson.cpp:135-149) on [ra0, rb0): own rows + halo
    {
        const int a0 = R.ra[0], n0 = R.rb[0] - a0;
        double* b0 = psm + bo[0];
        for (int i = tid; i < n0 * PS; i += nth) {
            const int m = i / n0, q = i - (i / n0) * n0, cc = a0 + q;
            b0[i] = poisson_load<PS>(pd, stage, rho, cc, m);
        }
    }
    __syncthreads();
    // ---- reduction, levels 0 .. K-1, CTA-local
    for (int l = 0; l < K; ++l) {
        const int Nl = pd.level_n[l], Nn = pd.level_n[l + 1];
        const double* Al = pd.AlphaT + pd.keep_off[l] * pp;
        const double* Gl = pd.GammaT + pd.keep_off[l] * pp;
        const int al = R.ra[l], nl = R.rb[l] - al;
        const int an = R.ra[l + 1], nn = R.rb[l + 1] - an;
        const double* bl = psm + bo[l];
        double* bn = psm + bo[l + 1];
        for (int i = tid; i < nn * PS; i += nth) {
            const int m = i / nn, rr = i - (i / nn) * nn, r = an + rr, q = 2 * r;
            double v = bl[m * nl + (q - al)];
            if (q - 1 >= 0) {
                double acc = 0.0;
#pragma unroll
                for (int n = 0; n < PS; ++n) acc += Al[(long long)(m * PS + n) * Nn + r] * bl[n * nl + (q - 1 - al)];
                v += acc;
            }
            if (q + 1 < Nl) {
                double acc = 0.0;
#pragma unroll
                for (int n = 0; n < PS; ++n) acc += Gl[(long long)(m * PS + n) * Nn + r] * bl[n * nl + (q + 1 - al)];
                v += acc;
            }
            bn[m * nn + rr] = v;
        }
        __syncthreads();
    }
    cl.sync();  // every CTA's own level-K rows are in place
    double* top = psm + pc_vec_doubles(cm, R, PS);  // CTA 0: [b levels K.. | x levels K..]
    int tofs = 0;                                   // doubles of the top b levels (x levels follow)
    for (int l = K; l < L; ++l) tofs += pd.level_n[l] * PS;
    if (c == 0) {
        int tb[kPMaxLev], tx[kPMaxLev];
        int o = 0;
        for (int l = K; l < L; ++l) {
            tb[l] = o;
            o += pd.level_n[l] * PS;
        }
        for (int l = K; l < L; ++l) {
            tx[l] = o;
            o += pd.level_n[l] * PS;
        }
        const int NK = pd.level_n[K];
        // gather level K from the owners (DSMEM)
        for (int i = tid; i < NK * PS; i += nth) {
            const int m = i / NK, r = i - (i / NK) * NK;
            const int ow = min((int)(((long long)r << K) / cm.B), cm.C - 1);
            PRanges Ro;
            pc_ranges(cm, pd.level_n, ow, Ro);
            int off = 0;
            for (int l = 0; l < K; ++l) off += (Ro.rb[l] - Ro.ra[l]) * PS;
            const double* src = cl.map_shared_rank(psm, ow);
            top[tb[K] + i] = src[off + m * (Ro.rb[K] - Ro.ra[K]) + (r - Ro.ra[K])];
        }
        __syncthreads();
        for (int l = K; l + 1 < L; ++l) {
            const int Nl = pd.level_n[l], Nn = pd.level_n[l + 1];
            const double* bl = top + tb[l];
            double* bn = top + tb[l + 1];
            const double* Al = pd.AlphaT + pd.keep_off[l] * pp;
            const double* Gl = pd.GammaT + pd.keep_off[l] * pp;
            for (int i = tid; i < Nn * PS; i += nth) {
                const int m = i / Nn, r = i - (i / Nn) * Nn, q = 2 * r;
                double v = bl[m * Nl + q];
                if (q - 1 >= 0) {
                    double acc = 0.0;
#pragma unroll
                    for (int n = 0; n < PS; ++n) acc += Al[(long long)(m * PS + n) * Nn + r] * bl[n * Nl + q - 1];
                    v += acc;
                }
                if (q + 1 < Nl) {
                    double acc = 0.0;
#pragma unroll
                    for (int n = 0; n < PS; ++n) acc += Gl[(long long)(m * PS + n) * Nn + r] * bl[n * Nl + q + 1];
                    v += acc;
                }
                bn[m * Nn + r] = v;
            }
            __syncthreads();
        }
        if (tid < PS) {
            const double* bt = top + tb[L - 1];
            double acc = 0.0;
#pragma unroll
            for (int n = 0; n < PS; ++n) acc += pd.DinvTop[tid * PS + n] * bt[n];
            top[tx[L - 1] + tid] = acc;
        }
        __syncthreads();
        for (int l = L - 2; l >= K; --l) {
            const int Nl = pd.level_n[l], Nn = pd.level_n[l + 1], No = Nl / 2;
            double* bl = top + tb[l];
            double* xl = top + tx[l];
            const double* xn = top + tx[l + 1];
            const double* Lo = pd.LoT + pd.odd_off[l] * pp;
            const double* Up = pd.UpT + pd.odd_off[l] * pp;
            const double* Di = pd.DinvT + pd.odd_off[l] * pp;
            for (int i = tid; i < Nl * PS; i += nth) {
                const int m = i / Nl, q = i - (i / Nl) * Nl;
                if ((q & 1) == 0) {
                    xl[m * Nl + q] = xn[m * Nn + q / 2];
                } else {
                    const int oo = q >> 1;
                    double t = bl[m * Nl + q];
                    double acc = 0.0;
#pragma unroll
                    for (int n = 0; n < PS; ++n) acc += Lo[(long long)(m * PS + n) * No + oo] * xn[n * Nn + oo];
                    t -= acc;
                    if (q + 1 < Nl) {
                        acc = 0.0;
#pragma unroll
                        for (int n = 0; n < PS; ++n) acc += Up[(long long)(m * PS + n) * No + oo] * xn[n * Nn + oo + 1];
                        t -= acc;
                    }
                    bl[m * Nl + q] = t;
                }
            }
            __syncthreads();
            for (int i = tid; i < No * PS; i += nth) {
                const int m = i / No, oo = i - (i / No) * No, q = 2 * oo + 1;
                double acc = 0.0;
#pragma unroll
                for (int n = 0; n < PS; ++n) acc += Di[(long long)(m * PS + n) * No + oo] * bl[n * Nl + q];
                xl[m * Nl + q] = acc;
            }
            __syncthreads();
        }
    }
    cl.sync();  // x_K complete in CTA 0
    {
        const int NK = pd.level_n[K], xa = R.xa[K], nx = R.xb[K] - xa;
        // CTA 0's top area sits after CTA 0's own vectors
        PRanges R0;
        pc_ranges(cm, pd.level_n, 0, R0);
        const double* xK0 = cl.map_shared_rank(psm, 0) + pc_vec_doubles(cm, R0, PS) + tofs;
        double* xK = psm + xo[K];
        for (int i = tid; i < nx * PS; i += nth) {
            const int m = i / nx, r = i - (i / nx) * nx;
            xK[i] = xK0[m * NK + xa + r];
        }
    }
    cl.sync();  // CTA 0's top area is no longer read
    // ---- back substitution, levels K-1 .. 0, CTA-local on [xa_l, xb_l)
    for (int l = K - 1; l >= 0; --l) {
        const int Nl = pd.level_n[l], No = Nl / 2;
        const int xa = R.xa[l], nx = R.xb[l] - xa, ax = R.xa[l + 1], nxn = R.xb[l + 1] - ax;
        const int al = R.ra[l], nl = R.rb[l] - al;
        double* bl = psm + bo[l];
        double* xl = psm + xo[l];
        const double* xn = psm + xo[l + 1];
        const double* Lo = pd.LoT + pd.odd_off[l] * pp;
        const double* Up = pd.UpT + pd.odd_off[l] * pp;
        const double* Di = pd.DinvT + pd.odd_off[l] * pp;
        for (int i = tid; i < nx * PS; i += nth) {
            const int m = i / nx, qq = i - (i / nx) * nx, q = xa + qq;
            if ((q & 1) == 0) {
                xl[m * nx + qq] = xn[m * nxn + (q / 2 - ax)];
            } else {
                const int oo = q >> 1;
                double t = bl[m * nl + (q - al)];
                double acc = 0.0;
#pragma unroll
                for (int n = 0; n < PS; ++n) acc += Lo[(long long)(m * PS + n) * No + oo] * xn[n * nxn + (oo - ax)];
                t -= acc;
                if (q + 1 < Nl) {
                    acc = 0.0;
#pragma unroll
                    for (int n = 0; n < PS; ++n)
                        acc += Up[(long long)(m * PS + n) * No + oo] * xn[n * nxn + (oo + 1 - ax)];
                    t -= acc;
                }
                bl[m * nl + (q - al)] = t;
            }
        }
        __syncthreads();
        for (int i = tid; i < nx * PS; i += nth) {
            const int m = i / nx, qq = i - (i / nx) * nx, q = xa + qq;
            if ((q & 1) == 0) continue;
            const int oo = q >> 1;
            double acc = 0.0;
#pragma unroll
            for (int n = 0; n < PS; ++n) acc += Di[(long long)(m * PS + n) * No + oo] * bl[n * nl + (q - al)];
            xl[m * nx + qq] = acc;
        }
        __syncthreads();
    }
    // ---- phi and E = -phi' (poisson.cpp:176-192), own cells
    {
        const int l0 = R.xa[0], n0 = R.xb[0] - l0;
        const double* x0 = psm + xo[0];
        if (stage == 1) {  // first solve of the refinement: keep x, no E yet
            for (int i = tid; i < n0 * PS; i += nth) {
                const int q = i / PS, m = i - (i / PS) * PS;
                pd.ir_x[(long long)(l0 + q) * PS + m] = x0[m * n0 + q];
            }
            return;
        }
        auto xv = [&](int n, int q) {
            return stage == 2 ? pd.ir_x[(long long)(l0 + q) * PS + n] + x0[n * n0 + q] : x0[n * n0 + q];
        };
        if (phi)
            for (int i = tid; i < n0 * PS; i += nth) {
                const int q = i / PS, m = i - (i / PS) * PS;
                phi[(long long)(l0 + q) * PS + m] = xv(m, q);
            }
        for (int i = tid; i < n0 * (k + 1); i += nth) {
            const int q = i / (k + 1), m = i - (i / (k + 1)) * (k + 1), cc = l0 + q;
            double dphi = 0.0;
#pragma unroll
            for (int n = 0; n < PS; ++n) dphi += pd.deriv[m * PS + n] * xv(n, q);
            E[(long long)cc * (k + 1) + m] = -dphi / pd.h[cc];
        }
    }
}

// ---------------------------------------------------------------------------
// exact-reduction mode: the reference's serial orders, so that a whole
// trajectory is bitwise the reference's (parity mode, not the fast path)
// ---------------------------------------------------------------------------
// charge_density (poisson.cpp:194-216): per x dof, ions then electrons,
// rows ascending, rho += ((sign*w_vn)*dv) * f. The sum is one sequential chain
// per x dof (nx*p of them), so the parallelism for HBM is in the loads: each
// thread streams its column through a cp.async ring in shared memory
// ([slot][thread]: a warp's slot is one coalesced 256-byte row piece), one
// commit group per v cell (P rows), kRhoRingCells cells in flight while the
// adds retire in order. (Per-row groups cost ~140 cycles of issue overhead per
// row, and a 96-row ring left C5's 2048 CTAs in two waves: C5 36.3 -> 18.4 ms,
// C3 2.33 -> 1.32 ms.)
constexpr int kRhoThreads = 32, kRhoRingCells = 12;  // 12.3 KB per CTA at P = 4: 18 CTAs/SM, C5 in one wave
template <int P>
__global__ void __launch_bounds__(kRhoThreads) rho_exact_kernel(const __grid_constant__ RhoArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    constexpr int RC = kRhoRingCells;
    __shared__ double ring[RC * P * kRhoThreads];
    const int xd = blockIdx.x * blockDim.x + threadIdx.x;
    if (xd >= a.nxd) return;
    const double* fs[2];
    double wv[2][P];
    for (int s = 0; s < 2; ++s) {  // s = 0: ions (sign +1), s = 1: electrons (sign -1)
        const int sp = s == 0 ? 1 : 0;
        const double sign = s == 0 ? 1.0 : -1.0;
        const double dv = a.vg[sp]->dx;
        fs[s] = (field_flipped(a.flip[sp]) ? a.alt[sp] : a.f[sp]) + xd;
#pragma unroll
        for (int vn = 0; vn < P; ++vn) wv[s][vn] = sign * a.basis.weights[vn] * dv;
    }
    const long long nr = a.nrows;            // rows per species (a multiple of P)
    const long long ncell = 2 * (nr / P);    // v cells of both species, ions first
    double* my = ring + threadIdx.x;
    auto issue = [&](long long g, int slot) {  // the P rows of v cell g
        if (g < ncell) {
            const long long r0 = g * P;
            const int s = r0 >= nr;
            const double* src = fs[s] + (r0 - s * nr) * a.ld;
#pragma unroll
            for (int vn = 0; vn < P; ++vn) cp_async8(my + (slot * P + vn) * kRhoThreads, src + vn * a.ld, true);
        }
        cp_commit();
    };
#pragma unroll 1
    for (int c = 0; c < RC - 1; ++c) issue(c, c);
    double acc = 0.0;
#pragma unroll
    for (int s = 0; s < 2; ++s) {  // (unrolled: the species' weights stay in registers)
#pragma unroll 1
        for (long long g = s * (ncell / 2); g < (s + 1) * (ncell / 2); ++g) {
            const int slot = (int)(g % RC);
            cp_wait<RC - 2>();
            double v[P];
#pragma unroll
            for (int vn = 0; vn < P; ++vn) v[vn] = my[(slot * P + vn) * kRhoThreads];
            // refill the slot consumed one cell ago (its values are in acc already)
            issue(g + RC - 1, slot == 0 ? RC - 1 : slot - 1);
#pragma unroll
            for (int vn = 0; vn < P; ++vn) acc += wv[s][vn] * v[vn];
        }
    }
    cp_wait<0>();
    a.rho[xd] = acc;
}

// PoissonOperator::solve with dpbtrs('L') = dtbsv('L','N') + dtbsv('L','T')
// replayed in reference-BLAS order (poisson.cpp:135-192), bitwise.
//
// Both triangular sweeps are one dependence chain (column j's division needs
// every earlier column's update of x[j]; the transposed sweep's dot product is
// a fixed sequential sum), so the arithmetic stays on one thread. What is not
// serial is moved off it:
//  * the band window x[j..j+kd] lives in that thread's registers (no memory
//    round trip between dependent columns), and the rest of the block stages
//    the next chunk of factor columns, right-hand sides and reciprocals of the
//    diagonal into shared memory while it works on the current chunk;
//  * each IEEE division a/c on the chain becomes q = a*r, q += (a - q*c)*r
//    with r = RN(1/c) precomputed (Markstein's correction: RN(a/c) except in
//    cases a few ulp^2 from a rounding boundary). The dividends are recorded;
//    afterwards all threads re-divide them in parallel and compare bit for
//    bit, and a pass with any mismatch is replayed with true divisions -- the
//    result is the reference's either way.
// The load and E = -phi' phases are parallel over dofs.
#ifndef SK_PEX_UNROLL
#define SK_PEX_UNROLL 4
#endif
constexpr int kPexUnroll = SK_PEX_UNROLL;  // exact Poisson: columns per unrolled step of the serial sweeps
__device__ __forceinline__ double div_markstein(double a, double c, double r) {
    const double q = __dmul_rn(a, r);
    const double e = __fma_rn(-q, c, a);  // exact remainder
    return __fma_rn(e, r, q);
}

template <int PS>
__global__ void __launch_bounds__(256) poisson_exact_kernel(const __grid_constant__ PoissonDev pd,
                                                            const double* __restrict__ rho,
                                                            double* __restrict__ E,
                                                            double* __restrict__ phi) {
    pdl_enter();
    if (halted(pd.st)) return;
    constexpr int KD = 2 * PS - 1, LD = KD + 1, CH = 128;
    __shared__ double scol[2][CH * LD];
    __shared__ double sx[2][CH];
    __shared__ double srcp[2][CH];
    __shared__ int redo;
    const int k = pd.k, N = pd.ncells, n = N * PS;
    double* x = pd.xws;
    double* rhs = pd.exws;              // load vector (replay source of the forward pass)
    double* fwd = pd.exws + n;          // forward result (replay source of the backward pass)
    double* dvd = pd.exws + 2 * n;      // dividends on the chain
    for (int i = threadIdx.x; i < n; i += blockDim.x) {  // build_load (poisson.cpp:135-149)
        const int c = i / PS, m = i - (i / PS) * PS;
        double val = 0.0;
        for (int q = 0; q <= k; ++q) val += pd.interp[m * (k + 1) + q] * rho[c * (k + 1) + q];
        x[i] = rhs[i] = pd.ws[m] * pd.h[c] * val;
    }
    const int nch = (n + CH - 1) / CH;
    // chunk ch of factor columns, 1/diagonal and x[xoff + ch*CH + i] into buffer
    // b; warp 0 computes, the other warps stage (or, with all = true, warp 0)
    auto stage = [&](int ch, int b, int xoff, bool all) {
        const int j0 = ch * CH, ncol = min(CH, n - j0);
        const double* src = pd.chol + (long long)j0 * LD;
        const int t0 = all ? (int)threadIdx.x : (int)threadIdx.x - 32;
        const int nt = all ? 32 : (int)blockDim.x - 32;
        for (int i = t0; i >= 0 && i < ncol * LD; i += nt) scol[b][i] = src[i];
        for (int i = t0; i >= 0 && i < CH; i += nt) {
            const int g = j0 + i + xoff;
            sx[b][i] = g >= 0 && g < n ? x[g] : 0.0;
            srcp[b][i] = i < ncol ? 1.0 / src[(long long)i * LD] : 0.0;
        }
    };
    // ---- dtbsv('L','N'): forward, column oriented ----
    auto forward = [&](auto fast_c) {
        constexpr bool FAST = decltype(fast_c)::value;
        double w[LD];  // x[j .. j+KD]
        if (threadIdx.x == 0)
#pragma unroll
            for (int l = 0; l < LD; ++l) w[l] = l < n ? x[l] : 0.0;
        if (threadIdx.x < 32) stage(0, 0, LD, true);
        __syncthreads();
        for (int ch = 0; ch < nch; ++ch) {
            const int b = ch & 1;
            if (ch + 1 < nch) stage(ch + 1, b ^ 1, LD, false);
            if (threadIdx.x == 0) {
                const int j0 = ch * CH, j1 = min(n, j0 + CH);
                // (unrolled, branch-free: the column loads and the off-chain updates of
                // the next columns overlap this column's division; a zero x[j] keeps
                // every value through selects, as the reference's skip does)
#pragma unroll kPexUnroll
                for (int j = j0; j < j1; ++j) {
                    const double* col = &scol[b][(j - j0) * LD];
                    if (FAST) dvd[j] = w[0];
                    const bool nz = w[0] != 0.0;
                    const double q = FAST ? div_markstein(w[0], col[0], srcp[b][j - j0]) : w[0] / col[0];
                    w[0] = nz ? q : w[0];
                    const double temp = w[0];
#pragma unroll
                    for (int l = 1; l < LD; ++l)
                        if (j + l < n) w[l] = nz ? w[l] - temp * col[l] : w[l];
                    x[j] = w[0];
#pragma unroll
                    for (int l = 0; l + 1 < LD; ++l) w[l] = w[l + 1];
                    w[LD - 1] = sx[b][j - j0];  // x[j + LD], untouched by columns <= j
                }
            }
            __syncthreads();
        }
    };
    // ---- dtbsv('L','T'): backward, dot-product form, i from imax down to j+1 ----
    auto backward = [&](auto fast_c) {
        constexpr bool FAST = decltype(fast_c)::value;
        double u[LD];  // u[l] = x[j + l] (final), l = 1..KD
#pragma unroll
        for (int l = 0; l < LD; ++l) u[l] = 0.0;
        const int last = nch - 1;
        if (threadIdx.x < 32) stage(last, last & 1, 0, true);
        __syncthreads();
        for (int ch = last; ch >= 0; --ch) {
            const int b = ch & 1;
            if (ch > 0) stage(ch - 1, b ^ 1, 0, false);
            if (threadIdx.x == 0) {
                const int j0 = ch * CH, j1 = min(n, j0 + CH);
#pragma unroll kPexUnroll
                for (int j = j1 - 1; j >= j0; --j) {  // (unrolled: the chain's first KD - 1 terms overlap)
                    const double* col = &scol[b][(j - j0) * LD];
                    double temp = sx[b][j - j0];
#pragma unroll
                    for (int l = LD - 1; l >= 1; --l)
                        if (j + l < n) temp = temp - col[l] * u[l];
                    if (FAST) dvd[j] = temp;
                    temp = FAST ? div_markstein(temp, col[0], srcp[b][j - j0]) : temp / col[0];
#pragma unroll
                    for (int l = LD - 1; l >= 2; --l) u[l] = u[l - 1];
                    u[1] = temp;
                    x[j] = temp;
                }
            }
            __syncthreads();
        }
    };
    // every recorded dividend divided again (IEEE), bit for bit against x
    auto verify = [&](bool skip_zero) {
        if (threadIdx.x == 0) redo = 0;
        __syncthreads();
        int bad = 0;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            const double a = dvd[j];
            if (skip_zero && a == 0.0) continue;  // forward: zero columns are not divided
            bad |= __double_as_longlong(a / pd.chol[(long long)j * LD]) != __double_as_longlong(x[j]);
        }
        if (__syncthreads_or(bad) && threadIdx.x == 0) redo = 1;
        __syncthreads();
        return redo != 0;
    };
    __syncthreads();
    forward(std::true_type{});
    if (verify(true)) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = rhs[i];
        __syncthreads();
        forward(std::false_type{});
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) fwd[i] = x[i];
    __syncthreads();
    backward(std::true_type{});
    if (verify(false)) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = fwd[i];
        __syncthreads();
        backward(std::false_type{});
    }
    if (phi)
        for (int i = threadIdx.x; i < n; i += blockDim.x) phi[i] = x[i];
    for (int i = threadIdx.x; i < N * (k + 1); i += blockDim.x) {  // E = -phi' (poisson.cpp:182-190)
        const int c = i / (k + 1), m = i - (i / (k + 1)) * (k + 1);
        double dphi = 0.0;
        for (int q = 0; q < PS; ++q) dphi += pd.deriv[m * PS + q] * x[c * PS + q];
        E[i] = -dphi / pd.h[c];
    }
}

// ---------------------------------------------------------------------------
// step end: step counter, nonfinite -> SimulationError (stepper.cpp:99-102),
// shrink cooldown gate (run.cpp:98-101)
// ---------------------------------------------------------------------------
__global__ void step_end_kernel(DevStatus* st, double dt, int v_adjust, long long cooldown, int mask) {
    pdl_enter();
    if (halted(st)) return;  // no step after a failed one (the step counter stays at it)
    st->time += dt;  // stepper.cpp:98
    st->step += 1;
    if (st->nonfinite) raise_error(st, 2, 3, 0, 0, st->step);
    for (int sp = 0; sp < 2; ++sp)
        st->shrink_flag[sp] =
            ((mask >> sp) & 1) && v_adjust && (st->step - st->last_shrink[sp] >= cooldown) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// K5/K6: velocity cut-off (adaptivity.cpp:16-130)
// ---------------------------------------------------------------------------
template <int P>
__global__ void shrink_check_kernel(const __grid_constant__ ShrinkArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    const int sp = blockIdx.y;
    if (!((a.species_mask >> sp) & 1)) return;
    if (a.st->shrink_flag[sp] == 0) return;
    const int xd = blockIdx.x * blockDim.x + threadIdx.x;
    if (xd >= a.nxd) return;
    const DevVGrid vg = *a.vg[sp];
    const double dv = vg.dx;
    const double right = vg.left + vg.cells * vg.dx;
    const double probe = right * (1.0 - a.p - a.gamma);
    const double* f = field_flipped(a.flip[sp]) ? a.out[sp] : a.f[sp];
    bool fail = false;
    for (int s = 0; s < 2; ++s) {
        double vp = (s == 0 ? 1.0 : -1.0) * probe;
        int vc = (int)floor((vp - vg.left) / dv);
        vc = min(max(vc, 0), vg.cells - 1);
        const int vl = vc - a.cell0;  // a v shard evaluates only the probe cells it holds
        if (vl < 0 || vl >= a.nv) continue;
        double xi = (vp - (vg.left + vc * vg.dx)) / dv;
        double val = 0.0;
#pragma unroll
        for (int vn = 0; vn < P; ++vn)
            val += lagrange<P>(a.basis, vn, xi) * f[((long long)vl * P + vn) * a.ld + xd];
        if (fabs(val) >= a.tol) fail = true;
    }
    if (fail) a.st->shrink_flag[sp] = 0;
}

// build_v_transfer (adaptivity.cpp:52-90): one thread per new cell
template <int P>
__global__ void shrink_table_kernel(const __grid_constant__ ShrinkArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    const int sp = blockIdx.y;
    if (!((a.species_mask >> sp) & 1) || a.st->shrink_flag[sp] == 0) return;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;  // global new cell
    if (j >= a.nv_global) return;
    const DevVGrid ov = *a.vg[sp];
    const double vmax_before = ov.left + ov.cells * ov.dx;
    const double new_vmax = vmax_before * (1.0 - a.p);
    const double nleft = -new_vmax;
    const double ndx = (new_vmax - (-new_vmax)) / a.nv_global;  // Grid1D::uniform (grid.cpp:31-34)
    const double old_dx = ov.dx;
    const double aa = nleft + j * ndx;
    const double h = ndx;
    const double bb = aa + h;
    int i0 = (int)floor((aa - ov.left) / old_dx);
    i0 = min(max(i0, 0), ov.cells - 1);
    int np = 0;
    double* T = a.ttab[sp] + (long long)j * 4 * P * P;
    int* cellv = a.tcell[sp] + (long long)j * 4;
    for (int i = i0; i < ov.cells; ++i) {
        double oa = ov.left + i * ov.dx, ob = oa + old_dx;
        double s0 = dmax2(aa, oa), s1 = dmin2(bb, ob);
        if (s1 <= s0) {
            if (oa >= bb) break;
            continue;
        }
        if (np >= 4) {
            raise_error(a.st, 1, 4, np, 4, a.st->step);
            break;
        }
        double Tm[P * P];
#pragma unroll
        for (int t = 0; t < P * P; ++t) Tm[t] = 0.0;
        const double len = s1 - s0;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            double x = s0 + len * a.basis.nodes[q];
            double xi_src = (x - oa) / old_dx;
            double xi_tgt = (x - aa) / h;
            double wq = a.basis.weights[q] * len;
#pragma unroll
            for (int m = 0; m < P; ++m) {
                double lm = lagrange<P>(a.basis, m, xi_tgt) / (a.basis.weights[m] * h);
#pragma unroll
                for (int n = 0; n < P; ++n) Tm[m * P + n] += wq * lm * lagrange<P>(a.basis, n, xi_src);
            }
        }
#pragma unroll
        for (int t = 0; t < P * P; ++t) T[np * P * P + t] = Tm[t];
        cellv[np] = i;
        ++np;
    }
    for (int q = np; q < 4; ++q) cellv[q] = -1;
}

// wait until at most n cp.async groups are pending (n < 8, run time value)
__device__ __forceinline__ void cp_wait_dyn(int n) {
    switch (n) {
        case 0: cp_wait<0>(); break;
        case 1: cp_wait<1>(); break;
        case 2: cp_wait<2>(); break;
        case 3: cp_wait<3>(); break;
        case 4: cp_wait<4>(); break;
        case 5: cp_wait<5>(); break;
        case 6: cp_wait<6>(); break;
        default: cp_wait<7>(); break;
    }
}

// per x dof, new cell j: dst[m] = sum_pieces (sum_n T[m][n] src[n]) (adaptivity.cpp:109-124).
// The old cells of a chunk of new cells form one increasing run [olo, ohi];
// they stream through the v sweep's per-thread cp.async ring (old cell c in
// slot (c - olo) % R, one commit group per cell), so R*P loads stay in flight
// per thread. Consecutive new cells share their boundary old cell, and the
// rounded new-cell edges (aa_{j+1} vs bb_j) can send cell j+1 one old cell
// back: a slot is refilled only once the current new cell starts two old
// cells past it. A cell outside the ring window is read from global directly.
template <int P>
__global__ void __launch_bounds__(kVThreads) shrink_project_kernel(const __grid_constant__ ShrinkArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    // the block's threads share the chunk: its transfer matrices are staged
    // once per item (coalesced) instead of each warp re-reading them per cell;
    // a 4-deep ring then keeps the CTA at 32 KB (7 CTAs, 28 warps per SM)
    constexpr bool TS = P <= 4;
    constexpr int R = TS ? 4 : vring<P>();
    static_assert(R <= 8, "cp_wait_dyn covers 8 groups");
    __shared__ double ring[R * P * kVThreads];
    constexpr int TN = 4 * P * P;  // doubles per new cell
    __shared__ __align__(16) double tsh[TS ? kVChunk * TN : 2];
    __shared__ int csh[TS ? kVChunk * 4 : 1];  // the chunk's old-cell lists
    const int sp = blockIdx.z;
    // bounded grid, (x block, v chunk) items by grid stride: on the (usual)
    // steps without a shrink the whole launch is a few hundred early exits
    if (!((a.species_mask >> sp) & 1) || a.st->shrink_flag[sp] == 0) return;
    const int nxb = (a.nxd + kVThreads - 1) / kVThreads;
    const long long nitems = (long long)nxb * ((a.nv + kVChunk - 1) / kVChunk);
    const bool fl = field_flipped(a.flip[sp]);
    const double* f = fl ? a.out[sp] : a.f[sp];
    double* out = fl ? a.f[sp] : a.out[sp];
    double* my = ring + threadIdx.x;
    const long long ld = a.ld;
    for (long long w = blockIdx.x; w < nitems; w += gridDim.x) {
        const int xd = (int)(w % nxb) * kVThreads + threadIdx.x;
        const int j0 = (int)(w / nxb) * kVChunk, j1 = min(j0 + kVChunk, a.nv);
        if constexpr (TS) {
            const double* tg = a.ttab[sp] + ((long long)a.cell0 + j0) * TN;
            __syncthreads();  // the previous item's readers are done
            for (int i = threadIdx.x; i < (j1 - j0) * TN; i += kVThreads) tsh[i] = tg[i];
            const int* cg = a.tcell[sp] + ((long long)a.cell0 + j0) * 4;
            for (int i = threadIdx.x; i < (j1 - j0) * 4; i += kVThreads) csh[i] = cg[i];
            __syncthreads();
        }
        if (xd >= a.nxd) continue;
        const int* cv0 = TS ? csh : a.tcell[sp] + ((long long)a.cell0 + j0) * 4;
        const int* cv1 = cv0 + (j1 - 1 - j0) * 4;
        const int olo = cv0[0] - a.cell0;
        int ohi = olo;
        for (int pc = 0; pc < 4 && cv1[pc] >= 0; ++pc) ohi = cv1[pc] - a.cell0;
        // old cells outside the allocated rows are reported when consumed
        auto issue = [&](int c) {
            const bool ok = c >= -a.halo && c < a.nv + a.halo;
            const double* g = f + xd + (ok ? (long long)c * P * ld : 0);
            double* slot = my + ((c - olo) % R) * P * kVThreads;
#pragma unroll
            for (int n = 0; n < P; ++n) cp_async8(slot + n * kVThreads, g + n * ld, ok);
            cp_commit();
        };
        int iss = olo;  // next old cell to issue; groups committed = iss - olo
        for (; iss <= ohi && iss < olo + R; ++iss) issue(iss);
        for (int j = j0; j < j1; ++j) {
            double dst[P];
#pragma unroll
            for (int m = 0; m < P; ++m) dst[m] = 0.0;
            const long long jg = (long long)a.cell0 + j;  // global new cell
            const double* T = TS ? tsh + (j - j0) * TN : a.ttab[sp] + jg * TN;
            const int* cellv = cv0 + (j - j0) * 4;
            int oc = olo;
            for (int pc = 0; pc < 4; ++pc) {
                const int c = cellv[pc];
                if (c < 0) break;
                oc = c - a.cell0;  // local old cell; a shard reads up to `halo` beyond its range
                if (oc < -a.halo || oc >= a.nv + a.halo) {
                    raise_error(a.st, 1, 6, oc, a.halo, a.st->step);
                    break;
                }
                double src[P];
                if (oc >= iss - R && oc < iss && oc >= olo) {
                    cp_wait_dyn(iss - 1 - oc);
                    const double* sl = my + ((oc - olo) % R) * P * kVThreads;
#pragma unroll
                    for (int n = 0; n < P; ++n) src[n] = sl[n * kVThreads];
                } else {
#pragma unroll
                    for (int n = 0; n < P; ++n) src[n] = f[((long long)oc * P + n) * ld + xd];
                }
#pragma unroll
                for (int m = 0; m < P; ++m) {
                    double tr[P];  // row m of piece pc (16-byte shared loads when staged)
                    if constexpr (TS && P % 2 == 0) {
#pragma unroll
                        for (int n = 0; n < P; n += 2) {
                            const double2 t2 = *reinterpret_cast<const double2*>(T + pc * P * P + m * P + n);
                            tr[n] = t2.x;
                            tr[n + 1] = t2.y;
                        }
                    } else {
#pragma unroll
                        for (int n = 0; n < P; ++n) tr[n] = T[pc * P * P + m * P + n];
                    }
                    double acc = 0.0;
#pragma unroll
                    for (int n = 0; n < P; ++n) acc += tr[n] * src[n];
                    dst[m] += acc;
                }
            }
#pragma unroll
            for (int m = 0; m < P; ++m) out[((long long)j * P + m) * ld + xd] = dst[m];
            // cells below oc - 1 are done: their slots take cells up to oc - 2 + R
            for (; iss <= ohi && iss < oc - 1 + R; ++iss) issue(iss);
        }
        cp_wait<0>();
    }
}

// commit the new v grid (field.cpp:96-101); the projection already sits in
// the field's other buffer, so the buffers exchange roles instead of copying
__global__ void shrink_finalize_kernel(const __grid_constant__ ShrinkArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    const int sp = threadIdx.x;
    if (sp >= 2 || !((a.species_mask >> sp) & 1) || a.st->shrink_flag[sp] == 0) return;
    DevVGrid ov = *a.vg[sp];
    const double vmax_before = ov.left + ov.cells * ov.dx;
    const double new_vmax = vmax_before * (1.0 - a.p);
    a.vg[sp]->left = -new_vmax;
    a.vg[sp]->dx = (new_vmax - (-new_vmax)) / a.nv_global;
    a.st->vmax_before[sp] = vmax_before;
    a.st->last_shrink[sp] = a.st->step;
    a.st->shrink_count[sp] += 1;
    *a.flip_w[sp] ^= 1;
}

__global__ void shrink_force_kernel(DevStatus* st, int mask) {
    pdl_enter();
    for (int sp = 0; sp < 2; ++sp) st->shrink_flag[sp] = (mask >> sp) & 1;
}

// ---------------------------------------------------------------------------
// K8: diagnostics (field.cpp:52-88 + harness moments), deterministic
// ---------------------------------------------------------------------------
constexpr int kDiagBlocks = 592;
constexpr int kDiagThreads = 256;

template <int P>
__global__ void __launch_bounds__(kDiagThreads) diag_partial_kernel(const __grid_constant__ DiagArgs a) {
    pdl_enter();
    const DevVGrid vg = a.vg[0];
    const double* fb = field_flipped(a.flip) ? a.alt : a.f;
    const long long total = (long long)a.nrows * a.nxd;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int r = (int)(i / a.nxd);
        const int xd = (int)(i - (long long)r * a.nxd);
        const int vc = r / P, vn = r - (r / P) * P;
        const int xc = xd / P, xn = xd - (xd / P) * P;
        int b = 0;
        while (xc >= a.grid.start[b + 1]) ++b;
        const double wv = a.basis.weights[vn] * vg.dx;
        const double w = wv * a.basis.weights[xn] * a.grid.dx[b];
        const double v = (vg.left + (vc + vg.cell0) * vg.dx) + vg.dx * a.basis.nodes[vn];
        const double f = fb[(long long)r * a.ld + xd];
        s[0] += w * f;
        s[1] += w * f * f;
        s[2] += w * (v * f);
        s[3] += w * ((0.5 * v * v) * f);
    }
    __shared__ double red[4][kDiagThreads];
#pragma unroll
    for (int q = 0; q < 4; ++q) red[q][threadIdx.x] = s[q];
    __syncthreads();
    for (int w = kDiagThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
#pragma unroll
            for (int q = 0; q < 4; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x < 4) a.partial[blockIdx.x * 4 + threadIdx.x] = red[threadIdx.x][0];
}

__global__ void diag_final_kernel(const double* partial, int nblk, double* out) {
    pdl_enter();
    const int q = threadIdx.x;
    if (q >= 4) return;
    double acc = 0.0;
    for (int b = 0; b < nblk; ++b) acc += partial[b * 4 + q];
    out[q] = q == 1 ? sqrt(acc) : acc;
}

__global__ void fill_separable_kernel(double* f, const double* gx, const double* gv, long long ld,
                                      long long total) {
    pdl_enter();
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const long long r = i / ld;
        const long long xd = i - r * ld;
        f[i] = gx[xd] * gv[r];  // run.cpp:19-22: (c*exp(x-part))*exp(v-part)
    }
}

__global__ void copy_kernel(double* dst, const double* src, long long n) {
    pdl_enter();
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = src[i];
}

// ---------------------------------------------------------------------------
// K3: literature post-limiters (limiters.cpp:254-345). Flags from pre-pass data
// (out of place). X: tiles with a 1-cell halo (block ghosts via fill_ghost j=1).
// ---------------------------------------------------------------------------
template <int P, bool FAST>
__device__ __forceinline__ void post_modify(const PostCfg& cfg, const Basis& b, const double* um,
                                            const double* u0, const double* up, double* out) {
    if constexpr (FAST) {  // (tolerance mode: precomputed functionals, see modify_simple_weno_fast)
        if (cfg.modifier == 1)
            modify_simple_weno_fast<P>(b, um, u0, up, cfg, out);
        else
            modify_line_weno_fast<P>(b, um, u0, up, cfg, out);
        return;
    }
    if (cfg.modifier == 1)
        modify_simple_weno<P>(b, um, u0, up, cfg, out);
    else
        modify_line_weno<P>(b, um, u0, up, cfg, out);
}

// Post limiters in place, like the sweeps' limiter: a flag pass reads the
// field once (x: xsweep_kernel MODE 1 on the TMA pipeline; v: post_v_kernel)
// and queues the flagged cells; post_fix_kernel computes their (rare,
// expensive, divergent) WENO modifications from the untouched field into a
// side buffer, and post_scatter_kernel writes them -- so every modification
// sees pre-pass data, exactly the reference's single out-of-place pass. If the
// queue overflowed, post_copy_kernel first copies the field to the other
// buffer and the fix kernel rescans every cell from that copy.

// the three cells of x stencil (line, block-local cell c) from the pre-pass data
template <int P>
__device__ __forceinline__ void post_x_stencil(const PostArgs& a, const double* src, int b, int c,
                                               double* um, double* u0, double* up) {
    const Grid& g = a.grid;
    const int cells_b = g.cells[b];
    const long long gbase = (long long)g.start[b] * P;
    double* u[3] = {um, u0, up};
    for (int h = 0; h < 3; ++h) {
        const int s = c - 1 + h;
        if (s >= 0 && s < cells_b) {
#pragma unroll
            for (int n = 0; n < P; ++n) u[h][n] = src[gbase + (long long)s * P + n];
        } else if (a.periodic) {
            const int ss = ((s % cells_b) + cells_b) % cells_b;
#pragma unroll
            for (int n = 0; n < P; ++n) u[h][n] = src[gbase + (long long)ss * P + n];
        } else {
#pragma unroll
            for (int n = 0; n < P; ++n) u[h][n] = x_fetch_outside_ool<P>(a.basis, g, src, b, s, n);
        }
    }
}

// the field (live buffer) and the other buffer of species sp
__device__ __forceinline__ double* post_live(const PostArgs& a, int sp) {
    return const_cast<double*>(field_flipped(a.flip[sp]) ? a.dst[sp] : a.src[sp]);
}
__device__ __forceinline__ double* post_other(const PostArgs& a, int sp) {
    return const_cast<double*>(field_flipped(a.flip[sp]) ? a.src[sp] : a.dst[sp]);
}

// a modified cell's change to the charge density the x sweep fused (its
// moment summed the unmodified values): exact integer corrections as the
// sweep's clamp fixups add them (xfix_cell), same weight arithmetic
template <int P>
__device__ __forceinline__ void post_rho_corr(const PostArgs& a, int sp, int line, int cell, const double* o0,
                                              const double* o) {
    const int vn = line - (line / P) * P;
    const double wdv = a.charge_w[sp] * a.basis.weights[vn] * a.vg[sp]->dx;
#pragma unroll
    for (int q = 0; q < P; ++q) {
        if (o[q] == o0[q]) continue;
        const double d = wdv * o[q] - wdv * o0[q];
        rho_corr_add(a.rho_corr + (long long)(line % kRhoCorrCopies) * a.grid.ncells * P,
                     (long long)kRhoCorrCopies * a.grid.ncells * P, (long long)cell * P + q, d);
    }
}

// v flag pass: one thread per x dof walks kVChunk v cells (in place)
template <int P, bool FAST, int IND>
__global__ void __launch_bounds__(kVThreads) post_v_kernel(const __grid_constant__ PostArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    const int xd = blockIdx.x * blockDim.x + threadIdx.x;
    const int sp = a.species0 + blockIdx.z;
    const int j0 = blockIdx.y * kVChunk, j1 = min(j0 + kVChunk, a.nv);
    const unsigned members = __ballot_sync(0xffffffffu, xd < a.nxd);
    __shared__ unsigned long long wqueue[kVThreads / 32][kQCap];
    unsigned long long* wq = wqueue[threadIdx.x >> 5];
    int wq_n = 0;
    if (xd < a.nxd) {
        const double* f = post_live(a, sp);
        double um[P], u0[P], up[P];
        // a v shard reads one halo cell from each neighbour (zero at the walls)
        const int lo = -a.gl, hi = a.nv + a.gr;
        vload<P>(f, a.ld, xd, j0 - 1, lo, hi, a.periodic, a.nv, um);
        vload<P>(f, a.ld, xd, j0, lo, hi, a.periodic, a.nv, u0);
        for (int j = j0; j < j1; ++j) {
            vload<P>(f, a.ld, xd, j + 1, lo, hi, a.periodic, a.nv, up);
            const bool tr[1] = {post_flag_t<P, FAST, IND>(a.cfg, a.basis, um, u0, up)};
            const unsigned long long entry[1] = {((unsigned long long)(sp & 1) << 63) |
                                                 ((unsigned long long)j << 32) | (unsigned)xd};
            wq_push<1>(wq, wq_n, a.fix_count, a.fix_cap, a.fix_list, tr, entry, members);
#pragma unroll
            for (int n = 0; n < P; ++n) {
                um[n] = u0[n];
                u0[n] = up[n];
            }
        }
        wq_flush(wq, wq_n, a.fix_count, a.fix_cap, a.fix_list, members);
    }
}

// overflow only: the field (with its readable v halo rows) into the other buffer
__global__ void post_copy_kernel(const __grid_constant__ PostArgs a, int P) {
    pdl_enter();
    if (halted(a.st)) return;
    if (*a.fix_count <= a.fix_cap) return;
    const long long r0 = -(long long)a.gl * P, r1 = (long long)(a.nv + a.gr) * P;
    const long long n = (r1 - r0) * a.ld;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (int k = 0; k < a.nspecies; ++k) {
        const int sp = a.species0 + k;
        const double* src = post_live(a, sp) + r0 * a.ld;
        double* dst = post_other(a, sp) + r0 * a.ld;
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i];
    }
}

// modifier of queued cells into fix_vals (or, after an overflow, of every
// re-flagged cell from the copy straight into the field)
template <int P, int DIR, bool FAST>
__global__ void __launch_bounds__(128) post_fix_kernel(const __grid_constant__ PostArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    const unsigned cnt = *a.fix_count;
    const bool rescan = cnt > a.fix_cap;
    const Grid& g = a.grid;
    const long long per_sp = DIR == 0 ? (long long)a.nrows * g.ncells : (long long)a.nv * a.nxd;
    const long long n = rescan ? (long long)a.nspecies * per_sp : (long long)cnt;
    unsigned flagged[2] = {0, 0};
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        int sp, row, col;  // x: row = line, col = cell; v: row = v cell, col = x dof
        bool cand = false;  // queued by a sweep whose stencil crossed its tile: decide here
        if (!rescan) {
            const unsigned long long e = a.fix_list[i];
            sp = (int)(e >> 63);
            cand = (e & kPostCandidate) != 0;
            row = (int)((e >> 32) & 0x3fffffffu);
            col = (int)(e & 0xffffffffu);
        } else {
            sp = a.species0 + (int)(i / per_sp);
            const long long r = i - (i / per_sp) * per_sp;
            const long long ncol = DIR == 0 ? g.ncells : a.nxd;
            row = (int)(r / ncol);
            col = (int)(r - (r / ncol) * ncol);
        }
        const double* f = rescan ? post_other(a, sp) : post_live(a, sp);
        double um[P], u0[P], up[P], o[P];
        long long at;  // first dof of the cell, stride ds between its nodes
        long long ds;
        if constexpr (DIR == 0) {
            int b = 0;
            while (col >= g.start[b + 1]) ++b;
            const long long lb = (long long)row * g.ncells * P;
            post_x_stencil<P>(a, f + lb, b, col - g.start[b], um, u0, up);
            at = lb + (long long)col * P;
            ds = 1;
        } else {
            const int lo = -a.gl, hi = a.nv + a.gr;
            vload<P>(f, a.ld, col, row - 1, lo, hi, a.periodic, a.nv, um);
            vload<P>(f, a.ld, col, row, lo, hi, a.periodic, a.nv, u0);
            vload<P>(f, a.ld, col, row + 1, lo, hi, a.periodic, a.nv, up);
            at = (long long)row * P * a.ld + col;
            ds = a.ld;
        }
        if ((rescan || cand) && !post_flag<P, FAST>(a.cfg, a.basis, um, u0, up)) {
            if (cand)  // not flagged: the scatter writes the cell's own values back
#pragma unroll
                for (int m = 0; m < P; ++m) a.fix_vals[i * P + m] = u0[m];
            continue;
        }
        post_modify<P, FAST>(a.cfg, a.basis, um, u0, up, o);
        if (rescan) {
            double* out = post_live(a, sp);
            if (DIR == 0 && a.rho_corr) post_rho_corr<P>(a, sp, row, col, u0, o);
#pragma unroll
            for (int m = 0; m < P; ++m) out[at + m * ds] = o[m];
        } else {
#pragma unroll
            for (int m = 0; m < P; ++m) a.fix_vals[i * P + m] = o[m];
        }
        flagged[sp & 1] += 1;
    }
    // limiter counters (post_troubled): block reduction, one atomic per block
    __shared__ unsigned acc[2];
    if (threadIdx.x < 2) acc[threadIdx.x] = 0;
    __syncthreads();
    for (int sp = 0; sp < 2; ++sp) {
        const unsigned v = __reduce_add_sync(0xffffffffu, flagged[sp]);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&acc[sp], v);
    }
    __syncthreads();
    if (threadIdx.x < 2 && acc[threadIdx.x])
        atomicAdd(&a.st->stats[threadIdx.x][3], (unsigned long long)acc[threadIdx.x]);
}

// the queued modifications into the field (list mode only)
template <int P, int DIR>
__global__ void __launch_bounds__(128) post_scatter_kernel(const __grid_constant__ PostArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    const unsigned cnt = *a.fix_count;
    if (cnt > a.fix_cap) return;
    const Grid& g = a.grid;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride) {
        const unsigned long long e = a.fix_list[i];
        const int sp = (int)(e >> 63);
        const int row = (int)((e >> 32) & 0x3fffffffu);
        const int col = (int)(e & 0xffffffffu);
        double* out = post_live(a, sp);
        const long long at = DIR == 0 ? ((long long)row * g.ncells + col) * P : (long long)row * P * a.ld + col;
        const long long ds = DIR == 0 ? 1 : a.ld;
        if (DIR == 0 && a.rho_corr) {  // the sweep's fused moment summed the unmodified cell
            double o0[P];
#pragma unroll
            for (int m = 0; m < P; ++m) o0[m] = out[at + m];
            post_rho_corr<P>(a, sp, row, col, o0, a.fix_vals + i * P);
        }
#pragma unroll
        for (int m = 0; m < P; ++m) out[at + m * ds] = a.fix_vals[i * P + m];
    }
}

__global__ void post_v_count_kernel(DevStatus* st, int mask, unsigned long long per_species) {
    pdl_enter();
    for (int sp = 0; sp < 2; ++sp)
        if ((mask >> sp) & 1) st->post_checked[sp] += per_species;
}

}  // namespace

// ===========================================================================
// launchers
// ===========================================================================
constexpr int kPdlDefault = 0;  // measured: no gain (profiles/r02_pdl.txt)
// Every launch of the step goes through here: programmatic stream serialisation
// lets the next kernel's CTAs be scheduled while this one's last wave drains
// (each kernel opens with pdl_enter(), which waits for the full completion and
// memory flush of its predecessor before any access). SK_PDL selects the mode
// (A/B measurement).
static int pdl_mode() {
    // SK_PDL: 0 off, 1 launch attribute + trigger at kernel entry, 2 attribute only
    static const int mode = [] {
        const char* e = std::getenv("SK_PDL");
        return e && *e ? std::atoi(e) : kPdlDefault;
    }();
    return mode;
}
static bool pdl_on() { return pdl_mode() != 0; }
// per device, before any launch or capture (sk_ctx_create)
cudaError_t launch_init_device() {
    const int trig = pdl_mode() == 1;
    return cudaMemcpyToSymbol(c_pdl_trigger, &trig, sizeof(int));
}
template <typename... KP, typename... A>
static cudaError_t pdl_launch(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = pdl_on() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

#define SK_DISPATCH_P(P_, CALL)                               \
    switch (P_) {                                             \
        case 1: { constexpr int PP = 1; CALL; } break;        \
        case 2: { constexpr int PP = 2; CALL; } break;        \
        case 3: { constexpr int PP = 3; CALL; } break;        \
        case 4: { constexpr int PP = 4; CALL; } break;        \
        case 5: { constexpr int PP = 5; CALL; } break;        \
        case 6: { constexpr int PP = 6; CALL; } break;        \
        case 7: { constexpr int PP = 7; CALL; } break;        \
        default: return cudaErrorInvalidValue;                \
    }

cudaError_t launch_xtab(const XTabArgs& a, cudaStream_t s) {
    dim3 grid((a.nlines + 127) / 128, a.nspecies);
    SK_DISPATCH_P(a.basis.p, (pdl_launch(xtab_kernel<PP>, grid, 128, 0, s, a)));
    return cudaGetLastError();
}

static int sm_count() {
    static int n[32] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!n[dev & 31]) cudaDeviceGetAttribute(&n[dev & 31], cudaDevAttrMultiProcessorCount, dev);
    return n[dev & 31];
}

// fast-mode DFMA variants exist for k <= 3 (P <= 4); other degrees always
// run the reference-order kernels
template <int P>
constexpr bool kHasFma = kHasFmaDev<P>;

template <int P, bool INLINE, bool RHO, bool FMA, int MODE = 0, int SRC = 0>
static cudaError_t configure_xsweep() {
    using Cf = XCfg<P>;
    static unsigned configured = 0;  // per-device bit
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(configured & (1u << (dev & 31)))) {
        cudaError_t e = cudaFuncSetAttribute(xsweep_kernel<P, INLINE, RHO, FMA, MODE, SRC>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)Cf::template smem<MODE>());
        if (e != cudaSuccess) return e;
        // full shared-memory carveout so two pipelines share each SM
        e = cudaFuncSetAttribute(xsweep_kernel<P, INLINE, RHO, FMA, MODE, SRC>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
        configured |= 1u << (dev & 31);
    }
    return cudaSuccess;
}

// persistent grid of one x-sweep variant: resident CTAs, and for the fused
// moment a multiple of the tiles per line (each CTA then always sees the same
// tile column, so the per-group partial rows sum in a fixed order)
// (the grid is sized from the SRC = 0 variant, so a source-fused sweep lays out
// the fused-moment partials exactly like xsweep_rho_groups expects)
template <int P, bool INLINE, bool RHO, bool FMA, int MODE = 0, int SRC = 0>
static cudaError_t xsweep_plan(const XSweepArgs& a, XSweepArgs& b, int& grid_out) {
    using Cf = XCfg<P>;
    constexpr int TT = Cf::T;
    if (cudaError_t e = configure_xsweep<P, INLINE, RHO, FMA, MODE, SRC>()) return e;
    if (SRC != 0)
        if (cudaError_t e = configure_xsweep<P, INLINE, RHO, FMA, MODE, 0>()) return e;
    b = a;
    b.tile_start[0] = 0;
    for (int i = 0; i < a.grid.nblocks; ++i)
        b.tile_start[i + 1] = b.tile_start[i] + (a.grid.cells[i] + TT - 1) / TT;
    const int ntl = b.tile_start[a.grid.nblocks];
    const long long ntot = (long long)a.nspecies * a.nlines * ntl;
    int blocks_per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, xsweep_kernel<P, INLINE, RHO, FMA, MODE, 0>,
                                                  (Cf::NC + 1) * 32, Cf::template smem<MODE>());
    long long grid = (long long)sm_count() * (blocks_per_sm > 0 ? blocks_per_sm : 1);
    if (RHO) {
        grid = grid >= ntl ? (grid / ntl) * ntl : ntl;
        const long long lines = (long long)a.nspecies * a.nlines;
        if (grid > lines * ntl) grid = lines * ntl;
    }
    if (grid > ntot) grid = ntot;
    grid_out = (int)grid;
    return cudaSuccess;
}

template <int P, bool INLINE, bool RHO, bool FMA, int MODE = 0, int SRC = 0>
static cudaError_t launch_xsweep_t(const XSweepArgs& a, cudaStream_t s) {
    XSweepArgs b;
    int grid = 0;
    if (cudaError_t e = xsweep_plan<P, INLINE, RHO, FMA, MODE, SRC>(a, b, grid)) return e;
    pdl_launch(xsweep_kernel<P, INLINE, RHO, FMA, MODE, SRC>, grid, (XCfg<P>::NC + 1) * 32, XCfg<P>::template smem<MODE>(), s, b);
    return cudaGetLastError();
}

template <int P>
static cudaError_t launch_xghost_t(const XSweepArgs& a, cudaStream_t s) {
    const long long warps = (long long)a.nspecies * a.nlines;
    const int grid = (int)((warps * 32 + 255) / 256);
    if (grid > 0) pdl_launch(xghost_kernel<P>, grid, 256, 0, s, a);
    return cudaGetLastError();
}

cudaError_t launch_xghost(const XSweepArgs& a, cudaStream_t s) {
    SK_DISPATCH_P(a.basis.p, return launch_xghost_t<PP>(a, s))
    return cudaErrorInvalidValue;
}

template <int P, bool INLINE, bool RHO, bool FMA>
static cudaError_t launch_xsweep_s(const XSweepArgs& a, cudaStream_t s) {
    if constexpr (!INLINE)
        if (a.post_x == 1 || a.post_x == 2) {  // (the host fuses only without a fused source)
            if (a.src_mode) return cudaErrorInvalidValue;
            return a.post_x == 1 ? launch_xsweep_t<P, false, RHO, FMA, 4, 0>(a, s)
                                 : launch_xsweep_t<P, false, RHO, FMA, 5, 0>(a, s);
        }
    if (a.src_mode == 1) return launch_xsweep_t<P, INLINE, RHO, FMA, 0, 1>(a, s);
    if constexpr (!RHO)  // (the second source half step rides in the second x sweep: no moment)
        if (a.src_mode == 2) return launch_xsweep_t<P, INLINE, RHO, FMA, 0, 2>(a, s);
    return launch_xsweep_t<P, INLINE, RHO, FMA>(a, s);
}
template <int P, bool INLINE, bool RHO>
static cudaError_t launch_xsweep_f(const XSweepArgs& a, cudaStream_t s) {
    if constexpr (kHasFma<P>)
        if (a.fma) return launch_xsweep_s<P, INLINE, RHO, true>(a, s);
    return launch_xsweep_s<P, INLINE, RHO, false>(a, s);
}

template <int P, bool INLINE, int MODE>
static int rho_groups_t(const XSweepArgs& a) {
    XSweepArgs b;
    int grid = 0, ntl = 0;
    cudaError_t e;
    if constexpr (MODE == 3) {
        if constexpr (kHasFma<P>)
            e = xsweep_plan<P, INLINE, true, true, 3>(a, b, grid);
        else
            return 0;
    } else if constexpr (MODE >= 4) {  // sweep + post flags (no inline limiter)
        if constexpr (kHasFma<P>)
            e = a.fma ? xsweep_plan<P, false, true, true, MODE>(a, b, grid)
                      : xsweep_plan<P, false, true, false, MODE>(a, b, grid);
        else
            e = xsweep_plan<P, false, true, false, MODE>(a, b, grid);
    } else if constexpr (kHasFma<P>) {
        e = a.fma ? xsweep_plan<P, INLINE, true, true>(a, b, grid) : xsweep_plan<P, INLINE, true, false>(a, b, grid);
    } else {
        e = xsweep_plan<P, INLINE, true, false>(a, b, grid);
    }
    if (e != cudaSuccess) return 0;
    ntl = b.tile_start[a.grid.nblocks];
    return grid / ntl;
}

int xsweep_rho_groups(const XSweepArgs& a, int fused) {
    if (fused) {
        if (a.inline_sldg) {
            SK_DISPATCH_P(a.basis.p, return (rho_groups_t<PP, true, 3>(a)))
        } else {
            SK_DISPATCH_P(a.basis.p, return (rho_groups_t<PP, false, 3>(a)))
        }
    } else if (a.inline_sldg) {
        SK_DISPATCH_P(a.basis.p, return (rho_groups_t<PP, true, 0>(a)))
    } else if (a.post_x == 1) {
        SK_DISPATCH_P(a.basis.p, return (rho_groups_t<PP, false, 4>(a)))
    } else if (a.post_x == 2) {
        SK_DISPATCH_P(a.basis.p, return (rho_groups_t<PP, false, 5>(a)))
    } else {
        SK_DISPATCH_P(a.basis.p, return (rho_groups_t<PP, false, 0>(a)))
    }
    return 0;
}

bool xsweep_fused_supported(int P) { return P >= 1 && P <= 4; }

// MODE 3 (two half sweeps fused, fast mode, always with the fused moment)
template <int P>
static cudaError_t launch_xsweep_fused_t(const XSweepArgs& a, cudaStream_t s) {
    if constexpr (kHasFma<P>) {
        if (a.inline_sldg) return launch_xsweep_t<P, true, true, true, 3>(a, s);
        return launch_xsweep_t<P, false, true, true, 3>(a, s);
    }
    return cudaErrorInvalidValue;
}
cudaError_t launch_xfix2(const XSweepArgs& a, cudaStream_t s) {
    if (!a.inline_sldg) return cudaSuccess;
    SK_DISPATCH_P(a.basis.p, (pdl_launch(xfix2_kernel<PP, kHasFma<PP>>, sm_count() * 4, 128, 0, s, a)));
    return cudaGetLastError();
}

cudaError_t launch_xsweep_fused(const XSweepArgs& a, cudaStream_t s) {
    if (!a.fma || !a.rho_fuse || a.periodic) return cudaErrorInvalidValue;
    SK_DISPATCH_P(a.basis.p, return launch_xsweep_fused_t<PP>(a, s))
    return cudaErrorInvalidValue;
}

// rho[x] = sum of the groups' partial rows + the clamp corrections. 32 x dofs
// per CTA, 8 threads per x dof each summing a fixed residue class of rows,
// combined in a fixed order: deterministic, and 64x more loads in flight than
// one thread per x dof.
constexpr int kRhoRedParts = 8;
__global__ void __launch_bounds__(32 * kRhoRedParts)
    rho_fused_reduce_kernel(const double* partial, const unsigned long long* corr, int groups, int nxd,
                            double* rho, const DevStatus* st, const int* gate, int gate_on) {
    pdl_enter();
    if (halted(st)) return;
    if (gate && ((*gate != 0) != (gate_on != 0))) return;
    __shared__ double sp[kRhoRedParts][32];
    __shared__ unsigned long long sh[kRhoRedParts][32], sl[kRhoRedParts][32];
    const int l = threadIdx.x & 31, q = threadIdx.x >> 5;
    const int xd = blockIdx.x * 32 + l;
    double acc = 0.0;
    unsigned long long ih = 0, il = 0;
    if (xd < nxd) {
#pragma unroll 4
        for (int k = q; k < groups; k += kRhoRedParts) acc += __ldg(partial + (long long)k * nxd + xd);
        // clamp corrections (rho_corr_add): integer sums are exact, so neither
        // the atomics' order nor the copy split changes rho
#pragma unroll 4
        for (int k = q; k < kRhoCorrCopies; k += kRhoRedParts) {
            ih += __ldg(corr + (long long)k * nxd + xd);
            il += __ldg(corr + (long long)(kRhoCorrCopies + k) * nxd + xd);
        }
    }
    sp[q][l] = acc;
    sh[q][l] = ih;
    sl[q][l] = il;
    __syncthreads();
    if (q == 0 && xd < nxd) {
        for (int j = 1; j < kRhoRedParts; ++j) {
            acc += sp[j][l];
            ih += sh[j][l];
            il += sl[j][l];
        }
        rho[xd] = acc + rho_corr_value(ih, il);
    }
}

cudaError_t launch_rho_fused_reduce(const XSweepArgs& a, double* rho, cudaStream_t s, int fused) {
    const int nxd = a.grid.ncells * a.basis.p;
    const int groups = xsweep_rho_groups(a, fused);
    pdl_launch(rho_fused_reduce_kernel, (nxd + 31) / 32, 32 * kRhoRedParts, 0, s, a.rho_partial, a.rho_corr, groups,
                                                                        nxd, rho, a.st, a.gate, a.gate_on);
    return cudaGetLastError();
}

cudaError_t launch_xsweep(const XSweepArgs& a, int /*ntiles*/, cudaStream_t s) {
    if (a.inline_sldg && a.rho_fuse)
        SK_DISPATCH_P(a.basis.p, return (launch_xsweep_f<PP, true, true>(a, s)))
    else if (a.inline_sldg)
        SK_DISPATCH_P(a.basis.p, return (launch_xsweep_f<PP, true, false>(a, s)))
    else if (a.rho_fuse)
        SK_DISPATCH_P(a.basis.p, return (launch_xsweep_f<PP, false, true>(a, s)))
    else
        SK_DISPATCH_P(a.basis.p, return (launch_xsweep_f<PP, false, false>(a, s)))
    return cudaSuccess;
}

template <int P>
static void launch_xfix_t(const XSweepArgs& a, cudaStream_t s) {
    if constexpr (kHasFma<P>)
        if (a.fma) {
            pdl_launch(xfix_kernel<P, true>, sm_count() * 8, 128, 0, s, a);
            return;
        }
    pdl_launch(xfix_kernel<P, false>, sm_count() * 8, 128, 0, s, a);
}
template <int P>
static void launch_vfix_t(const VSweepArgs& a, cudaStream_t s) {
    if constexpr (kHasFma<P>)
        if (a.fma) {
            pdl_launch(vfix_kernel<P, true>, sm_count() * 8, 128, 0, s, a);
            return;
        }
    pdl_launch(vfix_kernel<P, false>, sm_count() * 8, 128, 0, s, a);
}

cudaError_t launch_xfix(const XSweepArgs& a, cudaStream_t s) {
    SK_DISPATCH_P(a.basis.p, (launch_xfix_t<PP>(a, s)));
    return cudaGetLastError();
}

cudaError_t launch_vfix(const VSweepArgs& a, cudaStream_t s) {
    SK_DISPATCH_P(a.basis.p, (launch_vfix_t<PP>(a, s)));
    return cudaGetLastError();
}

cudaError_t launch_vtab(const VTabArgs& a, cudaStream_t s) {
    dim3 grid((a.nxd + 127) / 128, a.nspecies);
    SK_DISPATCH_P(a.basis.p, (pdl_launch(vtab_kernel<PP>, grid, 128, 0, s, a)));
    return cudaGetLastError();
}

template <int P, bool INLINE>
static void launch_vsweep_f(const VSweepArgs& a, dim3 grid, cudaStream_t s) {
    if constexpr (!INLINE) {
        if (a.post_v == 1 || a.post_v == 2) {  // (the host fuses only where FAST == the sweep's FMA)
            const bool f = kHasFma<P> && a.fma;
            if (a.post_v == 1)
                pdl_launch(f ? vsweep_kernel<P, false, false, kHasFma<P>, 1> : vsweep_kernel<P, false, false, false, 1>,
                           grid, kVThreads, 0, s, a);
            else
                pdl_launch(f ? vsweep_kernel<P, false, false, kHasFma<P>, 2> : vsweep_kernel<P, false, false, false, 2>,
                           grid, kVThreads, 0, s, a);
            return;
        }
    }
    if constexpr (kHasFma<P>)
        if (a.fma) {
            pdl_launch(vsweep_kernel<P, INLINE, false, true>, grid, kVThreads, 0, s, a);
            return;
        }
    pdl_launch(vsweep_kernel<P, INLINE, false, false>, grid, kVThreads, 0, s, a);
}

cudaError_t launch_vsweep(const VSweepArgs& a, cudaStream_t s) {
    const int nxb = (a.nxd + kVThreads - 1) / kVThreads;
    const int nch = a.nchunks > 0 ? a.nchunks : (a.n + kVChunk - 1) / kVChunk;
    dim3 grid = a.chunk_major ? dim3(nch, nxb, a.nspecies) : dim3(nxb, nch, a.nspecies);
    if (a.periodic)
        SK_DISPATCH_P(a.basis.p, (pdl_launch(vsweep_kernel<PP, true, true, false>, grid, kVThreads, 0, s, a)))
    else if (a.inline_sldg)
        SK_DISPATCH_P(a.basis.p, (launch_vsweep_f<PP, true>(a, grid, s)))
    else
        SK_DISPATCH_P(a.basis.p, (launch_vsweep_f<PP, false>(a, grid, s)))
    return cudaGetLastError();
}

cudaError_t launch_rho(const RhoArgs& a, int nspecies, cudaStream_t s) {
    dim3 grid((a.nxd + 127) / 128, a.nchunks, nspecies);
    SK_DISPATCH_P(a.basis.p, (pdl_launch(rho_partial_kernel<PP>, grid, 128, 0, s, a)));
    pdl_launch(rho_reduce_kernel, (a.nxd + 127) / 128, 128, 0, s, a);
    return cudaGetLastError();
}

// cluster shape for the Poisson solve: largest cluster (16 non-portable, else
// 8) the device can co-schedule with the needed shared memory; 0 = single CTA
template <int PS>
static int poisson_cluster_plan(const PoissonDev& pd, PClusterMap& cm, size_t& smem) {
    const int N = pd.ncells;
    if (getenv("SK_POISSON_CLUSTER_MIN")) {
        if (N < atoi(getenv("SK_POISSON_CLUSTER_MIN"))) return 0;
    } else if (N < 512) {  // (measured: C2's nx = 512 -2.5 % per step on the cluster, C1's 128 +9 %)
        return 0;
    }
    for (int C : {16, 8}) {
        if (N < 4 * C) continue;
        int Kmax = 0;
        const int per = (N + C - 1) / C;
        while ((2 << Kmax) <= per) ++Kmax;  // 2^K <= ceil(N/C)
        if (Kmax >= pd.nlevels - 1) Kmax = pd.nlevels - 2;
        // fewer CTA-local levels shrink the recomputed halos (2^K rows per side)
        // at the price of more rows for CTA 0's top levels: largest K that fits
        PClusterMap m{};
        size_t need = 0;
        for (int K = Kmax; K >= 1; --K) {
            if (K >= kPMaxLev - 1) continue;
            const int B = ((per + (1 << K) - 1) >> K) << K;
            const PClusterMap t{N, C, B, K};
            long long top = 0;
            for (int l = K; l < pd.nlevels; ++l) top += pd.level_n[l];
            int vmax = 0;
            for (int c = 0; c < C; ++c) {
                PRanges R;
                pc_ranges(t, pd.level_n, c, R);
                const int v = pc_vec_doubles(t, R, PS) + (c == 0 ? (int)(2 * top * PS) : 0);
                vmax = v > vmax ? v : vmax;
            }
            if (sizeof(double) * (size_t)vmax <= 220 * 1024) {
                m = t;
                need = sizeof(double) * (size_t)vmax;
                break;
            }
        }
        if (need == 0) continue;
        auto kern = poisson_cluster_kernel<PS>;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need) != cudaSuccess ||
            (C > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)) {
            cudaGetLastError();
            continue;
        }
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute attr{};
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = C;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.gridDim = dim3(C);
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = need;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters < 1) {
            cudaGetLastError();
            continue;
        }
        cm = m;
        smem = need;
        return C;
    }
    return 0;
}

template <int PS>
static cudaError_t launch_poisson_t(const PoissonDev& pd, int stage, const double* rho, double* E,
                                    double* phi, cudaStream_t s) {
    static int cached_n = -1, cached_c = 0;
    static PClusterMap cached_cm{};
    static size_t cached_smem = 0;
    if (cached_n != pd.ncells || getenv("SK_POISSON_SINGLE") || getenv("SK_POISSON_CLUSTER_MIN")) {
        cached_c = getenv("SK_POISSON_SINGLE") ? 0 : poisson_cluster_plan<PS>(pd, cached_cm, cached_smem);
        cached_n = pd.ncells;
    }
    if (cached_c == 0) {
        pdl_launch(poisson_kernel<PS>, 1, 1024, 0, s, pd, stage, rho, E, phi);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[2]{};
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cached_c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(cached_c);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = cached_smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_on() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, poisson_cluster_kernel<PS>, pd, cached_cm, stage, rho, E, phi);
}

cudaError_t launch_poisson(const PoissonDev& pd, int stage, const double* rho, double* E, double* phi,
                           cudaStream_t s) {
    SK_DISPATCH_P(pd.ps - 1, return (launch_poisson_t<PP + 1>(pd, stage, rho, E, phi, s)));
    return cudaErrorInvalidValue;
}

cudaError_t launch_rho_exact(const RhoArgs& a, cudaStream_t s) {
    SK_DISPATCH_P(a.basis.p, (pdl_launch(rho_exact_kernel<PP>, (a.nxd + kRhoThreads - 1) / kRhoThreads, kRhoThreads, 0, s, a)));
    return cudaGetLastError();
}

cudaError_t launch_poisson_exact(const PoissonDev& pd, const double* rho, double* E, double* phi,
                                 cudaStream_t s) {
    SK_DISPATCH_P(pd.ps - 1, (pdl_launch(poisson_exact_kernel<PP + 1>, 1, 256, 0, s, pd, rho, E, phi)));
    return cudaGetLastError();
}

// Step boundary n -> n+1 (before step_end of step n): the two x half sweeps
// around it may be fused unless the velocity cut-off checks at the end of
// step n -- checked only when its 10-step cooldown has run out (run.cpp:100),
// and a shrink there changes the v grid between the two sweeps.
__global__ void fuse_decide_kernel(DevStatus* st, int v_adjust, long long cooldown) {
    pdl_enter();
    if (halted(st)) return;
    const long long n = st->step + 1;
    int ok = 1;
    for (int sp = 0; sp < 2; ++sp)
        if (v_adjust && n - st->last_shrink[sp] >= cooldown) ok = 0;
    st->fuse_ok = ok;
}
// the unfused alternative of a fused boundary leaves the field in the buffer
// the fused sweep does not write: record it in the fields' flip flags
__global__ void flip_toggle_kernel(const DevStatus* st, int* f0, int* f1) {
    pdl_enter();
    if (halted(st) || st->fuse_ok) return;
    *f0 ^= 1;
    *f1 ^= 1;
}
cudaError_t launch_fuse_decide(DevStatus* st, int v_adjust, long long cooldown, cudaStream_t s) {
    pdl_launch(fuse_decide_kernel, 1, 1, 0, s, st, v_adjust, cooldown);
    return cudaGetLastError();
}
cudaError_t launch_flip_toggle(const DevStatus* st, int* f0, int* f1, cudaStream_t s) {
    pdl_launch(flip_toggle_kernel, 1, 1, 0, s, st, f0, f1);
    return cudaGetLastError();
}

cudaError_t launch_step_end(DevStatus* st, double dt, int v_adjust, long long cooldown, int mask,
                            cudaStream_t s) {
    pdl_launch(step_end_kernel, 1, 1, 0, s, st, dt, v_adjust, cooldown, mask);
    return cudaGetLastError();
}

// stepper.cpp:29-42 source_half_step with run.cpp:47-53's source: per node
// f += (0.5 half) (S(t) + S(t + half)), S = H(t0 - t) blob(x, v) / t0. The
// exponentials come from host tables (libm, as the reference computes them),
// indexed by the species' v-grid level (its shrink count), so the increment
// is bitwise the reference's.
__global__ void source_kernel(const __grid_constant__ SourceArgs a) {
    pdl_enter();
    if (halted(a.st)) return;
    const int sp = blockIdx.y;
    const double t = a.second ? a.st->time + a.half : a.st->time;
    if (!(t <= a.t0)) return;  // SourceTerm::active (stepper.hpp:19-21)
    const int lev = a.st->shrink_count[sp];
    if (lev >= kSourceLevels) {
        if (blockIdx.x == 0 && threadIdx.x == 0) raise_error(a.st, 1, 7, lev, kSourceLevels, a.st->step);
        return;
    }
    const double t2 = t + a.half;
    double* f = field_flipped(a.flip[sp]) ? a.alt[sp] : a.f[sp];
    const double* gv = a.gv[sp] + (long long)lev * a.nrows;
    const double w = 0.5 * a.half;
    const long long total = (long long)a.nrows * a.ld;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const long long r = i / a.ld;
        const int xd = (int)(i - r * a.ld);
        const double blob = a.gx[xd] * gv[r];  // run.cpp:19-22
        const double s1 = t > a.t0 ? 0.0 : blob / a.t0;
        const double s2 = t2 > a.t0 ? 0.0 : blob / a.t0;
        f[i] = f[i] + w * (s1 + s2);
    }
}

cudaError_t launch_source(const SourceArgs& a, cudaStream_t s) {
    pdl_launch(source_kernel, dim3(sm_count() * 8, 2), 256, 0, s, a);
    return cudaGetLastError();
}

cudaError_t launch_shrink(const ShrinkArgs& a, cudaStream_t s) {
    const int P = a.basis.p;
    // force: see ShrinkArgs
    if (a.force == 1 || a.force == -1) pdl_launch(shrink_force_kernel, 1, 1, 0, s, a.st, a.species_mask);
    if (a.force != 1 && a.force != 2)
        SK_DISPATCH_P(P, (pdl_launch(shrink_check_kernel<PP>, dim3((a.nxd + 255) / 256, 2), 256, 0, s, a)));
    if (a.force < 0) return cudaGetLastError();
    SK_DISPATCH_P(P, (pdl_launch(shrink_table_kernel<PP>, dim3((a.nv_global + 127) / 128, 2), 128, 0, s, a)));
    SK_DISPATCH_P(P, (pdl_launch(shrink_project_kernel<PP>, dim3(sm_count() * 8, 1, 2), kVThreads, 0, s, a)));
    pdl_launch(shrink_finalize_kernel, 1, 32, 0, s, a);
    return cudaGetLastError();
}

cudaError_t launch_diag(const DiagArgs& a, double* out4, double* partial, cudaStream_t s) {
    DiagArgs b = a;
    b.partial = partial;
    SK_DISPATCH_P(a.basis.p, (pdl_launch(diag_partial_kernel<PP>, kDiagBlocks, kDiagThreads, 0, s, b)));
    pdl_launch(diag_final_kernel, 1, 32, 0, s, partial, kDiagBlocks, out4);
    return cudaGetLastError();
}

cudaError_t launch_fill_separable(double* f, const double* gx, const double* gv, long long ld,
                                  int nrows, cudaStream_t s) {
    pdl_launch(fill_separable_kernel, 1184, 256, 0, s, f, gx, gv, ld, (long long)nrows * ld);
    return cudaGetLastError();
}

// after a flag pass: overflow copy (device-gated), modifications, scatter
template <int P, int DIR, bool FAST>
static void launch_post_tail(const PostArgs& a, cudaStream_t s) {
    pdl_launch(post_copy_kernel, sm_count() * 4, 256, 0, s, a, P);
    pdl_launch(post_fix_kernel<P, DIR, FAST>, sm_count() * 8, 128, 0, s, a);
    pdl_launch(post_scatter_kernel<P, DIR>, sm_count() * 4, 128, 0, s, a);
}

template <int P, bool FAST>
static cudaError_t launch_post_x_t(const PostArgs& a, cudaStream_t s) {
    // the x flag pass runs on the x-sweep pipeline (xsweep_kernel MODE 1)
    XSweepArgs x{};
    x.basis = a.basis;
    x.grid = a.grid;
    x.st = a.st;
    for (int sp = 0; sp < 2; ++sp) {
        x.src[sp] = a.src[sp];
        x.dst[sp] = a.dst[sp];
        x.flip[sp] = a.flip[sp];
    }
    x.nlines = a.nrows;
    x.nspecies = a.nspecies;
    x.species0 = a.species0;
    x.periodic = a.periodic;
    x.fma = a.fma;
    x.fix_list = a.fix_list;
    x.fix_count = a.fix_count;
    x.fix_cap = a.fix_cap;
    x.post = a.cfg;
    XSweepArgs b;
    int grid = 0;
    if (a.flags_queued) {  // the x sweep queued them (MODE 4 / 5)
    } else if (a.cfg.indicator == 1) {
        if (cudaError_t e = xsweep_plan<P, false, false, FAST, 1>(x, b, grid)) return e;
        if (grid > 0)
            pdl_launch(xsweep_kernel<P, false, false, FAST, 1>, grid, (XCfg<P>::NC + 1) * 32, XCfg<P>::template smem<1>(), s, b);
    } else {
        if (cudaError_t e = xsweep_plan<P, false, false, FAST, 2>(x, b, grid)) return e;
        if (grid > 0)
            pdl_launch(xsweep_kernel<P, false, false, FAST, 2>, grid, (XCfg<P>::NC + 1) * 32, XCfg<P>::template smem<2>(), s, b);
    }
    launch_post_tail<P, 0, FAST>(a, s);
    return cudaGetLastError();
}

template <int P, bool FAST>
static cudaError_t launch_post_v_t(const PostArgs& a, cudaStream_t s) {
    dim3 grid((a.nxd + kVThreads - 1) / kVThreads, (a.nv + kVChunk - 1) / kVChunk, a.nspecies);
    if (a.flags_queued) {
    } else if (a.cfg.indicator == 1) {
        pdl_launch(post_v_kernel<P, FAST, 1>, grid, kVThreads, 0, s, a);
    } else {
        pdl_launch(post_v_kernel<P, FAST, 2>, grid, kVThreads, 0, s, a);
    }
    launch_post_tail<P, 1, FAST>(a, s);
    return cudaGetLastError();
}

cudaError_t launch_post_x(const PostArgs& a, int ntiles, cudaStream_t s) {
    (void)ntiles;
    if (a.fma) {
        SK_DISPATCH_P(a.basis.p, if (cudaError_t e = launch_post_x_t<PP, true>(a, s)) return e)
    } else {
        SK_DISPATCH_P(a.basis.p, if (cudaError_t e = launch_post_x_t<PP, false>(a, s)) return e)
    }
    int mask = 0;
    for (int i = 0; i < a.nspecies; ++i) mask |= 1 << (a.species0 + i);
    pdl_launch(post_v_count_kernel, 1, 1, 0, s, a.st, mask, (unsigned long long)a.nrows * a.grid.ncells);
    return cudaGetLastError();
}

cudaError_t launch_post_v(const PostArgs& a, cudaStream_t s) {
    if (a.fma) {
        SK_DISPATCH_P(a.basis.p, if (cudaError_t e = launch_post_v_t<PP, true>(a, s)) return e)
    } else {
        SK_DISPATCH_P(a.basis.p, if (cudaError_t e = launch_post_v_t<PP, false>(a, s)) return e)
    }
    int mask = 0;
    for (int i = 0; i < a.nspecies; ++i) mask |= 1 << (a.species0 + i);
    pdl_launch(post_v_count_kernel, 1, 1, 0, s, a.st, mask, (unsigned long long)a.nv * a.nxd);
    return cudaGetLastError();
}

// stress variant of the benchmark input: f *= 1 + amp * xi,
// xi uniform in [-1, 1) from a counter-based hash of (seed, index) -- the
// same multiplicative noise as the reference's self-check perturbation, not
// its mt19937_64 sequence
namespace {
__global__ void perturb_kernel(double* f, long long n, unsigned long long seed, double amp) {
    pdl_enter();
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        unsigned long long z = seed + 0x9e3779b97f4a7c15ull * (unsigned long long)(i + 1);  // splitmix64
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        const double xi = (double)(z >> 11) * 0x1p-52 - 1.0;  // [-1, 1)
        f[i] *= 1.0 + amp * xi;
    }
}
}  // namespace
cudaError_t launch_perturb(double* f, size_t n, unsigned long long seed, double amp, cudaStream_t s) {
    pdl_launch(perturb_kernel, 1184, 256, 0, s, f, (long long)n, seed, amp);
    return cudaGetLastError();
}

cudaError_t launch_scale_copy(double* dst, const double* src, size_t n, cudaStream_t s) {
    pdl_launch(copy_kernel, 1184, 256, 0, s, dst, src, (long long)n);
    return cudaGetLastError();
}

}  // namespace sk
