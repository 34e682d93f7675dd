// bmc_kernels.cu -- sm_100a kernels of the Monte Carlo rollout path.
//
// Compiled with nvcc -gencode arch=compute_100a,code=sm_100a -fmad=false.
// Every FP64 operation of the rollout is spelled with an explicit _rn
// intrinsic, so the association order is the reference's
// (integrator.hpp:39-68, dynamics.hpp:115-132; paths under
// /root/reference/proj) regardless of compiler flags.
//
// Bound: the FP64 DADD/DMUL pipe.  Per RK4 step the
// reference formulation executes 57 FP64 flops; this kernel executes 32:
//   * the actuator lane (a, s2.a, s3.a, s4.a) is sample-independent and is
//     read from a per-batch table (bmc_host.cpp build_actuator_table): -21
//     (+ the table reaches an exact fixed point, after which the per-lane
//     clamped brake values are loop constants);
//   * k1 + 2.0*k2 is computed as fma(2.0, k2, k1): 2.0*k2 is exact in
//     binary64, so the single rounding of the FMA equals the reference's
//     rounding of the add, bit for bit (also for signed zeros): -4.
// Divergence from mixed stop times is removed by binning samples on a cheap
// FP32 prediction of their stop step (predict_kernel + counting sort), so a
// warp's lanes retire within a few steps of each other; warps pull sorted
// sample groups longest-first from a global counter (persistent CTAs).
// Launches of >= 1M samples run two chains per thread (samples i and i + 32
// of a 64-sample group share each table-row load); all table-mode loops use
// the blocked termination test (8 branch-free steps, exact replay on a hit).
// Measured: 95.8% FP64 pipe (ncu), profiles/round1_summary.md.
#include "bmc_kernels.h"
#include "bmc_rk4.cuh"

#include <cub/block/block_scan.cuh>

#include <climits>
#include <cstdlib>

namespace bmc {
namespace {

int sm_count_cached(int device);

// Actuator lane of rk4_step for the no-table fallback (dynamics.hpp:130).
__device__ __forceinline__ StageA actuator_stages(double a, double cmd, double inv_tau,
                                                  double dt, double half, double sixth,
                                                  double* a_next) {
    const double k1 = __dmul_rn(__dsub_rn(cmd, a), inv_tau);
    const double s2 = __dadd_rn(a, __dmul_rn(half, k1));
    const double k2 = __dmul_rn(__dsub_rn(cmd, s2), inv_tau);
    const double s3 = __dadd_rn(a, __dmul_rn(half, k2));
    const double k3 = __dmul_rn(__dsub_rn(cmd, s3), inv_tau);
    const double s4 = __dadd_rn(a, __dmul_rn(dt, k3));
    const double k4 = __dmul_rn(__dsub_rn(cmd, s4), inv_tau);
    const double c = __dadd_rn(__fma_rn(2.0, k3, __fma_rn(2.0, k2, k1)), k4);
    *a_next = __dadd_rn(a, __dmul_rn(sixth, c));
    return StageA{a, s2, s3, s4};
}

template <int MODE>
__device__ __forceinline__ StageA load_stage(const StageA* tab, int n) {
    if (MODE == kTableGlobal) {
        const double2* p = reinterpret_cast<const double2*>(tab) + 2 * n;
        const double2 lo = __ldg(p), hi = __ldg(p + 1);
        return StageA{lo.x, lo.y, hi.x, hi.y};
    } else {
        const double2* p = reinterpret_cast<const double2*>(tab) + 2 * n;
        const double2 lo = p[0], hi = p[1];
        return StageA{lo.x, lo.y, hi.x, hi.y};
    }
}

template <int MODE>
__device__ __forceinline__ double stage_value(const StageA* tab, int n, int s) {
    const double* p = reinterpret_cast<const double*>(tab) + 4 * n + s;
    return MODE == kTableGlobal ? __ldg(p) : *p;
}

// First step n at which clamp_brake(A_s[n], F) == F, i.e. !(A_s[n] > F).
// The host only hands over tables that are non-increasing in n for every
// stage, so the predicate is monotone and clamp_brake(A_s[n], F) equals
// (n < c_s ? A_s[n] : F) for every n -- bit for bit, including NaN F.
template <int MODE>
__device__ __forceinline__ int crossover(const StageA* tab, int len, int s, double F) {
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (stage_value<MODE>(tab, mid, s) > F) {
            lo = mid + 1;
        } else {
            hi = mid;
        }
    }
    return lo == len ? INT_MAX : lo;
}

struct LaneOut {
    double x;
    int32_t steps;
    bool stopped;
};

// One result: a packed 16-byte record in sorted order (binned schedule), or
// the compact SoA outputs at the sample's index.
__device__ __forceinline__ void store_out(const RolloutArgs& A, uint64_t j, const LaneOut& r) {
    if (A.packed_out) {
        PackedOut o;
        o.x = r.x;
        o.steps = r.steps;
        o.hit_horizon = r.stopped ? 0u : 1u;
        A.packed_out[j] = o;
        return;
    }
    if (A.stop_distance) A.stop_distance[j] = r.x;
    if (A.steps) A.steps[j] = r.steps;
    if (A.hit_horizon) A.hit_horizon[j] = r.stopped ? 0 : 1;
}

// simulate_rollout (integrator.cpp:13-29) for sample j, table modes.  The
// step loop is split at warp-uniform bounds so that almost every step runs
// a body with no clamp selects at all:
//   V1 [0, cmin_w)       brake = table stage values      (no lane clamped yet)
//   V2 [cmin_w, cmax_w)  brake = n < c_s ? table : floor (crossover band)
//   V3 [.., max_steps)   brake = per-lane constants      (all lanes clamped, or
//                        past the actuator fixed point)
struct Chain {
    double x, v, D, G, F;
    int c0, c1, c2, c3;
};

template <int MODE>
__device__ __forceinline__ void load_chain(const RolloutArgs& A, const StageA* tab, int len,
                                           uint64_t j, bool ok, Chain& c) {
    if (ok) {
        if (A.packed_in) {
            const double2* p = reinterpret_cast<const double2*>(A.packed_in + j);
            const double2 lo = __ldg(p), hi = __ldg(p + 1);
            c.v = lo.x;
            c.F = lo.y;
            c.D = hi.x;
            c.G = hi.y;
        } else {
            c.D = A.drag[j];
            c.G = A.grade[j];
            c.F = A.brake_floor[j];
            c.v = A.v0[j];
        }
        c.c0 = crossover<MODE>(tab, len, 0, c.F);
        c.c1 = crossover<MODE>(tab, len, 1, c.F);
        c.c2 = crossover<MODE>(tab, len, 2, c.F);
        c.c3 = crossover<MODE>(tab, len, 3, c.F);
    } else {
        // inert filler: stops after one step, never clamps, never written
        c.D = 0.0;
        c.G = 0.0;
        c.F = 0.0;
        c.v = -1.0;
        c.c0 = c.c1 = c.c2 = c.c3 = INT_MAX;
    }
    c.x = 0.0;
}

__device__ __forceinline__ int chain_cmin(const Chain& c) {
    return min(min(c.c0, c.c1), min(c.c2, c.c3));
}
__device__ __forceinline__ int chain_cmax(const Chain& c) {
    return max(max(c.c0, c.c1), max(c.c2, c.c3));
}

// The step loop of one chain from step n (its state after n steps) with the
// warp-uniform phase bounds p1 <= p2 <= head.
template <int MODE>
__device__ __forceinline__ LaneOut steps_from(const RolloutArgs& A, const StageA* tab, int len,
                                              Chain& c, int32_t n, int p1, int p2) {
    const int32_t M = A.max_steps;
    if (n < p2) {
        // the next table row is fetched one step ahead (n + 1 <= head <= len - 1)
        StageA nx = load_stage<MODE>(tab, n);
        for (; n < p1; ++n) {
            const StageA s = nx;
            nx = load_stage<MODE>(tab, n + 1);
            rk4_xv(c.x, c.v, s.a0, s.a1, s.a2, s.a3, c.D, c.G, A.dt, A.half, A.sixth);
            if (not_positive(c.v)) return LaneOut{c.x, n + 1, true};
        }
        for (; n < p2; ++n) {
            const StageA s = nx;
            nx = load_stage<MODE>(tab, n + 1);
            rk4_xv(c.x, c.v, n < c.c0 ? s.a0 : c.F, n < c.c1 ? s.a1 : c.F,
                   n < c.c2 ? s.a2 : c.F, n < c.c3 ? s.a3 : c.F, c.D, c.G, A.dt, A.half,
                   A.sixth);
            if (not_positive(c.v)) return LaneOut{c.x, n + 1, true};
        }
    }
    if (n < M) {
        const StageA s = load_stage<MODE>(tab, len - 1);
        const double b0 = c.c0 <= n ? c.F : s.a0, b1 = c.c1 <= n ? c.F : s.a1;
        const double b2 = c.c2 <= n ? c.F : s.a2, b3 = c.c3 <= n ? c.F : s.a3;
        for (; n < M; ++n) {
            rk4_xv(c.x, c.v, b0, b1, b2, b3, c.D, c.G, A.dt, A.half, A.sixth);
            if (not_positive(c.v)) return LaneOut{c.x, n + 1, true};
        }
    }
    return LaneOut{c.x, M, false};
}

// Blocked termination test (UNR = kTestBlock): the V1 and V3 loops run
// kTestBlock steps with no branch, folding hi_word(v) into a running
// minimum; a lane whose minimum says it may have stopped replays the block
// from its saved start state with the exact per-step test, so it returns
// exactly the step and position simulate_rollout returns (integrator.cpp:
// 20-26).  A false alarm (a positive subnormal v) replays to the identical
// state and carries on.  Removing the per-step branch takes ~25 cycles off
// each step's dependent chain (latency-bound small batches) and issue slots
// off the FP64 pipe (tools/rk4_step_probe.cu).
constexpr int kTestBlock = 8;

template <int MODE>
__device__ __forceinline__ LaneOut steps_from_blocked(const RolloutArgs& A, const StageA* tab,
                                                      int len, Chain& c, int32_t n, int p1,
                                                      int p2) {
    const int32_t M = A.max_steps;
    if (n < p2) {
        StageA nx = load_stage<MODE>(tab, n);  // row n; rows n+1.. fetched one step ahead
        for (; n + kTestBlock <= p1; n += kTestBlock) {
            const double x0 = c.x, v0 = c.v;
            int m = INT_MAX;
#pragma unroll
            for (int k = 0; k < kTestBlock; ++k) {
                const StageA s = nx;
                nx = load_stage<MODE>(tab, n + k + 1);  // n + k + 1 <= p1 <= head <= len - 1
                rk4_xv(c.x, c.v, s.a0, s.a1, s.a2, s.a3, c.D, c.G, A.dt, A.half, A.sixth);
                m = min(m, hi_word(c.v));
            }
            if (m <= 0) {
                c.x = x0;
                c.v = v0;
#pragma unroll 1
                for (int k = 0; k < kTestBlock; ++k) {
                    const StageA s = load_stage<MODE>(tab, n + k);
                    rk4_xv(c.x, c.v, s.a0, s.a1, s.a2, s.a3, c.D, c.G, A.dt, A.half, A.sixth);
                    if (not_positive(c.v)) return LaneOut{c.x, n + k + 1, true};
                }
            }
        }
        for (; n < p1; ++n) {
            const StageA s = nx;
            nx = load_stage<MODE>(tab, n + 1);
            rk4_xv(c.x, c.v, s.a0, s.a1, s.a2, s.a3, c.D, c.G, A.dt, A.half, A.sixth);
            if (not_positive(c.v)) return LaneOut{c.x, n + 1, true};
        }
        for (; n < p2; ++n) {
            const StageA s = nx;
            nx = load_stage<MODE>(tab, n + 1);
            rk4_xv(c.x, c.v, n < c.c0 ? s.a0 : c.F, n < c.c1 ? s.a1 : c.F,
                   n < c.c2 ? s.a2 : c.F, n < c.c3 ? s.a3 : c.F, c.D, c.G, A.dt, A.half,
                   A.sixth);
            if (not_positive(c.v)) return LaneOut{c.x, n + 1, true};
        }
    }
    if (n < M) {
        const StageA s = load_stage<MODE>(tab, len - 1);
        const double b0 = c.c0 <= n ? c.F : s.a0, b1 = c.c1 <= n ? c.F : s.a1;
        const double b2 = c.c2 <= n ? c.F : s.a2, b3 = c.c3 <= n ? c.F : s.a3;
        for (; n + kTestBlock <= M; n += kTestBlock) {
            const double x0 = c.x, v0 = c.v;
            int m = INT_MAX;
#pragma unroll
            for (int k = 0; k < kTestBlock; ++k) {
                rk4_xv(c.x, c.v, b0, b1, b2, b3, c.D, c.G, A.dt, A.half, A.sixth);
                m = min(m, hi_word(c.v));
            }
            if (m <= 0) {
                c.x = x0;
                c.v = v0;
#pragma unroll 1
                for (int k = 0; k < kTestBlock; ++k) {
                    rk4_xv(c.x, c.v, b0, b1, b2, b3, c.D, c.G, A.dt, A.half, A.sixth);
                    if (not_positive(c.v)) return LaneOut{c.x, n + k + 1, true};
                }
            }
        }
        for (; n < M; ++n) {
            rk4_xv(c.x, c.v, b0, b1, b2, b3, c.D, c.G, A.dt, A.half, A.sixth);
            if (not_positive(c.v)) return LaneOut{c.x, n + 1, true};
        }
    }
    return LaneOut{c.x, M, false};
}

template <int MODE, int UNR>
__device__ __forceinline__ LaneOut run_table(const RolloutArgs& A, const StageA* tab, int len,
                                             uint64_t j, unsigned mask) {
    Chain c;
    load_chain<MODE>(A, tab, len, j, true, c);
    const int head = min(len - 1, A.max_steps);
    const int p1 = min(__reduce_min_sync(mask, chain_cmin(c)), head);
    const int p2 = min(__reduce_max_sync(mask, chain_cmax(c)), head);
    if (UNR == kTestBlock) return steps_from_blocked<MODE>(A, tab, len, c, 0, p1, p2);
    return steps_from<MODE>(A, tab, len, c, 0, p1, p2);
}

// Two independent samples per thread (ILP = 2): the lanes of a warp own a
// sorted 64-sample group (i and i + 32), so both chains of a thread stop
// within a few steps of each other.  Both chains step together until the
// first one stops (one combined termination test per step, no per-chain
// latching in the hot loop); the survivor then finishes on the single-chain
// loop from that step.  Shared per-thread state (table row, loop control)
// is amortised over two dependency chains: one table-row load feeds both.
// BLK: the V1 and V3 loops use the blocked termination test of
// steps_from_blocked (running minimum over both chains, exact replay).
// First step n from which every stage brake value of this chain is <= G,
// i.e. every RK4 stage acceleration b - D*s^2 - G is <= 0 (exactly also in
// rounding: fl(fl(b - p) - G) <= fl(b - G) <= 0 for p >= 0).  The stage
// brake is max(A_s[n], F) (the crossover form of clamp_brake) and every
// stage sequence is non-increasing (host-checked), so the row maximum is
// too: binary search.  INT_MAX when it never happens (F > G: a downhill
// grade the brakes cannot hold, or NaN).
template <int MODE>
__device__ __forceinline__ int monotone_from(const StageA* tab, int len, double F, double G) {
    if (!(F <= G)) return INT_MAX;
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const StageA s = load_stage<MODE>(tab, mid);
        const double mx = fmax(fmax(s.a0, s.a1), fmax(s.a2, s.a3));
        if (mx > G) {
            lo = mid + 1;
        } else {
            hi = mid;
        }
    }
    return lo == len ? INT_MAX : lo;
}

// Blocked steps of both chains, L steps from row n.  PER_STEP: fold
// hi_word(v) of every step into the running minimum (exact detection of the
// first v <= 0).  Otherwise only the block's last speeds are tested: valid
// when every acceleration in the block is <= 0 (monotone_from), because then
// v is non-increasing -- rounding included: v + fl(h/6 * cv) with cv <= 0 --
// so a speed that reached <= 0 inside the block is still <= 0 at its end, and
// the exact replay finds the first such step.  The monotone blocks are also
// longer (kMonoBlock): the FP64 pipe binds and every other instruction in the
// loop (termination test, block bookkeeping) costs an issue cycle the pipe
// would have used (profiles/round2_summary.md).
#ifndef BMC_MONO_BLOCK
#define BMC_MONO_BLOCK 16
#endif
constexpr int kMonoBlock = BMC_MONO_BLOCK;

template <int MODE, int L, bool PER_STEP>
__device__ __forceinline__ int block_table(const RolloutArgs& A, const StageA* row, Chain& a,
                                           Chain& b) {
    int m = INT_MAX;
#pragma unroll
    for (int k = 0; k < L; ++k) {
        const StageA s = load_stage<MODE>(row, k);
        rk4_xv(a.x, a.v, s.a0, s.a1, s.a2, s.a3, a.D, a.G, A.dt, A.half, A.sixth);
        rk4_xv(b.x, b.v, s.a0, s.a1, s.a2, s.a3, b.D, b.G, A.dt, A.half, A.sixth);
        if (PER_STEP) m = min(m, min(hi_word(a.v), hi_word(b.v)));
    }
    return PER_STEP ? m : min(hi_word(a.v), hi_word(b.v));
}

template <int L, bool PER_STEP>
__device__ __forceinline__ int block_const(const RolloutArgs& A, Chain& a, Chain& b, double a0,
                                           double a1, double a2, double a3, double b0, double b1,
                                           double b2, double b3) {
    int m = INT_MAX;
#pragma unroll
    for (int k = 0; k < L; ++k) {
        rk4_xv(a.x, a.v, a0, a1, a2, a3, a.D, a.G, A.dt, A.half, A.sixth);
        rk4_xv(b.x, b.v, b0, b1, b2, b3, b.D, b.G, A.dt, A.half, A.sixth);
        if (PER_STEP) m = min(m, min(hi_word(a.v), hi_word(b.v)));
    }
    return PER_STEP ? m : min(hi_word(a.v), hi_word(b.v));
}

// Exact replay of up to L table steps from row n after a block test fired:
// true with n advanced to the first step where either chain's v <= 0;
// false (a false alarm: positive subnormal) with the state at the block end.
template <int MODE>
__device__ __forceinline__ bool replay_table(const RolloutArgs& A, const StageA* tab, Chain& a,
                                             Chain& b, int32_t& n, int L) {
#pragma unroll 1
    for (int k = 0; k < L; ++k) {
        const StageA s = load_stage<MODE>(tab, n + k);
        rk4_xv(a.x, a.v, s.a0, s.a1, s.a2, s.a3, a.D, a.G, A.dt, A.half, A.sixth);
        rk4_xv(b.x, b.v, s.a0, s.a1, s.a2, s.a3, b.D, b.G, A.dt, A.half, A.sixth);
        if (not_positive(a.v) | not_positive(b.v)) {
            n += k;
            return true;
        }
    }
    return false;
}

__device__ __forceinline__ bool replay_const(const RolloutArgs& A, Chain& a, Chain& b,
                                             int32_t& n, int L, double a0, double a1, double a2,
                                             double a3, double b0, double b1, double b2,
                                             double b3) {
#pragma unroll 1
    for (int k = 0; k < L; ++k) {
        rk4_xv(a.x, a.v, a0, a1, a2, a3, a.D, a.G, A.dt, A.half, A.sixth);
        rk4_xv(b.x, b.v, b0, b1, b2, b3, b.D, b.G, A.dt, A.half, A.sixth);
        if (not_positive(a.v) | not_positive(b.v)) {
            n += k;
            return true;
        }
    }
    return false;
}

template <int MODE, bool BLK>
__device__ __forceinline__ void run_table2(const RolloutArgs& A, const StageA* tab, int len,
                                           uint64_t j0, uint64_t j1, bool ok0, bool ok1,
                                           LaneOut& r0, LaneOut& r1) {
    Chain a, b;
    load_chain<MODE>(A, tab, len, j0, ok0, a);
    load_chain<MODE>(A, tab, len, j1, ok1, b);
    const int32_t M = A.max_steps;
    const int head = min(len - 1, M);
    const int lmin = min(ok0 ? chain_cmin(a) : INT_MAX, ok1 ? chain_cmin(b) : INT_MAX);
    const int lmax = max(ok0 ? chain_cmax(a) : INT_MIN, ok1 ? chain_cmax(b) : INT_MIN);
    const int p1 = min(__reduce_min_sync(0xffffffffu, lmin), head);
    const int p2 = max(min(__reduce_max_sync(0xffffffffu, lmax), head), p1);
    // warp-uniform step from which the table blocks may test only their end
    int ps = INT_MAX;
    if (BLK && A.monotone_blocks) {
        const int ma = ok0 ? monotone_from<MODE>(tab, len, a.F, a.G) : 0;
        const int mb = ok1 ? monotone_from<MODE>(tab, len, b.F, b.G) : 0;
        ps = __reduce_max_sync(0xffffffffu, max(ma, mb));
    }
    int32_t n = 0;
    bool hit = false;
    if (n < p2) {
        if (BLK) {
            // per-step test until the warp's chains are all monotone ...
            for (; n < ps && n + kTestBlock <= p1; n += kTestBlock) {
                const double xa0 = a.x, va0 = a.v, xb0 = b.x, vb0 = b.v;
                if (block_table<MODE, kTestBlock, true>(A, tab + n, a, b) <= 0) {
                    a.x = xa0, a.v = va0, b.x = xb0, b.v = vb0;
                    if ((hit = replay_table<MODE>(A, tab, a, b, n, kTestBlock))) break;
                }
            }
            // ... then longer blocks that test only their last speeds
            for (; !hit && n + kMonoBlock <= p1; n += kMonoBlock) {
                const double xa0 = a.x, va0 = a.v, xb0 = b.x, vb0 = b.v;
                if (block_table<MODE, kMonoBlock, false>(A, tab + n, a, b) <= 0) {
                    a.x = xa0, a.v = va0, b.x = xb0, b.v = vb0;
                    if ((hit = replay_table<MODE>(A, tab, a, b, n, kMonoBlock))) break;
                }
            }
        }
        StageA nx = load_stage<MODE>(tab, n);
        for (; !hit && n < p1; ++n) {
            const StageA s = nx;
            nx = load_stage<MODE>(tab, n + 1);
            rk4_xv(a.x, a.v, s.a0, s.a1, s.a2, s.a3, a.D, a.G, A.dt, A.half, A.sixth);
            rk4_xv(b.x, b.v, s.a0, s.a1, s.a2, s.a3, b.D, b.G, A.dt, A.half, A.sixth);
            if (not_positive(a.v) | not_positive(b.v)) {
                hit = true;
                break;
            }
        }
        if (!hit) {
            for (; n < p2; ++n) {
                const StageA s = nx;
                nx = load_stage<MODE>(tab, n + 1);
                rk4_xv(a.x, a.v, n < a.c0 ? s.a0 : a.F, n < a.c1 ? s.a1 : a.F,
                       n < a.c2 ? s.a2 : a.F, n < a.c3 ? s.a3 : a.F, a.D, a.G, A.dt, A.half,
                       A.sixth);
                rk4_xv(b.x, b.v, n < b.c0 ? s.a0 : b.F, n < b.c1 ? s.a1 : b.F,
                       n < b.c2 ? s.a2 : b.F, n < b.c3 ? s.a3 : b.F, b.D, b.G, A.dt, A.half,
                       A.sixth);
                if (not_positive(a.v) | not_positive(b.v)) {
                    hit = true;
                    break;
                }
            }
        }
    }
    if (!hit && n < M) {
        const StageA s = load_stage<MODE>(tab, len - 1);
        const double a0 = a.c0 <= n ? a.F : s.a0, a1 = a.c1 <= n ? a.F : s.a1;
        const double a2 = a.c2 <= n ? a.F : s.a2, a3 = a.c3 <= n ? a.F : s.a3;
        const double b0 = b.c0 <= n ? b.F : s.a0, b1 = b.c1 <= n ? b.F : s.a1;
        const double b2 = b.c2 <= n ? b.F : s.a2, b3 = b.c3 <= n ? b.F : s.a3;
        if (BLK) {
            // the constant stage brakes are F or the table's last row: every
            // one is <= G iff monotone_from found a step (warp-uniform; this
            // region is entered by a divergent subset of lanes, no votes here)
            if (ps != INT_MAX) {
                for (; n + kMonoBlock <= M; n += kMonoBlock) {
                    const double xa0 = a.x, va0 = a.v, xb0 = b.x, vb0 = b.v;
                    if (block_const<kMonoBlock, false>(A, a, b, a0, a1, a2, a3, b0, b1, b2, b3) <= 0) {
                        a.x = xa0, a.v = va0, b.x = xb0, b.v = vb0;
                        if ((hit = replay_const(A, a, b, n, kMonoBlock, a0, a1, a2, a3, b0, b1, b2, b3))) break;
                    }
                }
            } else {
                for (; n + kTestBlock <= M; n += kTestBlock) {
                    const double xa0 = a.x, va0 = a.v, xb0 = b.x, vb0 = b.v;
                    if (block_const<kTestBlock, true>(A, a, b, a0, a1, a2, a3, b0, b1, b2, b3) <= 0) {
                        a.x = xa0, a.v = va0, b.x = xb0, b.v = vb0;
                        if ((hit = replay_const(A, a, b, n, kTestBlock, a0, a1, a2, a3, b0, b1, b2, b3))) break;
                    }
                }
            }
        }
        for (; !hit && n < M; ++n) {
            rk4_xv(a.x, a.v, a0, a1, a2, a3, a.D, a.G, A.dt, A.half, A.sixth);
            rk4_xv(b.x, b.v, b0, b1, b2, b3, b.D, b.G, A.dt, A.half, A.sixth);
            if (not_positive(a.v) | not_positive(b.v)) {
                hit = true;
                break;
            }
        }
    }
    if (!hit) {  // both reached the horizon
        r0 = LaneOut{a.x, M, false};
        r1 = LaneOut{b.x, M, false};
        return;
    }
    const bool sa = not_positive(a.v), sb = not_positive(b.v);
    if (sa) r0 = LaneOut{a.x, n + 1, true};
    if (sb) r1 = LaneOut{b.x, n + 1, true};
    if (sa && sb) return;
    // finish the survivor from step n + 1 on the single-chain loop
    Chain& c = sa ? b : a;
    const LaneOut r = BLK ? steps_from_blocked<MODE>(A, tab, len, c, n + 1, p1, p2)
                          : steps_from<MODE>(A, tab, len, c, n + 1, p1, p2);
    if (sa) {
        r1 = r;
    } else {
        r0 = r;
    }
}

// Generic path (no usable table): the actuator lane is integrated inline
// exactly as the reference does, with the ternary clamp on every stage.
__device__ __forceinline__ LaneOut run_inline(const RolloutArgs& A, uint64_t j) {
    const double D = A.drag[j];
    const double G = A.grade[j];
    const double F = A.brake_floor[j];
    double v = A.v0[j];
    double x = 0.0;
    double a = 0.0;
    const int32_t M = A.max_steps;
    for (int32_t n = 0; n < M; ++n) {
        double an;
        const StageA s = actuator_stages(a, A.brake_cmd, A.inv_tau, A.dt, A.half, A.sixth, &an);
        rk4_xv(x, v, clamp_brake(s.a0, F), clamp_brake(s.a1, F), clamp_brake(s.a2, F),
               clamp_brake(s.a3, F), D, G, A.dt, A.half, A.sixth);
        a = an;
        if (v <= 0.0) return LaneOut{x, n + 1, true};
    }
    return LaneOut{x, M, false};
}

template <int MODE, int BT, int ILP, int UNR>
__global__ void __launch_bounds__(BT, 1) rollout_kernel(const RolloutArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const StageA* tab = A.table;
    const int len = A.table_len;
    if (MODE == kTableShared) {
        const double2* src = reinterpret_cast<const double2*>(A.table);
        double2* dst = reinterpret_cast<double2*>(smem_raw);
        for (int i = threadIdx.x; i < 2 * len; i += blockDim.x) dst[i] = src[i];
        tab = reinterpret_cast<const StageA*>(smem_raw);
    }
    // fused statistics pass 1: per-CTA partials after the table
    const bool fused = A.p1.sum != nullptr;
    const P1View sv = p1_view(smem_raw + (MODE == kTableShared ? static_cast<size_t>(len) * sizeof(StageA) : 0),
                              A.p1.m);
    if (fused) p1_init(sv, A.p1);
    if (MODE == kTableShared || fused) __syncthreads();
    const unsigned lane = threadIdx.x & 31u;
    unsigned long long my_steps = 0, my_slots = 0;
    for (;;) {
        unsigned g = 0;
        if (lane == 0) g = atomicAdd(A.work_counter, 1u);
        g = __shfl_sync(0xffffffffu, g, 0);
        const uint64_t base = static_cast<uint64_t>(g) * (32u * ILP);
        if (base >= A.n) break;
        if (ILP == 2) {
            const uint64_t i0 = base + lane, i1 = i0 + 32u;
            const bool ok0 = i0 < A.n, ok1 = i1 < A.n;
            const uint64_t j0 = ok0 ? (A.perm ? static_cast<uint64_t>(A.perm[i0]) : i0) : 0;
            const uint64_t j1 = ok1 ? (A.perm ? static_cast<uint64_t>(A.perm[i1]) : i1) : 0;
            LaneOut r0, r1;
            run_table2<MODE, UNR == kTestBlock>(A, tab, len, j0, j1, ok0, ok1, r0, r1);
            // outputs at the sample's own index (binned: through the forward map)
            const uint64_t o0 = (ok0 && A.fwd) ? static_cast<uint64_t>(A.fwd[j0]) : j0;
            const uint64_t o1 = (ok1 && A.fwd) ? static_cast<uint64_t>(A.fwd[j1]) : j1;
            if (ok0) {
                store_out(A, o0, r0);
                my_steps += static_cast<unsigned>(max(r0.steps, 0));
                if (fused) p1_add(sv, A.p1.m, r0.x, !r0.stopped);
            }
            if (ok1) {
                store_out(A, o1, r1);
                my_steps += static_cast<unsigned>(max(r1.steps, 0));
                if (fused) p1_add(sv, A.p1.m, r1.x, !r1.stopped);
            }
            const int lmax = max(ok0 ? r0.steps : 0, ok1 ? r1.steps : 0);
            const unsigned gmax = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(max(lmax, 0)));
            const unsigned chains = __popc(__ballot_sync(0xffffffffu, ok0)) +
                                    __popc(__ballot_sync(0xffffffffu, ok1));
            if (lane == 0) my_slots += static_cast<unsigned long long>(gmax) * chains;
            continue;
        }
        const uint64_t i = base + lane;
        const unsigned mask = __ballot_sync(0xffffffffu, i < A.n);
        if (i < A.n) {
            const uint64_t j = A.perm ? static_cast<uint64_t>(A.perm[i]) : i;
            const LaneOut r = MODE == kTableNone ? run_inline(A, j) : run_table<MODE, UNR>(A, tab, len, j, mask);
            store_out(A, A.fwd ? static_cast<uint64_t>(A.fwd[j]) : j, r);
            if (fused) p1_add(sv, A.p1.m, r.x, !r.stopped);
            const unsigned st = static_cast<unsigned>(max(r.steps, 0));
            my_steps += st;
            // lane-efficiency bookkeeping: the warp ran max(steps) slots per lane
            const unsigned gmax = __reduce_max_sync(mask, st);
            if (lane == static_cast<unsigned>(__ffs(mask) - 1)) {
                my_slots += static_cast<unsigned long long>(gmax) * __popc(mask);
            }
        }
    }
    if (fused) {
        __syncthreads();
        p1_flush(sv, A.p1);
    }
    for (int o = 16; o > 0; o >>= 1) {
        my_steps += __shfl_down_sync(0xffffffffu, my_steps, o);
        my_slots += __shfl_down_sync(0xffffffffu, my_slots, o);
    }
    if (lane == 0) {
        if (A.total_steps && my_steps) atomicAdd(A.total_steps, my_steps);
        if (A.counters) {
            atomicAdd(&A.counters[0], my_steps);
            atomicAdd(&A.counters[1], my_slots);
        }
    }
}

// ---------------------------------------------------------------- binning

constexpr int kMaxBuckets = 4096;

// FP32 coarse-step RK4 of the speed lane through the actuator transient
// (brake_accel sampled from the exact actuator table), then the stop time of
// dv/dt = c - D v^2 with the final constant c = max(a_inf, F) - G in closed
// form -> predicted stop step -> bucket (descending).  Only the schedule
// depends on this; results never do.
__global__ void __launch_bounds__(256) predict_kernel(const PredictArgs P) {
    extern __shared__ float s_a[];
    __shared__ unsigned int s_hist[kMaxBuckets];
    for (int i = threadIdx.x; i < P.coarse_len; i += blockDim.x) s_a[i] = P.coarse_a[i];
    for (int i = threadIdx.x; i < P.buckets; i += blockDim.x) s_hist[i] = 0u;
    __syncthreads();
    const float h = P.h, hh = 0.5f * P.h, h6 = P.h / 6.0f;
    const int ks = P.coarse_steps;  // <= (coarse_len - 1) / 2
    const float t_s = static_cast<float>(ks) * h;
    // blocks [w * bpw, (w + 1) * bpw) cover binning window w
    const unsigned bpw = gridDim.x / static_cast<unsigned>(bin_windows(P.n));
    const uint64_t w = blockIdx.x / bpw;
    const uint64_t lo = w << kBinWindowLog2;
    const uint64_t hi = min(P.n, lo + (uint64_t{1} << kBinWindowLog2));
    const uint64_t stride = static_cast<uint64_t>(bpw) * blockDim.x;
    for (uint64_t i = lo + static_cast<uint64_t>(blockIdx.x % bpw) * blockDim.x + threadIdx.x; i < hi;
         i += stride) {
        float v = static_cast<float>(P.v0[i]);
        const float F = static_cast<float>(P.brake_floor[i]);
        const float D = static_cast<float>(P.drag[i]);
        const float G = static_cast<float>(P.grade[i]);
        float tstar = -1.0f;
        // scheduling only: FP32 with explicit FMAs (the file is -fmad=false)
        const float nD = -D;
        float b1 = fmaxf(s_a[0], F) - G;
        for (int k = 0; k < ks; ++k) {
            const float b2 = fmaxf(s_a[2 * k + 1], F) - G;
            const float b4 = fmaxf(s_a[2 * k + 2], F) - G;
            const float k1 = __fmaf_rn(nD, v * v, b1);
            const float v2 = __fmaf_rn(hh, k1, v);
            const float k2 = __fmaf_rn(nD, v2 * v2, b2);
            const float v3 = __fmaf_rn(hh, k2, v);
            const float k3 = __fmaf_rn(nD, v3 * v3, b2);
            const float v4 = __fmaf_rn(h, k3, v);
            const float k4 = __fmaf_rn(nD, v4 * v4, b4);
            const float vn = __fmaf_rn(h6, __fmaf_rn(2.0f, k2 + k3, k1 + k4), v);
            b1 = b4;
            if (vn <= 0.0f) {
                tstar = (static_cast<float>(k) + v / (v - vn)) * h;
                break;
            }
            v = vn;
        }
        if (tstar < 0.0f) {
            // constant brake: dv/dt = -(q + D v^2), q = G - max(a_inf, F)
            const float q = G - fmaxf(P.a_inf, F);
            if (q > 0.0f) {
                const float r = sqrtf(q * D);
                tstar = t_s + (r > 0.0f ? atanf(v * D / r) / r : v / q);
            }
        }
        int pred = P.max_steps;
        if (tstar >= 0.0f) pred = static_cast<int>(fminf(ceilf(tstar * P.inv_dt), 2e9f));
        pred = max(1, min(pred, P.max_steps));
        // key = (clamp class, descending step bucket), class-major: warps see
        // one class, so the never-clamping majority runs the select-free loop
        // body.  Class-major because the sort is per binning window: with
        // step-major keys every window had hundreds of class boundaries, and
        // a warp straddling one ran the select + per-step-test band up to the
        // table head (+2.7% instructions, 96.2% FP64 pipe, ncu)
        const int sb = (P.max_steps - pred) / P.bucket_width;
        const int cls = P.brake_floor[i] < P.table_min ? 0 : 1;
        const int bucket = min(cls * (P.buckets >> 1) + sb, P.buckets - 1);
        P.keys[i] = static_cast<uint16_t>(bucket);
        atomicAdd(&s_hist[bucket], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < P.buckets; b += blockDim.x) {
        const unsigned int c = s_hist[b];
        if (c) atomicAdd(&P.hist[w * P.buckets + b], c);
    }
}

__global__ void __launch_bounds__(1024) bin_scan_kernel(unsigned int* hist_all, int buckets) {
    // exclusive scan, in place: counts -> start cursor of each bucket; block
    // w scans window w, whose sorted slots start at w * 2^kBinWindowLog2 (full windows)
    unsigned int* hist = hist_all + static_cast<size_t>(blockIdx.x) * buckets;
    const unsigned int base = static_cast<unsigned int>(blockIdx.x) << kBinWindowLog2;
    using Scan = cub::BlockScan<unsigned int, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    constexpr int kPer = kMaxBuckets / 1024;
    unsigned int items[kPer];
    for (int k = 0; k < kPer; ++k) {
        const int b = threadIdx.x * kPer + k;
        items[k] = b < buckets ? hist[b] : 0u;
    }
    Scan(tmp).ExclusiveSum(items, items);
    for (int k = 0; k < kPer; ++k) {
        const int b = threadIdx.x * kPer + k;
        if (b < buckets) hist[b] = base + items[k];
    }
}

#ifndef BMC_SCATTER_PRELOAD
#define BMC_SCATTER_PRELOAD 1
#endif
template <int kItems>
__global__ void __launch_bounds__(256, BMC_SCATTER_PRELOAD ? 2 : 1)
    bin_scatter_kernel(const uint16_t* keys, uint64_t n, unsigned int* cursor, const double* v0,
                       const double* floor_, const double* drag, const double* grade,
                       PackedTerms* packed, uint32_t* perm, int forward, int buckets) {
    // Tile-aggregated counting-sort scatter: ranks inside a 2048-sample tile
    // come from shared-memory atomics; each (tile, bucket) reserves its slots
    // with ONE global atomic, so hot buckets are not serialised per warp.
    // The tile's keys AND terms are loaded into registers first, so their
    // DRAM latency overlaps the shared-memory ranking and the bucket
    // reservations (loaded after them, each item's four term loads waited
    // behind the previous item's scattered stores: 1.5 TB/s, ncu).
    constexpr int kTile = 256 * kItems;
    __shared__ unsigned int s_cnt[kMaxBuckets];
    __shared__ unsigned int s_base[kMaxBuckets];
    for (uint64_t tile = static_cast<uint64_t>(blockIdx.x) * kTile; tile < n;
         tile += static_cast<uint64_t>(gridDim.x) * kTile) {
        unsigned key[kItems], rank[kItems];
        double tv[BMC_SCATTER_PRELOAD ? kItems : 1], tf[BMC_SCATTER_PRELOAD ? kItems : 1];
        double td[BMC_SCATTER_PRELOAD ? kItems : 1], tg[BMC_SCATTER_PRELOAD ? kItems : 1];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            const uint64_t i = tile + static_cast<uint64_t>(k) * 256 + threadIdx.x;
            if (i < n) {
                key[k] = keys[i];
                if (BMC_SCATTER_PRELOAD) {
                    tv[k] = __ldcs(v0 + i);
                    tf[k] = __ldcs(floor_ + i);
                    td[k] = __ldcs(drag + i);
                    tg[k] = __ldcs(grade + i);
                }
            }
        }
        for (int b = threadIdx.x; b < kMaxBuckets; b += 256) s_cnt[b] = 0u;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            const uint64_t i = tile + static_cast<uint64_t>(k) * 256 + threadIdx.x;
            if (i < n) rank[k] = atomicAdd(&s_cnt[key[k]], 1u);
        }
        __syncthreads();
        // a tile lies inside one binning window (2^kBinWindowLog2 is a multiple of kTile)
        unsigned int* wcur = cursor + (tile >> kBinWindowLog2) * static_cast<uint64_t>(buckets);
        for (int b = threadIdx.x; b < kMaxBuckets; b += 256) {
            const unsigned c = s_cnt[b];
            if (c) s_base[b] = atomicAdd(&wcur[b], c);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            const uint64_t i = tile + static_cast<uint64_t>(k) * 256 + threadIdx.x;
            if (i < n) {
                const uint32_t pos = s_base[key[k]] + rank[k];
                if (forward) {
                    perm[pos] = static_cast<uint32_t>(i);
                } else {
                    perm[i] = pos;
                }
                // one aligned 32-byte record = one full sector: no read-for-fill
                double2* dst = reinterpret_cast<double2*>(packed + pos);
                if (BMC_SCATTER_PRELOAD) {
                    dst[0] = make_double2(tv[k], tf[k]);
                    dst[1] = make_double2(td[k], tg[k]);
                } else {
                    dst[0] = make_double2(v0[i], floor_[i]);
                    dst[1] = make_double2(drag[i], grade[i]);
                }
            }
        }
        __syncthreads();
    }
}

// Index-order gather of the packed sorted outputs.  The 16-B records sit at
// random slots, so each costs a full 32-B sector (73 B/sample DRAM for 33
// algorithmic).  Measured and not adopted (ncu, profiles/round2_hbm_stage_ab.txt
// section F): 4 or 8 gathers in flight per thread with one 16-B streaming
// load each -- 2.68 / 2.47 ms against 2.66 ms, but 123 B/sample of DRAM reads.
__global__ void __launch_bounds__(256) unpermute_kernel(const PackedOut* packed_out,
                                                        const uint32_t* inv_perm, uint64_t n,
                                                        double* d, int32_t* steps, uint8_t* hz) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += stride) {
        const PackedOut r = packed_out[inv_perm[j]];
        if (d) d[j] = r.x;
        if (steps) steps[j] = r.steps;
        if (hz) hz[j] = static_cast<uint8_t>(r.hit_horizon);
    }
}

// FP64 issue-rate probe: 8 independent chains per thread of unfused
// x = x*a + b (one DMUL + one DADD each), so the pipe, not latency, binds.
__global__ void __launch_bounds__(512) fp64_probe_kernel(double* out, int iters, double a,
                                                         double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = 1.0 + 1e-9 * (threadIdx.x + 37 * k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], a), b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s = __dadd_rn(s, x[k]);
    if (s == 12345.678) out[0] = s;  // never true; keeps the chains alive
}

template <int MODE, int BT, int ILP, int UNR = 1>
cudaError_t launch_rollout_t(const RolloutArgs& a, cudaStream_t s) {
    size_t smem = 0;
    if (MODE == kTableShared) smem = static_cast<size_t>(a.table_len) * sizeof(StageA);
    if (a.p1.sum) smem += p1_smem_bytes(a.p1.m);
    if (smem > 0) {
        const cudaError_t e = cudaFuncSetAttribute(rollout_kernel<MODE, BT, ILP, UNR>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    int dev = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, rollout_kernel<MODE, BT, ILP, UNR>, BT, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    // Persistent grid.  Small batches (the real-time case) spread their
    // sample groups over every SM with narrower CTAs instead of packing
    // them into a few full ones: fewer warps per SM = shorter per-step
    // latency of each dependent RK4 chain.
    const uint64_t groups = (a.n + 32 * ILP - 1) / (32 * ILP);
    const uint64_t sms = static_cast<uint64_t>(sm_count_cached(dev));
    const uint64_t resident = static_cast<uint64_t>(per_sm) * sms;
    uint64_t warps_per_block = BT / 32;
    if (groups < resident * warps_per_block) {
        warps_per_block = std::max<uint64_t>(1, (groups + resident - 1) / resident);
    }
    const uint64_t need = (groups + warps_per_block - 1) / warps_per_block;
    const int grid = static_cast<int>(std::max<uint64_t>(1, std::min(need, resident)));
    rollout_kernel<MODE, BT, ILP, UNR><<<grid, static_cast<int>(warps_per_block * 32), smem, s>>>(a);
    return cudaGetLastError();
}

// Instantiated variants (results never depend on the choice): table modes
// with one chain per thread at 256/512/768/1024 threads or two chains at
// 512/640/768, each with the per-step or the blocked termination test; the
// no-table fallback only with one chain and the per-step test.
template <int MODE, int ILP, int UNR>
cudaError_t launch_rollout_b(const RolloutArgs& a, int block_threads, cudaStream_t s) {
    if constexpr (ILP == 2) {
        switch (block_threads) {
            case 512: return launch_rollout_t<MODE, 512, 2, UNR>(a, s);
            case 640: return launch_rollout_t<MODE, 640, 2, UNR>(a, s);
            case 768: return launch_rollout_t<MODE, 768, 2, UNR>(a, s);
            default: return cudaErrorInvalidValue;
        }
    } else {
        switch (block_threads) {
            case 256: return launch_rollout_t<MODE, 256, 1, UNR>(a, s);
            case 512: return launch_rollout_t<MODE, 512, 1, UNR>(a, s);
            case 768: return launch_rollout_t<MODE, 768, 1, UNR>(a, s);
            case 1024: return launch_rollout_t<MODE, 1024, 1, UNR>(a, s);
            default: return cudaErrorInvalidValue;
        }
    }
}

template <int MODE>
cudaError_t launch_rollout_m(const RolloutArgs& a, int block_threads, int ilp, int unroll,
                             cudaStream_t s) {
    if constexpr (MODE == kTableNone) {
        return launch_rollout_b<MODE, 1, 1>(a, block_threads, s);
    } else {
        const bool blk = unroll == kTestBlock;
        if (ilp == 2) {
            return blk ? launch_rollout_b<MODE, 2, kTestBlock>(a, block_threads, s)
                       : launch_rollout_b<MODE, 2, 1>(a, block_threads, s);
        }
        return blk ? launch_rollout_b<MODE, 1, kTestBlock>(a, block_threads, s)
                   : launch_rollout_b<MODE, 1, 1>(a, block_threads, s);
    }
}

int sm_count_cached(int device) {
    static int cache[64] = {0};
    if (device < 0 || device >= 64) return sm_count(device);
    if (cache[device] == 0) cache[device] = sm_count(device);
    return cache[device];
}

}  // namespace

int sm_count(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    return v;
}

cudaError_t launch_rollout(const RolloutArgs& a, int table_mode, int block_threads, int ilp,
                           int unroll, cudaStream_t s) {
    switch (table_mode) {
        case kTableShared: return launch_rollout_m<kTableShared>(a, block_threads, ilp, unroll, s);
        case kTableGlobal: return launch_rollout_m<kTableGlobal>(a, block_threads, ilp, unroll, s);
        case kTableNone: return launch_rollout_m<kTableNone>(a, block_threads, 1, 1, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_fp64_probe(double* out, int iters, uint64_t* ops, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int blocks = sm_count(dev) * 4;
    fp64_probe_kernel<<<blocks, 512, 0, s>>>(out, iters, 0.99999999, 1e-8);
    *ops = static_cast<uint64_t>(blocks) * 512u * static_cast<uint64_t>(iters) * 16u;
    return cudaGetLastError();
}

cudaError_t launch_predict(const PredictArgs& a, cudaStream_t s) {
    if (a.buckets > kMaxBuckets || a.buckets < 1) return cudaErrorInvalidValue;
    int dev = 0;
    cudaGetDevice(&dev);
    // bpw blocks per binning window, ~8 CTAs per SM in all
    const uint64_t nwin = bin_windows(a.n);
    const uint64_t target = static_cast<uint64_t>(sm_count_cached(dev)) * 8;
    const uint64_t per_win = std::min<uint64_t>(uint64_t{1} << kBinWindowLog2, a.n);
    const uint64_t bpw = std::max<uint64_t>(1, std::min<uint64_t>((per_win + 255) / 256,
                                                                  (target + nwin - 1) / nwin));
    const int grid = static_cast<int>(nwin * bpw);
    predict_kernel<<<grid, 256, static_cast<size_t>(a.coarse_len) * sizeof(float), s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_bin_scan(unsigned int* hist, int buckets, uint64_t n, cudaStream_t s) {
    if (buckets > kMaxBuckets) return cudaErrorInvalidValue;
    bin_scan_kernel<<<static_cast<int>(std::max<uint64_t>(1, bin_windows(n))), 1024, 0, s>>>(hist, buckets);
    return cudaGetLastError();
}

cudaError_t launch_bin_scatter(const uint16_t* keys, uint64_t n, unsigned int* cursor,
                               const double* v0, const double* brake_floor, const double* drag,
                               const double* grade, PackedTerms* packed, uint32_t* perm,
                               int forward, int buckets, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    // 8 items per thread (2048-sample tiles); 16 and 32 were measured slower
    // (profiles/round2_summary.md, A/B table)
    constexpr uint64_t tile = 256u * 8u;
    const uint64_t blocks_needed = (n + tile - 1) / tile;
    const int grid = static_cast<int>(std::min<uint64_t>(blocks_needed,
                                                         static_cast<uint64_t>(sm_count_cached(dev)) * 8));
    bin_scatter_kernel<8><<<grid, 256, 0, s>>>(keys, n, cursor, v0, brake_floor, drag, grade, packed,
                                               perm, forward, buckets);
    return cudaGetLastError();
}

cudaError_t launch_unpermute(const PackedOut* packed_out, const uint32_t* inv_perm, uint64_t n,
                             double* stop_distance, int32_t* steps, uint8_t* hit_horizon,
                             cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t blocks_needed = (n + 255) / 256;
    const int grid = static_cast<int>(std::min<uint64_t>(blocks_needed,
                                                         static_cast<uint64_t>(sm_count_cached(dev)) * 8));
    unpermute_kernel<<<grid, 256, 0, s>>>(packed_out, inv_perm, n, stop_distance, steps,
                                          hit_horizon);
    return cudaGetLastError();
}

}  // namespace bmc
