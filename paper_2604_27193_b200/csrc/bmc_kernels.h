// bmc_kernels.h -- launch interface of the sm_100a kernels (bmc_kernels.cu,
// bmc_stats.cu).  Host-only callers (bmc_capi.cpp) see plain structs.
#pragma once

#include "bmc_internal.h"
#include "bmc_stats_dev.cuh"

#include <cuda_runtime.h>

namespace bmc {

enum TableMode : int { kTableAuto = 0, kTableShared = 1, kTableGlobal = 2, kTableNone = 3 };
enum Schedule : int { kScheduleDefault = 0, kScheduleIndex = 1, kScheduleBinned = 2 };

// Largest actuator table kept in shared memory (entries of 32 B).
constexpr int kSmemTableMax = 6784;  // 217 KB of the 227 KB opt-in limit

// Packed per-sample records used by the binned schedule: the binning
// scatter writes each sample's inputs as one aligned 32-byte record in
// sorted order (one full DRAM sector), the rollout reads and writes packed
// records coalesced, and unpermute restores index order.
struct __align__(32) PackedTerms {
    double v0, brake_floor, drag, grade;
};
struct __align__(16) PackedOut {
    double x;
    int32_t steps;
    uint32_t hit_horizon;
};

struct RolloutArgs {
    const double* v0;
    const double* brake_floor;
    const double* drag;
    const double* grade;
    const uint32_t* perm;  // nullable: index order
    uint64_t n;
    double dt, half, sixth, brake_cmd, inv_tau;
    int32_t max_steps;
    const StageA* table;   // device, table_len entries (unused for kTableNone)
    int32_t table_len;
    double* stop_distance; // nullable
    int32_t* steps;        // nullable
    uint8_t* hit_horizon;  // nullable
    unsigned long long* total_steps;  // nullable
    unsigned int* work_counter;       // device, zeroed before launch
    unsigned long long* counters;     // nullable: [0] executed steps, [1] lane slots
    const PackedTerms* packed_in;     // nullable: sorted packed inputs (binned schedule)
    PackedOut* packed_out;            // nullable: sorted packed outputs (binned schedule)
    const uint32_t* fwd;              // nullable: sorted slot -> sample index; outputs are then
                                      // written SoA at the sample's index (no unpermute pass)
    P1Args p1;                        // fused statistics pass 1 (p1.sum nullptr: off)
    int32_t monotone_blocks;          // 1: blocks past monotone_from test only their end
};

struct PredictArgs {
    const double* v0;
    const double* brake_floor;
    const double* drag;
    const double* grade;
    uint64_t n;
    const float* coarse_a;  // brake_accel at t = k * h/2, k = 0..coarse_len-1
    int32_t coarse_len;
    float h;                // coarse step (s)
    int32_t coarse_steps;   // coarse RK4 steps through the actuator transient
    float a_inf;            // brake_accel after it (constant to float precision)
    float inv_dt;
    int32_t max_steps;
    int32_t bucket_width;   // steps per bucket
    int32_t buckets;        // total keys = 2 * step buckets (clamp class bit)
    double table_min;       // min actuator stage value: F < table_min never clamps
    uint16_t* keys;         // out: bucket per sample (descending predicted steps)
    unsigned int* hist;     // out: per-(window, bucket) counts (zeroed before launch)
};

// Binning windows: samples are sorted within consecutive index windows of
// 2^kBinWindowLog2 (window-major sorted order).  Smaller windows keep the
// counting-sort scatter's writes local (2^20: scatter 4.45 -> 2.0 ms at 1e8)
// but cost the rollout more than that (921.6 vs 916.4 ms with 2^20 / one
// window; 2^22: 919.2 ms), so the windows are 2^27 samples: one window up
// to 1.3e8 (profiles/round2_hbm_stage_ab.txt, section E).
constexpr int kBinWindowLog2 = 27;
#if defined(__CUDACC__)
__host__ __device__
#endif
inline uint64_t bin_windows(uint64_t n) {
    return (n + (uint64_t{1} << kBinWindowLog2) - 1) >> kBinWindowLog2;
}

// On-device sampler (bmc_sampler.cu): samples [first, first+n) of
// draw_batch(model, .) and their RolloutTerms, bit-identical to the host
// producers through the glibc port (bmc_libm.h).
enum DrawFlags : unsigned { kDrawDomain = 1u, kDrawUnported = 2u };
// Per-launch draw parameters read from device memory (CUDA-graph replays
// update them with a captured H2D copy instead of re-capturing).
struct DrawDyn {
    uint64_t seed;
    bmc_normal spec[5];
    uint64_t first;
};
struct DrawArgs {
    uint64_t seed;
    bmc_normal spec[5];    // v0, mu, theta, m, c_d (UncertaintyModel order)
    uint64_t first, n;
    double cg_height, wheelbase, gravity, air_density, frontal_area;
    double* v0;            // nullable (then no terms are formed)
    double* brake_floor;
    double* drag;
    double* grade;
    double* samples;       // nullable: AoS bmc_sample records (5 doubles)
    unsigned long long* clamps;  // device, accumulated
    unsigned int* flags;         // device, DrawFlags OR-ed
    const DrawDyn* dyn;          // nullable: overrides seed/spec/first
};
cudaError_t launch_draw_terms(const DrawArgs& a, int sms, cudaStream_t s);

// Sensor-noise TTC sweep (C4 extension; the reference has no noise model):
// sample i's AEB trigger fires at a measured TTC T_j + eps_i with
// eps_i = sigma * standard_normal_at(noise_seed, first + i) (the reference's
// Box-Muller on its own counter stream, through the glibc port), so its
// headway at brake onset is H_ij = (T_j + eps_i) * v_closing and it
// collides iff hit_horizon or stop_distance > H_ij.  With T sorted
// ascending, H_ij is non-decreasing in j and bucket p_i = #{j : H_ij < d_i}
// (m for a horizon hit) gives count_j = #{i : p_i > j}.  sigma = 0 reduces
// exactly to collision_probability(results, T_j * v) (analysis.cpp:145-159).
struct NoiseExceedArgs {
    const double* d;
    const uint8_t* hz;      // nullable
    uint64_t n, first, seed;
    double sigma, closing;
    const double* ttc;      // device, m sorted ascending
    int m;
    unsigned long long* buckets;  // device, m + 1, zeroed
    unsigned int* flags;          // device, DrawFlags OR-ed
};
constexpr int kNoiseMaxThresholds = 1024;
cudaError_t launch_noise_exceed(const NoiseExceedArgs& a, int sms, cudaStream_t s);

struct LaunchShape {
    int block_threads;
    int grid;
    size_t smem;
};

int sm_count(int device);

// Persistent launch: grid = min(resident CTAs, 32-sample groups / warps per CTA).
cudaError_t launch_rollout(const RolloutArgs& a, int table_mode, int block_threads, int ilp,
                           int unroll, cudaStream_t s);
cudaError_t launch_predict(const PredictArgs& a, cudaStream_t s);
cudaError_t launch_fp64_probe(double* out, int iters, uint64_t* ops, cudaStream_t s);
cudaError_t launch_bin_scan(unsigned int* hist_to_cursor, int buckets, uint64_t n, cudaStream_t s);
// counting-sort scatter: inv_perm[i] = sorted slot of sample i, and the
// sample's inputs are written packed into that slot
// forward != 0: perm[slot] = i (sorted slot -> sample, for direct SoA
// outputs); else perm[i] = slot (inverse, for unpermute)
cudaError_t launch_bin_scatter(const uint16_t* keys, uint64_t n, unsigned int* cursor,
                               const double* v0, const double* brake_floor, const double* drag,
                               const double* grade, PackedTerms* packed, uint32_t* perm,
                               int forward, int buckets, cudaStream_t s);
// outputs back to index order: out[j] = packed_out[inv_perm[j]]
cudaError_t launch_unpermute(const PackedOut* packed_out, const uint32_t* inv_perm, uint64_t n,
                             double* stop_distance, int32_t* steps, uint8_t* hit_horizon,
                             cudaStream_t s);

// statistics (bmc_stats.cu)
struct StatsScratch {
    void* buf = nullptr;
    size_t bytes = 0;
};

}  // namespace bmc
