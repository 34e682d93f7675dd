/*
 * brakemc_cuda.h -- C-ABI of the B200 (sm_100a) Monte Carlo rollout engine.
 *
 * This is the drop-in boundary for the reference's executor family
 * (/root/reference/proj/include/brakemc/backends.hpp:18-45).  The reference
 * has no FFI; its extension point is "an actual GPU backend ... behind the
 * same executor interface".  The C++ executor
 * brakemc::run_cuda (include/brakemc/cuda_executor.hpp) is a thin adapter
 * over these entry points; Python tests/bench bind them through ctypes.
 *
 * Conventions
 *   - Plain C types only; no exceptions cross this boundary.
 *   - Every int-returning call returns BMC_OK (0) or a negative BMC_E_* code;
 *     the message is available from bmc_last_error() (thread-local) and,
 *     for context calls, bmc_cuda_last_error(ctx).
 *   - BMC_E_CONFIG mirrors brakemc::ConfigError (errors.hpp:10-20): the
 *     message starts with the offending field path, e.g.
 *     "batch: must be non-empty" (backends.cpp:41-43).
 *   - Struct layouts equal the reference value types byte for byte
 *     (static_assert'ed in cuda_executor.cpp), so a std::vector<RolloutResult>
 *     or std::vector<ScenarioSample> can be passed by .data().
 *   - There is NO CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with BMC_E_CUDA.
 */
#ifndef BRAKEMC_CUDA_H
#define BRAKEMC_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BMC_ABI_VERSION 1

enum {
    BMC_OK = 0,
    BMC_E_CONFIG = -1,  /* invalid argument (ConfigError analogue)        */
    BMC_E_DOMAIN = -2,  /* friction_limit denominator <= 0 (domain_error) */
    BMC_E_CUDA = -3,    /* CUDA runtime / launch failure                  */
    BMC_E_NOMEM = -4,   /* host or device allocation failed               */
    BMC_E_RANGE = -5,   /* capacity exceeded (e.g. histogram buffer)      */
    BMC_E_IO = -6       /* file I/O / parse failure (IoError analogue)    */
};

/* == brakemc::ScenarioSample (dynamics.hpp:36-44), 40 bytes */
typedef struct {
    double initial_speed, friction, grade, mass, drag_coeff;
} bmc_sample;

/* == brakemc::RolloutResult (integrator.hpp:14-19), 32 bytes */
typedef struct {
    double stop_distance;
    double stop_time;
    int64_t steps;
    uint8_t hit_horizon;
    uint8_t pad_[7];
} bmc_result;

/* SimConfig (dynamics.hpp:54-60) + VehicleGeometry (:27-33) +
 * PhysicalConstants (:17-24), flattened in that order. */
typedef struct {
    double dt, t_max, brake_cmd;
    double cg_height, wheelbase, actuator_tau;
    double gravity, air_density, frontal_area;
} bmc_world;

/* == brakemc::NormalSpec (sampling.hpp:17-20) */
typedef struct {
    double mean, sd;
} bmc_normal;

/* == brakemc::UncertaintyModel (sampling.hpp:24-33), 88 bytes */
typedef struct {
    uint64_t seed;
    bmc_normal initial_speed, friction, grade, mass, drag_coeff;
} bmc_model;

/* Per-sample rollout inputs staged SoA: the sample-varying part of
 * brakemc::RolloutTerms (dynamics.hpp:96-106) plus v0.  brake_cmd and
 * inv_tau are batch constants and travel in bmc_world. 32 B/sample. */
typedef struct {
    const double* initial_speed;
    const double* brake_floor;
    const double* drag_factor;
    const double* grade_accel;
} bmc_terms;

/* Compact per-sample outputs (13 B/sample).  Any pointer may be NULL
 * (stats-only mode).  stop_time is not stored: it is (double)steps * dt. */
typedef struct {
    double* stop_distance;
    int32_t* steps;
    uint8_t* hit_horizon;
} bmc_outputs;

/* Scheduling knobs; zero-initialised means "defaults". Results never
 * depend on these (only timing does), exactly like run_parallel's chunk
 * size (backends.hpp:36-41). */
typedef struct {
    int32_t schedule;       /* 0 = default (binned), 1 = index order, 2 = binned by predicted stop step */
    int32_t block_threads;  /* 0 = default */
    int32_t table_mode;     /* 0 = auto, 1 = shared-mem a-table, 2 = global a-table, 3 = no table */
    int32_t host_threads;   /* 0 = all hardware threads (host staging / unpack) */
    uint64_t chunk_samples; /* 0 = default pipeline chunk for bmc_cuda_run */
    int32_t ilp;            /* samples per thread: 0 = default, 1, or 2 (table modes) */
    int32_t sampler;        /* model-driven runs: 0 = auto (device when bmc_device_sampler_available),
                               1 = host pool, 2 = device (BMC_E_CONFIG when unavailable) */
    int32_t test_block;     /* steps per termination-test block (ilp 1, table modes):
                               0 = default, 1 = every step, 8 = blocked test + exact replay */
} bmc_run_opts;

/* Timing breakdown of one bmc_cuda_run call (seconds). */
typedef struct {
    double wall_s;        /* whole call: staging + H2D + kernels + D2H + unpack */
    double kernel_ms;     /* sum of per-chunk rollout event spans (the two pipeline slots run on
                             their own streams, so spans of neighbouring chunks may overlap) */
    double predict_ms;    /* sum of predictor + binning kernel event times */
    uint64_t total_steps; /* sum of executed RK4 steps (roofline numerator) */
    uint64_t h2d_bytes, d2h_bytes;
    uint32_t launches;    /* kernels this call launched */
    uint32_t chunks;
} bmc_run_info;

typedef struct bmc_ctx bmc_ctx;

/* ------------------------------------------------------------- context */
int bmc_abi_version(void);
const char* bmc_last_error(void);
int bmc_device_count(int* out);
int bmc_cuda_init(int device, bmc_ctx** out);
void bmc_cuda_destroy(bmc_ctx* ctx);
const char* bmc_cuda_last_error(const bmc_ctx* ctx);
int bmc_cuda_sync(bmc_ctx* ctx);
/* the context's compute stream (cudaStream_t) */
void* bmc_cuda_stream(bmc_ctx* ctx);

/* ------------------------------------------------ host-side producers */
/* draw_batch (sampling.cpp:67-100) restricted to sample indices
 * [first, first + n); bit-identical to the same slice of draw_batch(model, N)
 * because the stream is counter-based (sampling.hpp:3-6). threads <= 0: all. */
int bmc_draw_range(const bmc_model* model, uint64_t first, size_t n, bmc_sample* out,
                   uint64_t* clamp_count, int threads);
/* RolloutTerms::from (dynamics.cpp:57-68) for each sample, SoA out. */
int bmc_stage_terms(const bmc_sample* samples, size_t n, const bmc_world* world,
                    double* initial_speed, double* brake_floor, double* drag_factor,
                    double* grade_accel, int threads);

/* On-device sampler gate.  The device sampler replays glibc 2.39's FMA
 * libm variants (__log_fma, __cos_fma, __sin_fma) op for op; it is
 * bit-identical to bmc_draw_range only on a host whose own libm is that
 * variant.  bmc_libm_selftest compares the port against the live host libm
 * over n sampler draws (+ every branch boundary); mismatches[7] =
 * {log, log near 1, cos(2 pi u), sin |x|<=1.5, sin/cos reduced, normal
 * deviate, boundaries/range}.  BMC_OK iff all are zero.
 * bmc_device_sampler_available caches a quick check for the process. */
int bmc_libm_selftest(uint64_t n, uint64_t seed, int threads, uint64_t* mismatches);
int bmc_device_sampler_available(int* available);

/* On-device draw_batch (sampling.cpp:67-100) of samples [first, first+n),
 * fused with RolloutTerms::from (dynamics.cpp:57-68): bit-identical to
 * bmc_draw_range + bmc_stage_terms when bmc_device_sampler_available.
 * terms: device, 4*n doubles laid out [v0 | brake_floor | drag_factor |
 * grade_accel] (nullable); samples: device AoS (nullable).  Synchronous;
 * BMC_E_DOMAIN for a non-positive friction_limit denominator, BMC_E_RANGE if
 * an argument left the ported glibc range. */
int bmc_cuda_draw_device(bmc_ctx* ctx, const bmc_model* model, uint64_t first, size_t n,
                         const bmc_world* world, double* terms, bmc_sample* samples,
                         uint64_t* clamp_count);

/* results.csv artifact (io.cpp:17-31 / 94-123): byte-identical writer
 * ("%.17g", so doubles round-trip exactly) and reader; the reader rebuilds
 * steps = llround(t_stop / dt) as cmd_verify does (cli.cpp:96-100). */
int bmc_write_results_csv(const char* path, const bmc_result* results, size_t n, int threads);
int bmc_read_results_csv(const char* path, double dt, bmc_result* out, size_t cap,
                         size_t* n_out);

/* ------------------------------------------------------------ executor */
/* Drop-in core of brakemc::run_cuda: host AoS samples in, host AoS results
 * out (index-aligned, bit-identical to run_sequential).  Synchronous.
 * Host staging, H2D, kernels, D2H and unpack are pipelined in chunks. */
int bmc_cuda_run(bmc_ctx* ctx, const bmc_sample* samples, size_t n, const bmc_world* world,
                 const bmc_run_opts* opts, bmc_result* out, bmc_run_info* info);

/* Model-driven streaming executor (no AoS batch is ever materialised):
 * samples [first, first+n) of draw_batch(model, .) are drawn by the host pool
 * straight into pinned SoA terms, streamed H2D per chunk on a side stream and
 * overlapped with the kernels of the previous chunk.  Exactly one of
 * host_out (AoS results, RolloutResult layout) or dev_out (device-resident
 * compact outputs with n entries each -- stats-only mode for 1e9-sample
 * runs) must be non-NULL.  clamp_count = draw_batch's clamp_count. */
int bmc_cuda_run_model(bmc_ctx* ctx, const bmc_model* model, uint64_t first, size_t n,
                       const bmc_world* world, const bmc_run_opts* opts, bmc_result* host_out,
                       const bmc_outputs* dev_out, uint64_t* clamp_count, bmc_run_info* info);

/* Real-time mode (C2): a fixed-size decision batch captured once as a CUDA
 * graph {H2D terms, predict/bin, rollout, D2H outputs}; each decision is
 * host staging + one cudaGraphLaunch + unpack.  The graph owns its buffers. */
typedef struct bmc_graph bmc_graph;
int bmc_cuda_graph_create(bmc_ctx* ctx, size_t n, const bmc_world* world,
                          const bmc_run_opts* opts, bmc_graph** out);
int bmc_cuda_graph_run(bmc_graph* g, const bmc_sample* samples, bmc_result* out,
                       bmc_run_info* info);
/* Same, drawing the n samples [first, first+n) of `model` on the host pool
 * (the reference's feasibility convention includes sampling,
 * analysis.cpp:331-338). */
int bmc_cuda_graph_run_model(bmc_graph* g, const bmc_model* model, uint64_t first,
                             bmc_result* out, uint64_t* clamp_count, bmc_run_info* info);
void bmc_cuda_graph_destroy(bmc_graph* g);

/* Device-resident rollout: terms and outputs are device pointers; enqueued
 * on `stream` (NULL = the context's stream); returns without synchronising.
 * total_steps_dev (device uint64, nullable) accumulates executed steps. */
int bmc_cuda_rollout_device(bmc_ctx* ctx, const bmc_terms* terms, size_t n,
                            const bmc_world* world, const bmc_run_opts* opts,
                            const bmc_outputs* out, unsigned long long* total_steps_dev,
                            void* stream);

/* Last rollout kernel's device time in ms, via CUDA events recorded around
 * it on its own stream (waits for the closing event). */
int bmc_cuda_last_kernel_ms(bmc_ctx* ctx, float* rollout_ms, float* predict_ms);
/* Per-stage device time of the last device-resident rollout (ms, CUDA
 * events on its stream): predictor + binning scatter, rollout kernel,
 * unpermute (0 when a stage did not run).  Waits for the closing events. */
int bmc_cuda_last_stage_ms(bmc_ctx* ctx, float* bin_ms, float* rollout_ms, float* unpermute_ms);
/* Executed RK4 steps and lane slots (sum over 32-sample groups of
 * active lanes x longest lane) of the last rollout launch on the context's
 * stream; steps / slots is the SIMT lane efficiency.  Synchronises. */
int bmc_cuda_last_lane_stats(bmc_ctx* ctx, uint64_t* steps, uint64_t* slots);
/* Number of kernels the last device call enqueued. */
int bmc_cuda_last_launches(bmc_ctx* ctx, uint32_t* launches);

/* ---------------------------------------------------------- statistics */
/* Everything analysis.cpp derives from a result vector, computed on device
 * from the compact outputs.  Counts / extrema / histogram / order statistics
 * are exact; mean/sd/skewness use an order-independent compensated sum
 * (the reference sums sequentially, analysis.cpp:34-37). */
typedef struct {
    uint64_t n, horizon_count, bins;
    double mean, sd, min, max, median, skewness, origin, bin_width;
    int32_t right_skewed;
    int32_t pad_;
} bmc_summary;

/* summarize (analysis.cpp:13-76). hist: host buffer of hist_cap counts
 * (nullable); BMC_E_RANGE if hist_cap < bins. */
int bmc_cuda_summarize(bmc_ctx* ctx, const double* stop_distance, const uint8_t* hit_horizon,
                       size_t n, double bin_width, bmc_summary* out, uint64_t* hist,
                       size_t hist_cap);
/* numerators of collision_probability (analysis.cpp:145-159) for m headways
 * (any order): counts[j] = #{hit_horizon || d > headways[j]}. */
int bmc_cuda_exceedance(bmc_ctx* ctx, const double* stop_distance, const uint8_t* hit_horizon,
                        size_t n, const double* headways, size_t m, uint64_t* counts);
/* Sensor-noise TTC sweep (BASELINE C4; an extension, the reference has no
 * noise model).  Result i (global sample index first + i) triggers braking
 * at a measured TTC ttc[j] + eps_i, eps_i = sigma * standard_normal_at(
 * noise_seed, first + i) -- the reference's Box-Muller (sampling.cpp:48-53)
 * on its own counter stream -- so counts[j] = #{hit_horizon ||
 * d > (ttc[j] + eps_i) * closing_speed}.  sigma = 0 equals bmc_cuda_exceedance
 * at headways ttc[j] * closing_speed.  Needs the device sampler gate
 * (bmc_device_sampler_available); m <= 1024 thresholds, any order. */
int bmc_cuda_exceedance_ttc_noise(bmc_ctx* ctx, const double* stop_distance,
                                  const uint8_t* hit_horizon, size_t n, uint64_t first,
                                  uint64_t noise_seed, double sigma, const double* ttc, size_t m,
                                  double closing_speed, uint64_t* counts);
/* Exact order statistics: out[j] = ranks[j]-th smallest (1-based) value of
 * stop_distance, over non-horizon results only when exclude_horizon != 0.
 * Ranks outside [1, count] give NaN. */
int bmc_cuda_order_stats(bmc_ctx* ctx, const double* stop_distance, const uint8_t* hit_horizon,
                         size_t n, int exclude_horizon, const uint64_t* ranks, size_t m,
                         double* out, uint64_t* count_out);

/* Mergeable building blocks for sharded (multi-GPU) statistics: counts add,
 * extrema take min/max, double-double sums merge exactly, so one allreduce
 * per quantity combines shards.  All inputs are device
 * pointers; outputs are host. */
typedef struct {
    uint64_t count, horizon_count;
    double min, max;          /* +inf / -inf for an empty shard */
    double sum_hi, sum_lo;    /* double-double sum of stop_distance */
    int32_t any_nan;
    int32_t pad_;
} bmc_partials;
int bmc_cuda_partials(bmc_ctx* ctx, const double* stop_distance, const uint8_t* hit_horizon,
                      size_t n, bmc_partials* out);
/* m2m3[4] = (sum dev^2 hi, lo, sum dev^3 hi, lo) with dev = d - mean */
int bmc_cuda_moments(bmc_ctx* ctx, const double* stop_distance, size_t n, double mean,
                     double* m2m3);
/* counts[bins]: idx = (size_t)((d - origin) / bin_width) clamped to bins-1
 * (analysis.cpp:61-75 with a caller-chosen origin and bin count) */
int bmc_cuda_histogram(bmc_ctx* ctx, const double* stop_distance, size_t n, double origin,
                       double bin_width, uint64_t bins, uint64_t* counts);
/* One 8-bit radix-select pass: hist[t*256 + digit] counts the candidates whose
 * order key matches prefixes[t] above bit shift+8 (shift = 56, 48, ..., 0). */
int bmc_cuda_select_pass(bmc_ctx* ctx, const double* stop_distance, const uint8_t* hit_horizon,
                         size_t n, int exclude_horizon, int shift, const uint64_t* prefixes,
                         size_t m, uint64_t* hist);

/* --------------------------------------------- fused statistics stage */
/* The statistics of analysis.cpp computed by a fixed device pipeline that
 * fuses its first pass into the rollout epilogue (SURVEY.md 8b's
 * bmc_stats / bmc_stats_req arguments of the rollout call):
 *   pass 1 (rollout epilogue, per-CTA shared-memory partials, one atomic
 *           flush per CTA): count, horizon count, min/max (order keys), the
 *           EXACT sum of stop distances, exceedance counts for the sorted
 *           headway grid (collision_probability :145-159, build_risk_curve
 *           :203-228);
 *   pass 2 (one streaming pass): exact m2/m3 about the mean, the summarize
 *           histogram (:59-75), level-1 order-statistic histograms;
 *   compact + select: exact median (:51-57) and min_safe_headway
 *           (:161-194) from the values of the bucket holding each rank.
 * Counts, extrema, histogram and order statistics are exact; the sums are
 * exact and rounded once, so every field is independent of order, chunking
 * and GPU count (the reference's sequential sum is within (n-1) eps sum|d|).
 * With no merge the stage has no host round trip before its final read, so
 * a CUDA graph captures it (bmc_cuda_graph_create_stats). */
typedef struct {
    const double* headways;     /* collision thresholds, any order, each >= 0 (nullable if 0) */
    size_t n_headways;
    const double* risk_levels;  /* min_safe_headway levels in (0,1), at most 16 (nullable if 0) */
    size_t n_risk;
    int32_t summarize;          /* 1: full summarize (moments, median, histogram) */
    int32_t pad_;
    double bin_width;           /* summarize histogram width (> 0 when summarize) */
    uint64_t hist_cap;          /* device histogram capacity in bins; 0 = 8192 (more bins
                                   take one exact follow-up pass) */
    uint64_t cand_cap;          /* order-statistic candidates per target; 0 = default
                                   (max(2^16, max_n/256)); overflow takes the exact
                                   multi-pass fallback -- results never depend on it */
} bmc_stats_req;

typedef struct {
    uint64_t n, horizon_count;
    bmc_summary summary;        /* valid when the request summarizes */
    uint64_t* exceed;           /* caller array [n_headways] (nullable): #{hit_horizon || d > h} */
    double* min_safe_headway;   /* caller array [n_risk] (nullable); +inf in the horizon tail */
    uint64_t* histogram;        /* caller array (nullable), at least summary.bins entries */
    size_t histogram_cap;
    uint32_t launches;          /* kernels the stage enqueued (rollout excluded) */
    uint32_t fallbacks;         /* order statistics that took the exact multi-pass path */
} bmc_stats;

/* Collective hooks for sharded (multi-GPU) statistics.  The stage calls them
 * at its three merge points with DEVICE buffers, ordered on `stream`
 * (NCCL on that stream, or torch.distributed with the stream made current).
 * Partials are exactly mergeable: SUM for counts / limbs / histograms, MIN
 * for the extrema keys; every rank then finishes with identical bits. */
enum { BMC_MERGE_SUM = 0, BMC_MERGE_MIN = 1, BMC_MERGE_MAX = 2 };
typedef struct {
    void* user;
    int32_t world;
    int32_t rank;
    int (*allreduce_u64)(void* user, uint64_t* buf, size_t count, int op, void* stream);
    /* recv holds world * count words, rank-ordered */
    int (*allgather_u64)(void* user, const uint64_t* send, uint64_t* recv, size_t count,
                         void* stream);
} bmc_merge;

typedef struct bmc_stats_stage bmc_stats_stage;
/* A stage sized for up to max_n results per call (candidate capacity). */
int bmc_stats_create(bmc_ctx* ctx, const bmc_stats_req* req, size_t max_n, bmc_stats_stage** out);
void bmc_stats_destroy(bmc_stats_stage* st);
/* Zero the partials (enqueued on stream; NULL = the context's stream). */
int bmc_stats_begin(bmc_stats_stage* st, void* stream);
/* Pass 1 over existing device outputs (when no fused rollout fed it). */
int bmc_stats_accumulate(bmc_stats_stage* st, const double* stop_distance,
                         const uint8_t* hit_horizon, size_t n, void* stream);
/* Merge (merge may be NULL: one device), pass 2, selection, read back and
 * host composition; synchronises the stream. d/hz are this rank's outputs. */
int bmc_stats_finish(bmc_stats_stage* st, const double* stop_distance, const uint8_t* hit_horizon,
                     size_t n, const bmc_merge* merge, bmc_stats* out, void* stream);
/* Rollout with pass 1 fused into its epilogue (st NULL: plain rollout).
 * Outputs as bmc_cuda_rollout_device; call bmc_stats_begin first. */
int bmc_cuda_rollout_stats(bmc_ctx* ctx, const bmc_terms* terms, size_t n,
                           const bmc_world* world, const bmc_run_opts* opts,
                           const bmc_outputs* out, unsigned long long* total_steps_dev,
                           bmc_stats_stage* st, void* stream);
/* bmc_cuda_run_model with pass 1 fused into every chunk's rollout (the
 * 1e9-sample stats-only stream); dev_out is required by the later passes. */
int bmc_cuda_run_model_stats(bmc_ctx* ctx, const bmc_model* model, uint64_t first, size_t n,
                             const bmc_world* world, const bmc_run_opts* opts, bmc_result* host_out,
                             const bmc_outputs* dev_out, uint64_t* clamp_count, bmc_run_info* info,
                             bmc_stats_stage* st);
/* One-call convenience over existing device outputs (begin + accumulate + finish). */
int bmc_cuda_stats(bmc_ctx* ctx, const double* stop_distance, const uint8_t* hit_horizon, size_t n,
                   const bmc_stats_req* req, bmc_stats* out);

/* Real-time decision with statistics: the graph additionally captures the
 * fused stage (no merge), so each decision also returns P(collision) per
 * headway / TTC threshold, min_safe_headway and (optionally) the summary. */
int bmc_cuda_graph_create_stats(bmc_ctx* ctx, size_t n, const bmc_world* world,
                                const bmc_run_opts* opts, const bmc_stats_req* req,
                                bmc_graph** out);
/* Statistics of the graph's last decision (host composition only). */
int bmc_cuda_graph_stats(bmc_graph* g, bmc_stats* out);

/* NCCL merge hooks for several devices driven from one process (the C++
 * MultiCudaRun): ncclCommInitAll over `devices`, one communicator per
 * device; bmc_nccl_merge(comm) is that rank's bmc_merge (ncclAllReduce /
 * ncclAllGather of u64 words on the stage's stream).  libnccl.so.2 is opened
 * at run time (BMC_NCCL_LIB overrides the path); BMC_E_CUDA when absent. */
typedef struct bmc_comm bmc_comm;
int bmc_nccl_available(int* version);
int bmc_nccl_init_all(int ndev, const int* devices, bmc_comm** comms);
const bmc_merge* bmc_nccl_merge(const bmc_comm* comm);
void bmc_nccl_destroy(bmc_comm* comm);

/* Device memory for callers without their own CUDA runtime (the C++
 * CudaRun keeps results in HBM through these). */
int bmc_cuda_alloc(bmc_ctx* ctx, size_t bytes, void** out);
int bmc_cuda_free(bmc_ctx* ctx, void* ptr);
int bmc_cuda_copy_to_host(bmc_ctx* ctx, void* host, const void* dev, size_t bytes);
int bmc_cuda_copy_to_device(bmc_ctx* ctx, void* dev, const void* host, size_t bytes);

/* ------------------------------------------------------- measurement */
/* FP64 DADD/DMUL issue-rate probe (the rollout's roofline denominator;
 * MEASURED_PEAKS.json carries no FP64 entry).  Independent chains of
 * unfused add/mul at full occupancy; best of `reps` launches, CUDA events. */
int bmc_cuda_fp64_peak(bmc_ctx* ctx, int reps, double* ops_per_s, double* best_ms);

#ifdef __cplusplus
}
#endif
#endif
