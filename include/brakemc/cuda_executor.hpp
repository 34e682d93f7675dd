#pragma once

// brakemc/cuda_executor.hpp -- the B200 executor, a drop-in sibling of
// run_sequential / run_parallel (/root/reference/proj/include/brakemc/
// backends.hpp:32-45).  SPEC.md:311 names "an actual GPU backend ... behind
// the same executor interface" as the reference's extension point; this
// header is that backend.  A maintainer adds it next to backends.hpp and
// links libbrakemc_b200.so.
//
// Contract (mirrors backends.hpp:22-45 and SPEC.md:261-269, 317):
//   * results[i] is index-aligned with batch.samples[i] and all four fields
//     are bit-identical to simulate_rollout (integrator.cpp:13-29);
//   * wall_time_s covers the rollout only (terms staging, H2D, kernels, D2H),
//     never batch generation (backends.hpp:22-24);
//   * externally synchronous; results are independent of device count,
//     chunking and scheduling (like worker_count / chunk_size);
//   * ConfigError("batch", "must be non-empty") on an empty batch
//     (backends.cpp:41-43); std::domain_error from friction_limit;
//     CUDA failures -> std::runtime_error.  No CPU fallback.
//
// Header-only over the C-ABI (brakemc_cuda.h): nothing here needs the
// reference's object code, only its value types.

#include "brakemc/backends.hpp"
#include "brakemc/errors.hpp"
#include "brakemc/sampling.hpp"
#include "brakemc_cuda.h"

#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace brakemc {

// backends.hpp:18 has {sequential, parallel}; the one-line enum extension a
// maintainer makes is `cuda` (value 2).  Not "gpu": test_io_cli.cpp:103-104
// requires executor_from_string("gpu") to keep throwing.
inline constexpr ExecutorKind kCudaExecutorKind = static_cast<ExecutorKind>(2);

struct CudaExecOptions {
    std::vector<int> devices{0};  ///< one host thread + context per device; empty = all
    int host_threads = 0;         ///< host staging threads; 0 = hardware concurrency
    std::size_t chunk_samples = 0;///< pipeline chunk; 0 = default (timing only)
    int schedule = 0;             ///< 0 default, 1 index order, 2 binned (timing only)
    int block_threads = 0;        ///< 0 default (timing only)
    int table_mode = 0;           ///< 0 auto (timing only)
    int ilp = 0;                  ///< samples per thread, 0 default (timing only)
    int sampler = 0;              ///< model-driven runs: 0 auto, 1 host pool, 2 device (timing only)
    int test_block = 0;           ///< termination test every step (1) or per 8-step block (8) (timing only)
};

static_assert(sizeof(ScenarioSample) == sizeof(bmc_sample), "ScenarioSample layout");
static_assert(sizeof(RolloutResult) == sizeof(bmc_result), "RolloutResult layout");

namespace cuda_detail {

[[noreturn]] inline void raise(int rc, const char* msg) {
    const std::string m = msg ? msg : "";
    if (rc == BMC_E_CONFIG) {
        const auto colon = m.find(": ");
        if (colon != std::string::npos) throw ConfigError(m.substr(0, colon), m.substr(colon + 2));
        throw ConfigError("execution", m);
    }
    if (rc == BMC_E_DOMAIN) throw std::domain_error(m);
    throw std::runtime_error("cuda executor: " + m);
}

// One cached context per device for the life of the process (the reference
// functions are reentrant; contexts serialise their own use internally).
inline bmc_ctx* context(int device) {
    static std::mutex mu;
    static std::map<int, bmc_ctx*> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(device);
    if (it != cache.end()) return it->second;
    bmc_ctx* ctx = nullptr;
    const int rc = bmc_cuda_init(device, &ctx);
    if (rc != BMC_OK) raise(rc, bmc_last_error());
    cache[device] = ctx;
    return ctx;
}

inline bmc_world world_of(const SimConfig& c, const VehicleGeometry& g, const PhysicalConstants& p) {
    return bmc_world{c.dt, c.t_max, c.brake_cmd, g.cg_height, g.wheelbase, g.actuator_tau,
                     p.gravity, p.air_density, p.frontal_area};
}

inline bmc_run_opts opts_of(const CudaExecOptions& o) {
    bmc_run_opts r{};
    r.schedule = o.schedule;
    r.block_threads = o.block_threads;
    r.table_mode = o.table_mode;
    r.host_threads = o.host_threads;
    r.chunk_samples = o.chunk_samples;
    r.ilp = o.ilp;
    r.sampler = o.sampler;
    r.test_block = o.test_block;
    return r;
}

inline bmc_model model_of(const UncertaintyModel& m) {
    return bmc_model{m.seed,
                     {m.initial_speed.mean, m.initial_speed.sd},
                     {m.friction.mean, m.friction.sd},
                     {m.grade.mean, m.grade.sd},
                     {m.mass.mean, m.mass.sd},
                     {m.drag_coeff.mean, m.drag_coeff.sd}};
}

}  // namespace cuda_detail

/// Runs every sample on the selected B200s: contiguous index shards, one
/// host thread and context per device, disjoint result slices (no merge
/// needed).  Bit-identical to run_sequential on the same batch.
inline ExecutionReport run_cuda(const SampleBatch& batch, const SimConfig& config,
                                const VehicleGeometry& geometry,
                                const PhysicalConstants& constants,
                                const CudaExecOptions& options = {}) {
    if (batch.size() == 0) {
        throw ConfigError("batch", "must be non-empty");
    }
    std::vector<int> devices = options.devices;
    if (devices.empty()) {
        int count = 0;
        if (bmc_device_count(&count) != BMC_OK || count == 0) {
            cuda_detail::raise(BMC_E_CUDA, "no CUDA device");
        }
        for (int d = 0; d < count; ++d) devices.push_back(d);
    }
    if (devices.size() > batch.size()) devices.resize(batch.size());

    ExecutionReport report;
    report.executor = kCudaExecutorKind;
    report.worker_count = static_cast<unsigned>(devices.size());
    report.results.resize(batch.size());

    const bmc_world w = cuda_detail::world_of(config, geometry, constants);
    const bmc_run_opts opts = cuda_detail::opts_of(options);

    std::vector<bmc_ctx*> ctxs;
    for (int d : devices) ctxs.push_back(cuda_detail::context(d));

    const std::size_t n = batch.size();
    const std::size_t G = devices.size();
    std::vector<int> codes(G, BMC_OK);
    std::vector<std::string> msgs(G);
    auto shard = [&](std::size_t g) {
        const std::size_t b = n * g / G, e = n * (g + 1) / G;
        const auto* in = reinterpret_cast<const bmc_sample*>(batch.samples.data() + b);
        auto* out = reinterpret_cast<bmc_result*>(report.results.data() + b);
        codes[g] = bmc_cuda_run(ctxs[g], in, e - b, &w, &opts, out, nullptr);
        if (codes[g] != BMC_OK) msgs[g] = bmc_cuda_last_error(ctxs[g]);
    };

    const auto start = std::chrono::steady_clock::now();
    if (G == 1) {
        shard(0);
    } else {
        std::vector<std::thread> pool;
        for (std::size_t g = 0; g < G; ++g) pool.emplace_back(shard, g);
        for (auto& t : pool) t.join();
    }
    report.wall_time_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    for (std::size_t g = 0; g < G; ++g) {
        if (codes[g] != BMC_OK) cuda_detail::raise(codes[g], msgs[g].c_str());
    }
    return report;
}

/// "cuda" for the extended kind, else the reference's own to_string.
inline const char* executor_name(ExecutorKind kind) {
    return kind == kCudaExecutorKind ? "cuda" : to_string(kind);
}

/// executor_from_string (run_config.cpp:107-115) extended with "cuda".
/// Every other name keeps the reference's behaviour: "gpu" still throws
/// (test_io_cli.cpp:103-104).
inline ExecutorKind executor_from_string_with_cuda(const std::string& name) {
    if (name == "sequential") return ExecutorKind::sequential;
    if (name == "parallel") return ExecutorKind::parallel;
    if (name == "cuda") return kCudaExecutorKind;
    throw ConfigError("execution.executor", "must be \"sequential\", \"parallel\" or \"cuda\"");
}

/// run_configured_executor (cli.cpp:20-26) with the cuda branch.
inline ExecutionReport run_executor(ExecutorKind kind, const SampleBatch& batch,
                                    const SimConfig& config, const VehicleGeometry& geometry,
                                    const PhysicalConstants& constants, unsigned workers = 0,
                                    std::size_t chunk_size = 256,
                                    const CudaExecOptions& cuda = {}) {
    if (kind == kCudaExecutorKind) return run_cuda(batch, config, geometry, constants, cuda);
    if (kind == ExecutorKind::sequential) {
        return run_sequential(batch, config, geometry, constants);
    }
    return run_parallel(batch, config, geometry, constants, workers, chunk_size);
}

}  // namespace brakemc
