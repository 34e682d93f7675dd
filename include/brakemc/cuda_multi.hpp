#pragma once

// brakemc/cuda_multi.hpp -- several B200s from one process with merged
// statistics: contiguous index shards, one host thread and
// context per device, outputs kept in each device's HBM, and the
// analysis.cpp statistics of the WHOLE batch computed by the fused
// statistics stage with its three merge points running over a Collective:
//
//   NcclCollective   ncclCommInitAll over the devices; ncclAllReduce /
//                    ncclAllGather of u64 words on each stage's stream
//                    (bmc_nccl_*; libnccl opened at run time)
//   (tests)          an in-process fake over host memory drives the same
//                    orchestration on CPU (tests/cpp/merge_main.cpp)
//
// Merged partials are exact (integer counts, u64 limbs of exact sums, min
// keys), so every field equals a single-device run bit for bit, for any
// device count.  Header-only over the C-ABI (brakemc_cuda.h).

#include "brakemc/analysis.hpp"
#include "brakemc/cuda_executor.hpp"

#include <cstdint>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace brakemc {

/// What the statistics stage computes (analysis.cpp:13-76, 145-194).
struct CudaStatsRequest {
    std::vector<double> headways;     ///< collision_probability grid (each >= 0)
    std::vector<double> risk_levels;  ///< min_safe_headway levels in (0, 1), at most 16
    bool summarize = false;           ///< full DistributionSummary
    double bin_width = 2.0;           ///< summarize histogram width
};

/// The merged answer (identical on every rank).
struct CudaStats {
    std::size_t n = 0;
    std::size_t horizon_count = 0;
    std::vector<std::uint64_t> exceed_counts;  ///< #{hit_horizon || d > h} per headway
    std::vector<double> collision_probability; ///< exceed_counts / n (analysis.cpp:158)
    std::vector<double> min_safe_headway;      ///< per risk level; +inf in the horizon tail
    DistributionSummary summary;               ///< when summarize
    unsigned fallbacks = 0;                    ///< exact multi-pass selections taken
};

/// Merge interface of the statistics stage: rank r's hooks over buffers in
/// rank r's memory, ordered on `stream`.  op: BMC_MERGE_SUM / MIN / MAX of
/// uint64 words; allgather: recv holds world() * count words, rank-ordered.
class Collective {
public:
    virtual ~Collective() = default;
    virtual int world() const = 0;
    virtual int allreduce_u64(int rank, std::uint64_t* buf, std::size_t count, int op,
                              void* stream) = 0;
    virtual int allgather_u64(int rank, const std::uint64_t* send, std::uint64_t* recv,
                              std::size_t count, void* stream) = 0;

    /// The bmc_merge the C-ABI stage calls for rank r (callable from every
    /// rank's thread).
    virtual bmc_merge merge(int rank) {
        {
            std::lock_guard<std::mutex> lk(hooks_mu_);
            if (hooks_.empty()) {
                for (int r = 0; r < world(); ++r) hooks_.push_back(Hook{this, r});
            }
        }
        bmc_merge m{};
        m.user = &hooks_[static_cast<std::size_t>(rank)];
        m.world = world();
        m.rank = rank;
        m.allreduce_u64 = [](void* u, uint64_t* b, size_t c, int op, void* s) {
            auto* h = static_cast<Hook*>(u);
            return h->self->allreduce_u64(h->rank, b, c, op, s);
        };
        m.allgather_u64 = [](void* u, const uint64_t* sb, uint64_t* rb, size_t c, void* s) {
            auto* h = static_cast<Hook*>(u);
            return h->self->allgather_u64(h->rank, sb, rb, c, s);
        };
        return m;
    }

private:
    struct Hook {
        Collective* self;
        int rank;
    };
    std::mutex hooks_mu_;
    std::vector<Hook> hooks_;  // built once; rank r's hook address is stable
};

/// NCCL over devices of this process (one communicator per device).
class NcclCollective : public Collective {
public:
    explicit NcclCollective(const std::vector<int>& devices) : comms_(devices.size(), nullptr) {
        for (std::size_t i = 0; i < devices.size(); ++i) {
            for (std::size_t j = 0; j < i; ++j) {
                if (devices[i] == devices[j]) {
                    throw ConfigError("execution.devices", "NCCL needs distinct devices");
                }
            }
        }
        const int rc = bmc_nccl_init_all(static_cast<int>(devices.size()), devices.data(),
                                         comms_.data());
        if (rc != BMC_OK) cuda_detail::raise(rc, bmc_last_error());
    }
    ~NcclCollective() override {
        for (bmc_comm* c : comms_) bmc_nccl_destroy(c);
    }
    NcclCollective(const NcclCollective&) = delete;
    NcclCollective& operator=(const NcclCollective&) = delete;

    int world() const override { return static_cast<int>(comms_.size()); }
    int allreduce_u64(int rank, std::uint64_t* buf, std::size_t count, int op,
                      void* stream) override {
        const bmc_merge* m = bmc_nccl_merge(comms_[static_cast<std::size_t>(rank)]);
        return m->allreduce_u64(m->user, buf, count, op, stream);
    }
    int allgather_u64(int rank, const std::uint64_t* send, std::uint64_t* recv, std::size_t count,
                      void* stream) override {
        const bmc_merge* m = bmc_nccl_merge(comms_[static_cast<std::size_t>(rank)]);
        return m->allgather_u64(m->user, send, recv, count, stream);
    }
    bmc_merge merge(int rank) override { return *bmc_nccl_merge(comms_[static_cast<std::size_t>(rank)]); }

private:
    std::vector<bmc_comm*> comms_;
};

namespace cuda_detail {

/// bmc_stats_req view of a request (arrays stay owned by `r`).
inline bmc_stats_req stats_req_of(const CudaStatsRequest& r) {
    bmc_stats_req q{};
    q.headways = r.headways.empty() ? nullptr : r.headways.data();
    q.n_headways = r.headways.size();
    q.risk_levels = r.risk_levels.empty() ? nullptr : r.risk_levels.data();
    q.n_risk = r.risk_levels.size();
    q.summarize = r.summarize ? 1 : 0;
    q.bin_width = r.bin_width;
    return q;
}

/// Caller-owned result arrays of one bmc_stats, then the C++ result.
struct StatsBuffers {
    std::vector<std::uint64_t> exceed, hist;
    std::vector<double> msh;
    bmc_stats s{};
    explicit StatsBuffers(const CudaStatsRequest& r, std::size_t hist_cap = 1u << 16)
        : exceed(r.headways.size()), hist(hist_cap), msh(r.risk_levels.size()) {
        s.exceed = exceed.empty() ? nullptr : exceed.data();
        s.min_safe_headway = msh.empty() ? nullptr : msh.data();
        s.histogram = hist.data();
        s.histogram_cap = hist.size();
    }
    CudaStats result(const CudaStatsRequest& r) const {
        CudaStats o;
        o.n = s.n;
        o.horizon_count = s.horizon_count;
        o.exceed_counts = exceed;
        for (std::uint64_t c : exceed) {
            o.collision_probability.push_back(static_cast<double>(c) / static_cast<double>(s.n));
        }
        o.min_safe_headway = msh;
        o.fallbacks = s.fallbacks;
        if (r.summarize) {
            DistributionSummary& d = o.summary;
            d.n = s.summary.n;
            d.mean = s.summary.mean;
            d.sd = s.summary.sd;
            d.min = s.summary.min;
            d.max = s.summary.max;
            d.median = s.summary.median;
            d.skewness = s.summary.skewness;
            d.right_skewed = s.summary.right_skewed != 0;
            d.horizon_count = s.summary.horizon_count;
            d.histogram.origin = s.summary.origin;
            d.histogram.bin_width = s.summary.bin_width;
            d.histogram.counts.assign(hist.begin(),
                                      hist.begin() + static_cast<std::ptrdiff_t>(s.summary.bins));
        }
        return o;
    }
};

}  // namespace cuda_detail

/// One batch simulated across several devices, outputs kept in each
/// device's HBM; statistics merged over a Collective (NCCL by default).
class MultiCudaRun {
public:
    MultiCudaRun(const MultiCudaRun&) = delete;
    MultiCudaRun& operator=(const MultiCudaRun&) = delete;
    MultiCudaRun(MultiCudaRun&&) = default;
    MultiCudaRun& operator=(MultiCudaRun&&) = default;
    ~MultiCudaRun() {
        for (Shard& s : shards_) {
            if (s.ctx) {
                bmc_cuda_free(s.ctx, s.d);
                bmc_cuda_free(s.ctx, s.st);
                bmc_cuda_free(s.ctx, s.hz);
            }
        }
    }

    /// Samples [0, n) of draw_batch(model, n): device g draws and simulates
    /// its contiguous shard [g n / G, (g+1) n / G) (bmc_cuda_run_model), so
    /// no batch is materialised on the host.  Host staging threads default
    /// to the host's cores divided among the devices.
    static MultiCudaRun from_model(const UncertaintyModel& model, std::size_t n,
                                   const SimConfig& config, const VehicleGeometry& geometry,
                                   const PhysicalConstants& constants,
                                   const CudaExecOptions& options = {}) {
        if (n == 0) throw ConfigError("samples", "must be >= 1");
        MultiCudaRun r(options, n);
        const bmc_world w = cuda_detail::world_of(config, geometry, constants);
        const bmc_model m = cuda_detail::model_of(model);
        const bmc_run_opts o = r.shard_opts(options);
        r.for_each_shard([&](Shard& s) {
            const bmc_outputs outs{static_cast<double*>(s.d), static_cast<int32_t*>(s.st),
                                   static_cast<uint8_t*>(s.hz)};
            std::uint64_t clamps = 0;
            bmc_run_info info{};
            const int rc = bmc_cuda_run_model(s.ctx, &m, s.first, s.n, &w, &o, nullptr, &outs,
                                              &clamps, &info);
            s.clamps = clamps;
            return rc;
        });
        return r;
    }

    /// A host batch split into device shards (run_cuda semantics per shard).
    static MultiCudaRun from_batch(const SampleBatch& batch, const SimConfig& config,
                                   const VehicleGeometry& geometry,
                                   const PhysicalConstants& constants,
                                   const CudaExecOptions& options = {}) {
        if (batch.size() == 0) throw ConfigError("batch", "must be non-empty");
        MultiCudaRun r(options, batch.size());
        const bmc_world w = cuda_detail::world_of(config, geometry, constants);
        const bmc_run_opts o = r.shard_opts(options);
        r.for_each_shard([&](Shard& s) {
            std::vector<double> t(4 * s.n);
            int rc = bmc_stage_terms(reinterpret_cast<const bmc_sample*>(batch.samples.data() + s.first),
                                     s.n, &w, t.data(), t.data() + s.n, t.data() + 2 * s.n,
                                     t.data() + 3 * s.n, o.host_threads);
            if (rc != BMC_OK) return rc;
            void* dt = nullptr;
            if ((rc = bmc_cuda_alloc(s.ctx, 32 * s.n, &dt)) != BMC_OK) return rc;
            rc = bmc_cuda_copy_to_device(s.ctx, dt, t.data(), 32 * s.n);
            const double* dv = static_cast<const double*>(dt);
            const bmc_terms terms{dv, dv + s.n, dv + 2 * s.n, dv + 3 * s.n};
            const bmc_outputs outs{static_cast<double*>(s.d), static_cast<int32_t*>(s.st),
                                   static_cast<uint8_t*>(s.hz)};
            if (rc == BMC_OK) rc = bmc_cuda_rollout_device(s.ctx, &terms, s.n, &w, &o, &outs, nullptr, nullptr);
            if (rc == BMC_OK) rc = bmc_cuda_sync(s.ctx);
            bmc_cuda_free(s.ctx, dt);
            return rc;
        });
        r.clamps_total_ = batch.clamp_count;
        return r;
    }

    std::size_t size() const { return n_; }
    std::size_t devices() const { return shards_.size(); }

    /// The statistics of the whole batch: every device runs the stage over
    /// its shard and the merge points run over `coll` (nullptr: NCCL over
    /// this run's devices, created on first use).  Bit-identical to a
    /// single-device run for any device count.
    CudaStats statistics(const CudaStatsRequest& req, Collective* coll = nullptr) const {
        if (!coll) {
            if (!nccl_) {
                std::vector<int> devs;
                for (const Shard& s : shards_) devs.push_back(s.device);
                nccl_ = std::make_unique<NcclCollective>(devs);
            }
            coll = nccl_.get();
        }
        if (coll->world() != static_cast<int>(shards_.size())) {
            throw ConfigError("execution.devices", "collective world differs from the device count");
        }
        // every rank's stage runs under its device context's lock while it
        // waits in the collective: two ranks on one device would deadlock
        for (std::size_t i = 0; i < shards_.size(); ++i) {
            for (std::size_t j = 0; j < i; ++j) {
                if (shards_[i].device == shards_[j].device) {
                    throw ConfigError("execution.devices", "merged statistics need distinct devices");
                }
            }
        }
        const bmc_stats_req q = cuda_detail::stats_req_of(req);
        std::vector<std::unique_ptr<cuda_detail::StatsBuffers>> bufs;
        for (std::size_t g = 0; g < shards_.size(); ++g) {
            bufs.push_back(std::make_unique<cuda_detail::StatsBuffers>(req));
        }
        std::vector<bmc_merge> merges;
        for (std::size_t g = 0; g < shards_.size(); ++g) merges.push_back(coll->merge(static_cast<int>(g)));
        const_cast<MultiCudaRun*>(this)->for_each_shard([&](Shard& s) {
            bmc_stats_stage* st = nullptr;
            int rc = bmc_stats_create(s.ctx, &q, s.n, &st);
            if (rc != BMC_OK) return rc;
            if ((rc = bmc_stats_begin(st, nullptr)) == BMC_OK &&
                (rc = bmc_stats_accumulate(st, static_cast<const double*>(s.d),
                                           static_cast<const uint8_t*>(s.hz), s.n, nullptr)) == BMC_OK) {
                rc = bmc_stats_finish(st, static_cast<const double*>(s.d),
                                      static_cast<const uint8_t*>(s.hz), s.n, &merges[s.rank],
                                      &bufs[s.rank]->s, nullptr);
            }
            bmc_stats_destroy(st);
            return rc;
        });
        return bufs[0]->result(req);
    }

    /// Per-sample results gathered to the host (RolloutResult layout).
    std::vector<RolloutResult> results(double dt) const {
        std::vector<RolloutResult> out(n_);
        const_cast<MultiCudaRun*>(this)->for_each_shard([&](Shard& s) {
            std::vector<double> d(s.n);
            std::vector<int32_t> st(s.n);
            std::vector<uint8_t> hz(s.n);
            int rc = bmc_cuda_copy_to_host(s.ctx, d.data(), s.d, 8 * s.n);
            if (rc == BMC_OK) rc = bmc_cuda_copy_to_host(s.ctx, st.data(), s.st, 4 * s.n);
            if (rc == BMC_OK) rc = bmc_cuda_copy_to_host(s.ctx, hz.data(), s.hz, s.n);
            for (std::size_t i = 0; i < s.n; ++i) {
                out[s.first + i] = RolloutResult{d[i], static_cast<double>(st[i]) * dt, st[i], hz[i] != 0};
            }
            return rc;
        });
        return out;
    }

private:
    struct Shard {
        int device = 0, rank = 0;
        bmc_ctx* ctx = nullptr;
        std::size_t first = 0, n = 0;
        void *d = nullptr, *st = nullptr, *hz = nullptr;
        std::uint64_t clamps = 0;
    };

    MultiCudaRun(const CudaExecOptions& options, std::size_t n) : n_(n) {
        std::vector<int> devices = options.devices;
        if (devices.empty()) {
            int count = 0;
            if (bmc_device_count(&count) != BMC_OK || count == 0) cuda_detail::raise(BMC_E_CUDA, "no CUDA device");
            for (int d = 0; d < count; ++d) devices.push_back(d);
        }
        if (devices.size() > n) devices.resize(n);
        const std::size_t G = devices.size();
        for (std::size_t g = 0; g < G; ++g) {
            Shard s;
            s.device = devices[g];
            s.rank = static_cast<int>(g);
            s.ctx = cuda_detail::context(s.device);
            s.first = n * g / G;
            s.n = n * (g + 1) / G - s.first;
            check(s.ctx, bmc_cuda_alloc(s.ctx, 8 * s.n, &s.d));
            check(s.ctx, bmc_cuda_alloc(s.ctx, 4 * s.n, &s.st));
            check(s.ctx, bmc_cuda_alloc(s.ctx, s.n, &s.hz));
            shards_.push_back(s);
        }
    }

    static void check(bmc_ctx* ctx, int rc) {
        if (rc != BMC_OK) cuda_detail::raise(rc, bmc_cuda_last_error(ctx));
    }

    bmc_run_opts shard_opts(const CudaExecOptions& options) const {
        bmc_run_opts o = cuda_detail::opts_of(options);
        if (o.host_threads == 0 && shards_.size() > 1) {
            // the host's cores divided among the devices (no oversubscription)
            const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
            o.host_threads = static_cast<int>(std::max<std::size_t>(1, hc / shards_.size()));
        }
        return o;
    }

    // One host thread per device (the collective's ranks must all be live).
    template <class F>
    void for_each_shard(F&& f) {
        std::vector<int> codes(shards_.size(), BMC_OK);
        std::vector<std::string> msgs(shards_.size());
        auto body = [&](std::size_t g) {
            codes[g] = f(shards_[g]);
            if (codes[g] != BMC_OK) msgs[g] = bmc_cuda_last_error(shards_[g].ctx);
        };
        if (shards_.size() == 1) {
            body(0);
        } else {
            std::vector<std::thread> pool;
            for (std::size_t g = 0; g < shards_.size(); ++g) pool.emplace_back(body, g);
            for (auto& t : pool) t.join();
        }
        for (std::size_t g = 0; g < shards_.size(); ++g) {
            if (codes[g] != BMC_OK) cuda_detail::raise(codes[g], msgs[g].c_str());
        }
    }

    std::vector<Shard> shards_;
    std::size_t n_ = 0;
    std::uint64_t clamps_total_ = 0;
    mutable std::unique_ptr<NcclCollective> nccl_;
};

}  // namespace brakemc
