#pragma once

// brakemc/cuda_analysis.hpp -- the statistics stage on the B200, with the
// reference's own result types (/root/reference/proj/include/brakemc/
// analysis.hpp).  A CudaRun keeps one batch's rollout outputs in HBM and
// answers the analysis.cpp questions there, so nothing per-sample crosses
// PCIe unless results() is asked for:
//
//   summarize              analysis.cpp:13-76   exact counts/extrema/median/
//                                               histogram; mean/sd/skew via
//                                               double-double sums (<= few ulp)
//   convergence            analysis.cpp:85-124  prefix [0, n_k) reductions
//   collision_probability  analysis.cpp:145-159 exact count / n
//   min_safe_headway       analysis.cpp:161-194 exact order statistic (fused
//                                               statistics stage, bmc_cuda_stats)
//   build_risk_curve       analysis.cpp:203-228 one O(n log m) pass for the
//                                               whole grid (reference: O(n m))
//
// max_samples_within_budget_cuda is the reference's feasibility search
// (analysis.cpp:320-370) with the CUDA executor as the timed pipeline.
// Header-only over the C-ABI; the feasibility driver calls the reference's
// own max_feasible_n / median_wall_time_s (brakemc_core).

#include "brakemc/analysis.hpp"
#include "brakemc/cuda_executor.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <vector>

namespace brakemc {

class CudaRun {
public:
    CudaRun(const CudaRun&) = delete;
    CudaRun& operator=(const CudaRun&) = delete;
    CudaRun(CudaRun&& o) noexcept { *this = std::move(o); }
    CudaRun& operator=(CudaRun&& o) noexcept {
        std::swap(ctx_, o.ctx_);
        std::swap(d_, o.d_);
        std::swap(st_, o.st_);
        std::swap(hz_, o.hz_);
        std::swap(n_, o.n_);
        std::swap(dt_, o.dt_);
        std::swap(clamps_, o.clamps_);
        std::swap(wall_, o.wall_);
        return *this;
    }
    ~CudaRun() {
        if (ctx_) {
            bmc_cuda_free(ctx_, d_);
            bmc_cuda_free(ctx_, st_);
            bmc_cuda_free(ctx_, hz_);
        }
    }

    /// run_cuda semantics (index-aligned, bit-identical), outputs kept in HBM.
    static CudaRun from_batch(const SampleBatch& batch, const SimConfig& config,
                              const VehicleGeometry& geometry, const PhysicalConstants& constants,
                              const CudaExecOptions& options = {}, int device = 0) {
        if (batch.size() == 0) throw ConfigError("batch", "must be non-empty");
        CudaRun r(device, batch.size(), config.dt);
        r.clamps_ = batch.clamp_count;
        // device-resident run: stage terms on the host (same libm as the
        // reference), then the device rollout writes straight into HBM
        const bmc_world w = cuda_detail::world_of(config, geometry, constants);
        std::vector<double> t(4 * batch.size());
        const std::size_t n = batch.size();
        const auto start = std::chrono::steady_clock::now();
        int rc = bmc_stage_terms(reinterpret_cast<const bmc_sample*>(batch.samples.data()), n, &w,
                                 t.data(), t.data() + n, t.data() + 2 * n, t.data() + 3 * n,
                                 options.host_threads);
        if (rc != BMC_OK) cuda_detail::raise(rc, bmc_last_error());
        void* dterms = nullptr;
        rc = bmc_cuda_alloc(r.ctx_, 32 * n, &dterms);
        if (rc != BMC_OK) cuda_detail::raise(rc, bmc_cuda_last_error(r.ctx_));
        struct Guard {
            bmc_ctx* c;
            void* p;
            ~Guard() { bmc_cuda_free(c, p); }
        } guard{r.ctx_, dterms};
        rc = r.upload(dterms, t.data(), 32 * n);
        if (rc != BMC_OK) cuda_detail::raise(rc, bmc_cuda_last_error(r.ctx_));
        const double* dv = static_cast<const double*>(dterms);
        const bmc_terms terms{dv, dv + n, dv + 2 * n, dv + 3 * n};
        const bmc_outputs outs{static_cast<double*>(r.d_), static_cast<int32_t*>(r.st_),
                               static_cast<uint8_t*>(r.hz_)};
        const bmc_run_opts o = cuda_detail::opts_of(options);
        rc = bmc_cuda_rollout_device(r.ctx_, &terms, n, &w, &o, &outs, nullptr, nullptr);
        if (rc == BMC_OK) rc = bmc_cuda_sync(r.ctx_);
        if (rc != BMC_OK) cuda_detail::raise(rc, bmc_cuda_last_error(r.ctx_));
        r.wall_ = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
        return r;
    }

    /// Streaming: samples [first, first+n) of draw_batch(model, .) drawn on the
    /// host pool into pinned buffers, overlapped with the GPU; outputs in HBM
    /// (the 1e9-sample stats-only mode).
    static CudaRun from_model(const UncertaintyModel& model, std::size_t n,
                              const SimConfig& config, const VehicleGeometry& geometry,
                              const PhysicalConstants& constants,
                              const CudaExecOptions& options = {}, std::uint64_t first = 0,
                              int device = 0) {
        if (n == 0) throw ConfigError("samples", "must be >= 1");
        CudaRun r(device, n, config.dt);
        const bmc_world w = cuda_detail::world_of(config, geometry, constants);
        const bmc_model m = cuda_detail::model_of(model);
        const bmc_outputs outs{static_cast<double*>(r.d_), static_cast<int32_t*>(r.st_),
                               static_cast<uint8_t*>(r.hz_)};
        const bmc_run_opts o = cuda_detail::opts_of(options);
        bmc_run_info info{};
        std::uint64_t clamps = 0;
        const int rc = bmc_cuda_run_model(r.ctx_, &m, first, n, &w, &o, nullptr, &outs, &clamps, &info);
        if (rc != BMC_OK) cuda_detail::raise(rc, bmc_cuda_last_error(r.ctx_));
        r.clamps_ = clamps;
        r.wall_ = info.wall_s;
        return r;
    }

    std::size_t size() const { return n_; }
    std::uint64_t clamp_count() const { return clamps_; }
    double wall_time_s() const { return wall_; }

    /// Per-sample results back on the host (RolloutResult layout).
    std::vector<RolloutResult> results() const {
        std::vector<double> d(n_);
        std::vector<int32_t> st(n_);
        std::vector<uint8_t> hz(n_);
        check(bmc_cuda_copy_to_host(ctx_, d.data(), d_, 8 * n_));
        check(bmc_cuda_copy_to_host(ctx_, st.data(), st_, 4 * n_));
        check(bmc_cuda_copy_to_host(ctx_, hz.data(), hz_, n_));
        std::vector<RolloutResult> out(n_);
        for (std::size_t i = 0; i < n_; ++i) {
            out[i] = RolloutResult{d[i], static_cast<double>(st[i]) * dt_, st[i], hz[i] != 0};
        }
        return out;
    }

    /// summarize (analysis.cpp:13-76)
    DistributionSummary summarize(double bin_width = 2.0) const {
        bmc_summary s{};
        std::vector<uint64_t> hist(1u << 16);
        int rc = bmc_cuda_summarize(ctx_, dd(), hzp(), n_, bin_width, &s, hist.data(), hist.size());
        if (rc == BMC_E_RANGE) {
            hist.resize(s.bins);
            rc = bmc_cuda_summarize(ctx_, dd(), hzp(), n_, bin_width, &s, hist.data(), hist.size());
        }
        check(rc);
        DistributionSummary out;
        out.n = s.n;
        out.mean = s.mean;
        out.sd = s.sd;
        out.min = s.min;
        out.max = s.max;
        out.median = s.median;
        out.skewness = s.skewness;
        out.right_skewed = s.right_skewed != 0;
        out.horizon_count = s.horizon_count;
        out.histogram.origin = s.origin;
        out.histogram.bin_width = s.bin_width;
        out.histogram.counts.assign(hist.begin(), hist.begin() + static_cast<std::ptrdiff_t>(s.bins));
        return out;
    }

    /// collision_probability (analysis.cpp:145-159)
    double collision_probability(double headway_m) const {
        if (!(headway_m >= 0.0)) throw ConfigError("risk.headway", "must be >= 0");
        uint64_t c = 0;
        check(bmc_cuda_exceedance(ctx_, dd(), hzp(), n_, &headway_m, 1, &c));
        return static_cast<double>(c) / static_cast<double>(n_);
    }

    /// Collision probability per trigger TTC with sensor noise (BASELINE C4;
    /// an extension -- the reference has no noise model): sample i triggers
    /// at ttc + eps_i, eps_i = sigma * standard_normal_at(noise_seed, first_index + i)
    /// (sampling.cpp:48-53 on its own counter stream), and collides iff it
    /// hits the horizon or stops beyond (ttc + eps_i) * closing_speed.
    /// sigma = 0 gives collision_probability(ttc * closing_speed) exactly.
    std::vector<double> collision_probability_ttc_noise(const std::vector<double>& ttc,
                                                        double closing_speed, double sigma,
                                                        uint64_t noise_seed,
                                                        uint64_t first_index = 0) const {
        std::vector<uint64_t> c(ttc.size());
        check(bmc_cuda_exceedance_ttc_noise(ctx_, dd(), hzp(), n_, first_index, noise_seed, sigma,
                                            ttc.data(), ttc.size(), closing_speed, c.data()));
        std::vector<double> p(ttc.size());
        for (std::size_t j = 0; j < ttc.size(); ++j) {
            p[j] = static_cast<double>(c[j]) / static_cast<double>(n_);
        }
        return p;
    }

    /// min_safe_headway (analysis.cpp:161-194)
    double min_safe_headway(double risk) const { return min_safe_headways({risk})[0]; }

    /// min_safe_headway per level through the fused statistics stage: one
    /// level-1 bucket pass, compaction and exact selection (16 levels a call).
    std::vector<double> min_safe_headways(const std::vector<double>& risks) const {
        for (double risk : risks) {
            if (!(risk > 0.0 && risk < 1.0)) {
                throw ConfigError("risk.level", "must be strictly between 0 and 1");
            }
        }
        std::vector<double> vals(risks.size());
        for (std::size_t k0 = 0; k0 < risks.size(); k0 += 16) {
            const std::size_t m = std::min<std::size_t>(16, risks.size() - k0);
            bmc_stats_req q{};
            q.risk_levels = risks.data() + k0;
            q.n_risk = m;
            bmc_stats out{};
            out.min_safe_headway = vals.data() + k0;
            check(bmc_cuda_stats(ctx_, dd(), hzp(), n_, &q, &out));
        }
        return vals;
    }

    /// build_risk_curve (analysis.cpp:203-228)
    RiskCurve build_risk_curve(const std::vector<double>& grid,
                               const std::vector<double>& risk_levels,
                               double closing_speed_mps) const {
        RiskCurve curve;
        curve.headways_m = grid;
        std::vector<uint64_t> counts(grid.size());
        for (double h : grid) {
            if (!(h >= 0.0)) throw ConfigError("risk.headway", "must be >= 0");
        }
        if (!grid.empty()) {
            check(bmc_cuda_exceedance(ctx_, dd(), hzp(), n_, grid.data(), grid.size(), counts.data()));
        }
        for (uint64_t c : counts) {
            curve.probabilities.push_back(static_cast<double>(c) / static_cast<double>(n_));
        }
        for (std::size_t i = 1; i < curve.probabilities.size(); ++i) {
            if (curve.headways_m[i] >= curve.headways_m[i - 1] &&
                curve.probabilities[i] > curve.probabilities[i - 1]) {
                throw std::logic_error("risk curve must be non-increasing in headway");
            }
        }
        std::vector<double> levels = risk_levels;
        std::sort(levels.begin(), levels.end(), std::greater<>());
        const std::vector<double> heads = levels.empty() ? std::vector<double>{} : min_safe_headways(levels);
        for (std::size_t k = 0; k < levels.size(); ++k) {
            curve.thresholds.push_back(
                RiskThreshold{levels[k], heads[k], ttc_for_headway(heads[k], closing_speed_mps)});
        }
        return curve;
    }

    /// convergence_from_results (analysis.cpp:102-124) over prefixes of this run
    std::vector<ConvergenceRow> convergence(const std::vector<std::size_t>& n_values,
                                            std::size_t baseline_n = kConvergenceBaselineN) const {
        if (std::find(n_values.begin(), n_values.end(), baseline_n) == n_values.end()) {
            throw ConfigError("converge.n_values", "must include the baseline sample count");
        }
        for (std::size_t n : n_values) {
            if (n == 0 || n > n_) {
                throw ConfigError("converge.n_values", "entries must be in [1, master result count]");
            }
        }
        const auto base = prefix_stats(baseline_n);
        std::vector<ConvergenceRow> rows;
        for (std::size_t n : n_values) {
            const auto s = prefix_stats(n);
            rows.push_back(ConvergenceRow{n, s.first, s.second, s.first - base.first,
                                          s.second - base.second});
        }
        return rows;
    }

private:
    CudaRun(int device, std::size_t n, double dt) : n_(n), dt_(dt) {
        ctx_ = cuda_detail::context(device);
        check(bmc_cuda_alloc(ctx_, 8 * n, &d_));
        check(bmc_cuda_alloc(ctx_, 4 * n, &st_));
        check(bmc_cuda_alloc(ctx_, n, &hz_));
    }

    void check(int rc) const {
        if (rc != BMC_OK) cuda_detail::raise(rc, bmc_cuda_last_error(ctx_));
    }

    int upload(void* dev, const void* host, std::size_t bytes) const {
        return bmc_cuda_copy_to_device(ctx_, dev, host, bytes);
    }

    const double* dd() const { return static_cast<const double*>(d_); }
    const uint8_t* hzp() const { return static_cast<const uint8_t*>(hz_); }

    // prefix_stats (analysis.cpp:85-98): mean / sd (n-1) of the first n,
    // with the same exact sums as summarize (so the two agree bit for bit,
    // like the reference's identical formulas)
    std::pair<double, double> prefix_stats(std::size_t n) const {
        bmc_stats_req q{};
        q.summarize = 1;
        q.bin_width = 1e300;  // one bin: only the moments are wanted
        bmc_stats out{};
        check(bmc_cuda_stats(ctx_, dd(), hzp(), n, &q, &out));
        return {out.summary.mean, out.summary.sd};
    }

    bmc_ctx* ctx_ = nullptr;
    void* d_ = nullptr;
    void* st_ = nullptr;
    void* hz_ = nullptr;
    std::size_t n_ = 0;
    double dt_ = 0.0;
    std::uint64_t clamps_ = 0;
    double wall_ = 0.0;
};

/// max_samples_within_budget (analysis.cpp:320-370) with the CUDA executor:
/// each probe is median_wall_time_s of {draw the batch on the host pool,
/// run_cuda}, exactly the reference's timed pipeline with the executor
/// swapped; the winner is re-measured with generation and simulation split.
inline TimingReport max_samples_within_budget_cuda(const UncertaintyModel& model,
                                                   const SimConfig& config,
                                                   const VehicleGeometry& geometry,
                                                   const PhysicalConstants& constants,
                                                   const TimingBudget& budget,
                                                   const FeasibilityOptions& options = {},
                                                   const CudaExecOptions& cuda = {}) {
    budget.validate();
    TimingReport report;
    report.budget = budget;
    report.mc_budget_ms = budget.mc_budget_ms();
    const double budget_s = report.mc_budget_ms * 1e-3;
    const bmc_model m = cuda_detail::model_of(model);
    SampleBatch batch;
    auto draw = [&](std::size_t n) {
        batch.samples.resize(n);
        uint64_t clamps = 0;
        const int rc = bmc_draw_range(&m, 0, n, reinterpret_cast<bmc_sample*>(batch.samples.data()),
                                      &clamps, cuda.host_threads);
        if (rc != BMC_OK) cuda_detail::raise(rc, bmc_last_error());
        batch.clamp_count = clamps;
    };
    auto timed_run = [&](std::size_t n) {
        return median_wall_time_s(
            [&]() {
                draw(n);
                run_cuda(batch, config, geometry, constants, cuda);
            },
            options.timing_reps, options.timing_warmup);
    };
    report.max_samples = max_feasible_n(timed_run, budget_s, options.search_start,
                                        options.search_cap, &report.capped);
    report.meets_convergence_threshold = report.max_samples >= kConvergenceBaselineN;
    if (report.max_samples > 0) {
        std::vector<double> totals, sim_only;
        for (int rep = 0; rep < std::max(1, options.timing_reps); ++rep) {
            const auto g0 = std::chrono::steady_clock::now();
            draw(report.max_samples);
            const double gen_s =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - g0).count();
            const ExecutionReport run = run_cuda(batch, config, geometry, constants, cuda);
            totals.push_back(gen_s + run.wall_time_s);
            sim_only.push_back(run.wall_time_s);
        }
        auto median = [](std::vector<double> v) {
            std::sort(v.begin(), v.end());
            const std::size_t mid = v.size() / 2;
            return v.size() % 2 == 1 ? v[mid] : 0.5 * (v[mid - 1] + v[mid]);
        };
        report.time_with_sampling_s = median(totals);
        report.sim_only_time_s = median(sim_only);
    }
    return report;
}

}  // namespace brakemc
