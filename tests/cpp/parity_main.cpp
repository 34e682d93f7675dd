// parity_main.cpp -- the reference's executor parity checks, re-run against
// brakemc::run_cuda through the reference's own C++ API.
//
// Links the UNMODIFIED reference (oracle/_ref/libbrakemc_ref.so: draw_batch,
// run_sequential, run_parallel, verify_consistency) and the product library
// (libbrakemc_b200.so via include/brakemc/cuda_executor.hpp).  Mirrors:
//   * acceptance criterion 1, backend_bit_exactness
//     (tests/acceptance/acceptance_main.cpp:65-107): seeds {1,2,3} x
//     n {1k, 12k, 100k}, pass and max_abs_deviation == 0.0;
//   * test_backends.cpp:26-68: single-sample report, chunk/scheduling
//     independence, repeat determinism, empty-batch ConfigError.
// Exit 0 on success; prints one line per check.  Run by
// tests/test_gpu_parity.py::test_cpp_executor_api on the GPU box.
#include "brakemc/backends.hpp"
#include "brakemc/cuda_analysis.hpp"
#include "brakemc/cuda_executor.hpp"
#include "brakemc/cuda_multi.hpp"
#include "brakemc/errors.hpp"
#include "brakemc/sampling.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

using namespace brakemc;

namespace {

int failures = 0;

void check(bool ok, const std::string& what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}

SampleBatch batch_of(std::uint64_t seed, std::size_t n, bool mixed = false) {
    UncertaintyModel m;
    m.seed = seed;
    if (mixed) {
        m.friction = NormalSpec{0.45, 0.20};
        m.grade = NormalSpec{0.0, std::atan(0.06)};
    }
    return draw_batch(m, n);
}

}  // namespace

int main(int argc, char** argv) {
    const bool quick = argc > 1 && std::string(argv[1]) == "--quick";
    const SimConfig cfg{};
    const VehicleGeometry geo{};
    const PhysicalConstants phys{};

    // acceptance_main.cpp:65-107 (criterion 1) with run_cuda as the backend
    for (std::uint64_t seed : {1ull, 2ull, 3ull}) {
        for (std::size_t n : {std::size_t{1000}, std::size_t{12000}, std::size_t{100000}}) {
            if (quick && n > 12000) continue;
            const SampleBatch b = batch_of(seed, n);
            const ExecutionReport ref = run_parallel(b, cfg, geo, phys, 0);
            const ExecutionReport gpu = run_cuda(b, cfg, geo, phys);
            const ConsistencyVerdict v = verify_consistency(ref, gpu);
            check(v.pass && v.max_abs_deviation == 0.0 && v.bitwise_equal &&
                      gpu.worker_count == 1 && gpu.executor == kCudaExecutorKind,
                  "criterion1 seed=" + std::to_string(seed) + " n=" + std::to_string(n));
        }
    }

    // mixed-condition (divergence-heavy, ~27% horizon hits) batch
    {
        const SampleBatch b = batch_of(3, quick ? 20000 : 100000, true);
        const ExecutionReport ref = run_parallel(b, cfg, geo, phys, 0);
        const ExecutionReport gpu = run_cuda(b, cfg, geo, phys);
        check(verify_consistency(ref, gpu).pass, "mixed model bit-exact");
    }

    // test_backends.cpp:26-36: a single-sample report equals the rollout
    {
        const SampleBatch b = batch_of(3, 1);
        const ExecutionReport gpu = run_cuda(b, cfg, geo, phys);
        const RolloutResult direct = simulate_rollout(b.samples[0], cfg, geo, phys);
        check(gpu.results.size() == 1 && gpu.results[0].stop_distance == direct.stop_distance &&
                  gpu.results[0].steps == direct.steps &&
                  gpu.results[0].stop_time == direct.stop_time &&
                  gpu.results[0].hit_horizon == direct.hit_horizon,
              "single-sample report equals simulate_rollout");
    }

    // test_backends.cpp:52-68: scheduling knobs never change results
    {
        const SampleBatch b = batch_of(5, 7000, true);
        const ExecutionReport ref = run_sequential(b, cfg, geo, phys);
        bool all = true;
        for (int sched : {1, 2}) {
            for (int tm : {1, 2, 3}) {
                for (std::size_t chunk : {std::size_t{0}, std::size_t{999}}) {
                    CudaExecOptions o;
                    o.schedule = sched;
                    o.table_mode = tm;
                    o.chunk_samples = chunk;
                    o.block_threads = tm == 3 ? 256 : 512;
                    all = all && verify_consistency(ref, run_cuda(b, cfg, geo, phys, o)).pass;
                }
            }
        }
        check(all, "schedule / table mode / chunk independence");
        const ExecutionReport a1 = run_cuda(b, cfg, geo, phys);
        const ExecutionReport a2 = run_cuda(b, cfg, geo, phys);
        check(verify_consistency(a1, a2).pass, "repeated runs identical");
    }

    // non-default configs (horizon shorter than the actuator fixed point, etc.)
    {
        const SampleBatch b = batch_of(8, 3000, true);
        bool all = true;
        SimConfig c2 = cfg;
        c2.t_max = 3.0;  // max_steps 3000 < actuator fixed point (4803)
        VehicleGeometry g2 = geo;
        g2.actuator_tau = 0.4;
        SimConfig c3 = cfg;
        c3.dt = 0.002;
        c3.brake_cmd = -8.0;
        all = all && verify_consistency(run_sequential(b, c2, geo, phys), run_cuda(b, c2, geo, phys)).pass;
        all = all && verify_consistency(run_sequential(b, cfg, g2, phys), run_cuda(b, cfg, g2, phys)).pass;
        all = all && verify_consistency(run_sequential(b, c3, geo, phys), run_cuda(b, c3, geo, phys)).pass;
        check(all, "non-default SimConfig / geometry bit-exact");
    }

    // analysis.cpp on the device (CudaRun) vs the reference's host analysis
    {
        UncertaintyModel m;
        m.seed = 3;
        m.friction = NormalSpec{0.45, 0.20};
        m.grade = NormalSpec{0.0, std::atan(0.06)};
        const std::size_t n = quick ? 20000 : 60000;
        const SampleBatch b = draw_batch(m, n);
        const ExecutionReport ref = run_parallel(b, cfg, geo, phys, 0);
        const CudaRun run = CudaRun::from_batch(b, cfg, geo, phys);
        ExecutionReport back;
        back.results = run.results();
        check(verify_consistency(ref, back).pass, "CudaRun::from_batch results bit-exact");
        const CudaRun streamed = CudaRun::from_model(m, n, cfg, geo, phys);
        back.results = streamed.results();
        check(verify_consistency(ref, back).pass && streamed.clamp_count() == b.clamp_count,
              "CudaRun::from_model (streamed sampler) bit-exact, clamp count equal");

        const DistributionSummary want = summarize(ref.results, 2.0);
        const DistributionSummary got = run.summarize(2.0);
        const auto rel = [](double a, double b) { return std::abs(a - b) <= 1e-12 * std::abs(b); };
        check(got.n == want.n && got.horizon_count == want.horizon_count && got.min == want.min &&
                  got.max == want.max && got.median == want.median &&
                  got.histogram.origin == want.histogram.origin &&
                  got.histogram.counts == want.histogram.counts &&
                  got.right_skewed == want.right_skewed && rel(got.mean, want.mean) &&
                  rel(got.sd, want.sd) && std::abs(got.skewness - want.skewness) <= 1e-9,
              "summarize: counts/extrema/median/histogram exact, moments <= 1e-12 rel");

        bool cp = true;
        for (double h : {0.0, 50.0, 77.7, 120.0, 400.0, 1e9}) {
            cp = cp && run.collision_probability(h) == collision_probability(ref.results, h);
        }
        check(cp, "collision_probability exact");
        // sensor-noise TTC sweep: sigma = 0 is the reference's collision_probability at T * v;
        // a noisy sweep is monotone in T and shards (first_index) add up to the whole
        std::vector<double> ttc;
        for (int k = 0; k <= 20; ++k) ttc.push_back(1.0 + 0.25 * k);
        const std::vector<double> p0 = run.collision_probability_ttc_noise(ttc, 30.0, 0.0, 17);
        bool tn = true;
        for (std::size_t j = 0; j < ttc.size(); ++j) {
            tn = tn && p0[j] == collision_probability(ref.results, ttc[j] * 30.0);
        }
        const std::vector<double> pn = run.collision_probability_ttc_noise(ttc, 30.0, 0.25, 17);
        for (std::size_t j = 1; j < ttc.size(); ++j) tn = tn && pn[j] <= pn[j - 1];
        check(tn, "sensor-noise TTC sweep: sigma = 0 equals collision_probability, noisy sweep monotone");
        bool msh = true;
        for (double r : {0.5, 0.3, 0.28, 0.05, 0.01, 0.001}) {
            const double a = run.min_safe_headway(r), bref = min_safe_headway(ref.results, r);
            msh = msh && (a == bref || (std::isinf(a) && std::isinf(bref)));
        }
        check(msh, "min_safe_headway exact (incl. +inf past the horizon tail)");
        std::vector<double> grid = headway_grid(std::floor(want.min) - 5.0, 200.0, 1.0);
        const RiskCurve rc_ref = build_risk_curve(ref.results, grid, {0.05, 0.01, 0.5}, 30.0);
        const RiskCurve rc_gpu = run.build_risk_curve(grid, {0.05, 0.01, 0.5}, 30.0);
        bool same = rc_ref.probabilities == rc_gpu.probabilities &&
                    rc_ref.thresholds.size() == rc_gpu.thresholds.size();
        for (std::size_t k = 0; same && k < rc_ref.thresholds.size(); ++k) {
            same = rc_ref.thresholds[k].risk == rc_gpu.thresholds[k].risk &&
                   rc_ref.thresholds[k].headway_m == rc_gpu.thresholds[k].headway_m &&
                   rc_ref.thresholds[k].ttc_s == rc_gpu.thresholds[k].ttc_s;
        }
        check(same, "build_risk_curve exact");
        const std::vector<std::size_t> nv{1000, 5000, 12000, n};
        const auto cw = convergence_from_results(ref.results, nv, 12000);
        const auto cg = run.convergence(nv, 12000);
        bool conv = cw.size() == cg.size();
        for (std::size_t k = 0; conv && k < cw.size(); ++k) {
            conv = cw[k].n == cg[k].n && rel(cg[k].mean, cw[k].mean) && rel(cg[k].sd, cw[k].sd) &&
                   std::abs(cg[k].delta_mean - cw[k].delta_mean) <= 1e-10 &&
                   std::abs(cg[k].delta_sd - cw[k].delta_sd) <= 1e-10;
        }
        check(conv, "convergence rows (prefix mean/sd <= 1e-12 rel)");
    }

    // analysis.cpp:320-370 with the CUDA executor as the timed pipeline
    {
        FeasibilityOptions fo;
        fo.search_cap = 1u << 16;  // bounded for the test
        fo.timing_reps = 3;
        const TimingReport tr = max_samples_within_budget_cuda(UncertaintyModel{}, cfg, geo, phys,
                                                               TimingBudget{}, fo);
        check(tr.max_samples == fo.search_cap && tr.capped && tr.meets_convergence_threshold &&
                  tr.time_with_sampling_s < 0.53 && tr.sim_only_time_s <= tr.time_with_sampling_s,
              "feasibility search on run_cuda (2^16 cap reached inside 530 ms)");
    }

    // multi-device sharding path (one host thread + context per entry); on a
    // single-GPU box the same device twice exercises the threading/slicing
    {
        const SampleBatch b = batch_of(21, 30001, true);
        const ExecutionReport seq = run_parallel(b, cfg, geo, phys, 0);
        CudaExecOptions o;
        o.devices = {0, 0, 0};
        const ExecutionReport gpu = run_cuda(b, cfg, geo, phys, o);
        check(verify_consistency(seq, gpu).pass && gpu.worker_count == 3,
              "run_cuda with 3 shards (threads) bit-exact, worker_count = shards");
    }

    // MultiCudaRun: one context + host thread per device, outputs in HBM, the
    // whole batch's statistics merged over NCCL (ncclCommInitAll over the
    // devices; a 1-device communicator on a 1-GPU box) -- every field must
    // equal the reference's analysis functions (moments: summation bound)
    {
        int ndev = 0;
        bmc_device_count(&ndev);
        CudaExecOptions o;
        o.devices.clear();
        for (int dv = 0; dv < ndev && dv < 8; ++dv) o.devices.push_back(dv);
        UncertaintyModel m;
        m.seed = 5;
        m.friction = NormalSpec{0.45, 0.20};
        m.grade = NormalSpec{0.0, std::atan(0.06)};
        const std::size_t n = quick ? 50000 : 300000;
        const SampleBatch b = draw_batch(m, n);
        const ExecutionReport ref = run_parallel(b, cfg, geo, phys, 0);
        int ver = 0;
        check(bmc_nccl_available(&ver) == BMC_OK, "libnccl opened at run time (version " +
                                                      std::to_string(ver) + ")");
        for (bool model_driven : {true, false}) {
            const MultiCudaRun mr = model_driven ? MultiCudaRun::from_model(m, n, cfg, geo, phys, o)
                                                 : MultiCudaRun::from_batch(b, cfg, geo, phys, o);
            ExecutionReport got;
            got.results = mr.results(cfg.dt);
            check(verify_consistency(ref, got).pass,
                  std::string("MultiCudaRun::") + (model_driven ? "from_model" : "from_batch") +
                      " results bit-exact on " + std::to_string(mr.devices()) + " device(s)");
            CudaStatsRequest req;
            req.headways = headway_grid(0.0, 400.0, 2.5);
            req.risk_levels = {0.5, 0.05, 0.01, 0.001};
            req.summarize = true;
            req.bin_width = 0.37;
            const CudaStats st = mr.statistics(req);  // NCCL merge
            const DistributionSummary want = summarize(ref.results, 0.37);
            bool ok = st.n == n && st.horizon_count == want.horizon_count &&
                      st.summary.min == want.min && st.summary.max == want.max &&
                      st.summary.median == want.median &&
                      st.summary.histogram.counts == want.histogram.counts &&
                      std::abs(st.summary.mean - want.mean) <= 1e-12 * std::abs(want.mean) &&
                      std::abs(st.summary.sd - want.sd) <= 1e-12 * want.sd;
            for (std::size_t j = 0; j < req.headways.size(); ++j) {
                ok = ok && st.collision_probability[j] ==
                               collision_probability(ref.results, req.headways[j]);
            }
            for (std::size_t k = 0; k < req.risk_levels.size(); ++k) {
                const double w = min_safe_headway(ref.results, req.risk_levels[k]);
                ok = ok && (st.min_safe_headway[k] == w ||
                            (std::isinf(w) && std::isinf(st.min_safe_headway[k])));
            }
            check(ok, "MultiCudaRun::statistics over NCCL: counts/extrema/median/histogram/"
                      "collision probabilities/min_safe_headway exact, moments <= 1e-12 rel");
        }
    }

    // run_config.cpp:107-115 / cli.cpp:20-26 with the cuda branch
    {
        bool ok = executor_from_string_with_cuda("cuda") == kCudaExecutorKind &&
                  executor_from_string_with_cuda("parallel") == ExecutorKind::parallel &&
                  std::string(executor_name(kCudaExecutorKind)) == "cuda";
        try {
            executor_from_string_with_cuda("gpu");
            ok = false;
        } catch (const ConfigError& e) {
            ok = ok && e.field() == "execution.executor";
        }
        const SampleBatch b = batch_of(11, 2000);
        const ExecutionReport seq = run_executor(ExecutorKind::sequential, b, cfg, geo, phys);
        const ExecutionReport gpu = run_executor(executor_from_string_with_cuda("cuda"), b, cfg, geo, phys);
        check(ok && verify_consistency(seq, gpu).pass && gpu.executor == kCudaExecutorKind,
              "executor selection: \"cuda\" dispatches to run_cuda, \"gpu\" still rejected");
    }

    // backends.cpp:41-43: empty batch -> ConfigError with the field path
    {
        bool threw = false;
        try {
            run_cuda(SampleBatch{}, cfg, geo, phys);
        } catch (const ConfigError& e) {
            threw = std::string(e.what()) == "batch: must be non-empty";
        }
        check(threw, "empty batch throws ConfigError(batch)");
    }

    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
