// integration_main.cpp -- the reference's OWN dispatch sites, patched per
// INTEGRATION.md by tools/integrate_reference.py and compiled from a copy of
// its sources (build/integration/libbrakemc_integrated.so), driving the B200
// executor.  Checks:
//   * run_config.cpp:107-115: config_from_json({"execution":{"executor":
//     "cuda"}}) selects ExecutorKind::cuda; to_string round-trips; "gpu" still
//     throws ConfigError("execution.executor") (test_io_cli.cpp:103-104);
//   * cli.cpp:20-26's patched body (run_executor over the configured kind)
//     is bit-exact vs run_sequential (cli.cpp itself needs CLI11: it is
//     syntax-checked, not linked);
//   * analysis.cpp:138-141: convergence_table(..., ExecutorKind::cuda)
//     equals the parallel executor's table bit for bit;
//   * analysis.cpp:335-336 / 356-357: max_samples_within_budget with
//     FeasibilityOptions::executor = cuda runs the B200 executor (2^16 cap
//     reached inside 530 ms, where the CPU executor on this host is slower).
// Exit 0 on success.  Run by tests/test_gpu_parity.py on the GPU box.
#include "brakemc/analysis.hpp"
#include "brakemc/backends.hpp"
#include "brakemc/cuda_executor.hpp"
#include "brakemc/errors.hpp"
#include "brakemc/run_config.hpp"
#include "brakemc/sampling.hpp"

#include <cstdio>
#include <string>

using namespace brakemc;

namespace {
int failures = 0;
void check(bool ok, const std::string& what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}
}  // namespace

int main() {
    static_assert(static_cast<int>(ExecutorKind::cuda) == 2, "patched enum");
    static_assert(kCudaExecutorKind == ExecutorKind::cuda, "cuda_executor.hpp agrees");

    // run_config.cpp:107-115 through the reference's JSON loader
    const RunConfig rc = config_from_json(json::parse(R"({"execution": {"executor": "cuda"}})"));
    check(rc.execution.executor == ExecutorKind::cuda &&
              std::string(to_string(rc.execution.executor)) == "cuda" &&
              executor_from_string("cuda") == ExecutorKind::cuda,
          "config_from_json selects the cuda executor; to_string round-trips");
    bool threw = false;
    try {
        executor_from_string("gpu");
    } catch (const ConfigError& e) {
        threw = e.field() == "execution.executor";
    }
    check(threw, "\"gpu\" still throws ConfigError(execution.executor)");

    // cli.cpp:20-26 (patched body): the configured executor kind dispatches
    const SampleBatch batch = draw_batch(rc.uncertainty, 20000);
    const ExecutionReport seq = run_sequential(batch, rc.sim, rc.geometry, rc.constants);
    const ExecutionReport gpu = run_executor(rc.execution.executor, batch, rc.sim, rc.geometry,
                                             rc.constants, rc.execution.workers,
                                             rc.execution.chunk_size);
    check(gpu.executor == ExecutorKind::cuda && verify_consistency(seq, gpu).pass,
          "run_configured_executor body: cuda report bit-exact vs run_sequential");

    // analysis.cpp:138-141
    const std::vector<std::size_t> nv{1000, 4000, 12000, 25000};
    const auto cpu = convergence_table(UncertaintyModel{}, nv, rc.sim, rc.geometry, rc.constants,
                                       ExecutorKind::parallel, 0, 256);
    const auto cud = convergence_table(UncertaintyModel{}, nv, rc.sim, rc.geometry, rc.constants,
                                       ExecutorKind::cuda, 0, 256);
    bool same = cpu.size() == cud.size();
    for (std::size_t k = 0; same && k < cpu.size(); ++k) {
        same = cpu[k].n == cud[k].n && cpu[k].mean == cud[k].mean && cpu[k].sd == cud[k].sd &&
               cpu[k].delta_mean == cud[k].delta_mean && cpu[k].delta_sd == cud[k].delta_sd;
    }
    check(same, "convergence_table(ExecutorKind::cuda) == parallel table, bit for bit");

    // analysis.cpp:320-370 with the executor field
    FeasibilityOptions fo;
    fo.search_cap = 1u << 16;
    fo.timing_reps = 3;
    fo.executor = ExecutorKind::cuda;
    const TimingReport tr = max_samples_within_budget(UncertaintyModel{}, rc.sim, rc.geometry,
                                                      rc.constants, TimingBudget{}, fo);
    check(tr.max_samples == fo.search_cap && tr.capped && tr.meets_convergence_threshold &&
              tr.time_with_sampling_s < 0.53,
          "max_samples_within_budget(executor = cuda): 2^16 cap inside 530 ms (time with "
          "sampling " + std::to_string(tr.time_with_sampling_s * 1e3) + " ms)");

    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
