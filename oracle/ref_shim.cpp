// ref_shim.cpp -- extern "C" door into the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together
// with the reference's own hot-path sources, straight from where they lie
// (/root/reference/proj/src/{dynamics,integrator,sampling,backends,analysis}.cpp
// and tests/oracles.cpp), into oracle/_ref/libbrakemc_ref.so.  Nothing here
// re-implements the algorithm: every entry point forwards to the reference
// API so tests/ and bench.py (--impl reference, cpu_baseline) can call the
// reference through ctypes on identical inputs.
#include "brakemc/analysis.hpp"
#include "brakemc/backends.hpp"
#include "brakemc/errors.hpp"
#include "brakemc/integrator.hpp"
#include "brakemc/io.hpp"
#include "brakemc/sampling.hpp"
#include "oracles.hpp"

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

using namespace brakemc;

namespace {

thread_local std::string g_error;

static_assert(sizeof(ScenarioSample) == 40, "ScenarioSample layout");
static_assert(sizeof(RolloutResult) == 32, "RolloutResult layout");

struct World {
    SimConfig sim;
    VehicleGeometry geo;
    PhysicalConstants phys;
};

World world_from(const double* w) {
    World out;
    out.sim.dt = w[0];
    out.sim.t_max = w[1];
    out.sim.brake_cmd = w[2];
    out.geo.cg_height = w[3];
    out.geo.wheelbase = w[4];
    out.geo.actuator_tau = w[5];
    out.phys.gravity = w[6];
    out.phys.air_density = w[7];
    out.phys.frontal_area = w[8];
    return out;
}

std::vector<RolloutResult> results_from(const void* p, std::size_t n) {
    std::vector<RolloutResult> r(n);
    if (n) std::memcpy(r.data(), p, n * sizeof(RolloutResult));
    return r;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_error = e.what();
        return -1;
    } catch (const std::exception& e) {
        g_error = e.what();
        return -2;
    }
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

uint64_t ref_stream_word(uint64_t seed, uint64_t counter) { return stream_word(seed, counter); }

double ref_stream_uniform(uint64_t seed, uint64_t counter) {
    return stream_uniform(seed, counter);
}

double ref_standard_normal_at(uint64_t seed, uint64_t idx) {
    return standard_normal_at(seed, idx);
}

// mean/sd in the fixed stream order (initial_speed, friction, grade, mass, drag_coeff)
int ref_draw_batch(uint64_t seed, const double* mean, const double* sd, std::size_t n,
                   double* out_samples, uint64_t* clamp_count) {
    return guarded([&] {
        UncertaintyModel m;
        m.seed = seed;
        NormalSpec* specs[5] = {&m.initial_speed, &m.friction, &m.grade, &m.mass,
                                &m.drag_coeff};
        for (int j = 0; j < 5; ++j) {
            specs[j]->mean = mean[j];
            specs[j]->sd = sd[j];
        }
        const SampleBatch b = draw_batch(m, n);
        std::memcpy(out_samples, b.samples.data(), n * sizeof(ScenarioSample));
        *clamp_count = b.clamp_count;
    });
}

int ref_rollout_terms(const double* sample, const double* world, double* out5) {
    return guarded([&] {
        const World w = world_from(world);
        ScenarioSample s;
        std::memcpy(&s, sample, sizeof s);
        const RolloutTerms t = RolloutTerms::from(s, w.sim, w.geo, w.phys);
        out5[0] = t.brake_floor;
        out5[1] = t.drag_factor;
        out5[2] = t.grade_accel;
        out5[3] = t.brake_cmd;
        out5[4] = t.inv_tau;
    });
}

// executor: 0 = run_sequential, 1 = run_parallel(workers, chunk)
int ref_run(const double* samples, std::size_t n, const double* world, int executor,
            unsigned workers, std::size_t chunk, void* out_results, double* wall_time_s,
            unsigned* worker_count) {
    return guarded([&] {
        const World w = world_from(world);
        SampleBatch b;
        b.samples.resize(n);
        if (n) std::memcpy(b.samples.data(), samples, n * sizeof(ScenarioSample));
        const ExecutionReport rep =
            executor == 0 ? run_sequential(b, w.sim, w.geo, w.phys)
                          : run_parallel(b, w.sim, w.geo, w.phys, workers, chunk);
        std::memcpy(out_results, rep.results.data(), n * sizeof(RolloutResult));
        if (wall_time_s) *wall_time_s = rep.wall_time_s;
        if (worker_count) *worker_count = rep.worker_count;
    });
}

int ref_simulate_rollout(const double* sample, const double* world, void* out_result) {
    return guarded([&] {
        const World w = world_from(world);
        ScenarioSample s;
        std::memcpy(&s, sample, sizeof s);
        const RolloutResult r = simulate_rollout(s, w.sim, w.geo, w.phys);
        std::memcpy(out_result, &r, sizeof r);
    });
}

// out8: n, mean, sd, min, max, median, skewness, origin; flags: right_skewed
int ref_summarize(const void* results, std::size_t n, double bin_width, double* out8,
                  uint64_t* horizon_count, int* right_skewed, uint64_t* hist,
                  std::size_t hist_cap, uint64_t* bins) {
    return guarded([&] {
        const DistributionSummary s = summarize(results_from(results, n), bin_width);
        out8[0] = static_cast<double>(s.n);
        out8[1] = s.mean;
        out8[2] = s.sd;
        out8[3] = s.min;
        out8[4] = s.max;
        out8[5] = s.median;
        out8[6] = s.skewness;
        out8[7] = s.histogram.origin;
        *horizon_count = s.horizon_count;
        *right_skewed = s.right_skewed ? 1 : 0;
        *bins = s.histogram.counts.size();
        const std::size_t k = std::min(hist_cap, s.histogram.counts.size());
        for (std::size_t i = 0; i < k; ++i) hist[i] = s.histogram.counts[i];
    });
}

int ref_collision_probability(const void* results, std::size_t n, double headway,
                              double* out) {
    return guarded([&] { *out = collision_probability(results_from(results, n), headway); });
}

int ref_min_safe_headway(const void* results, std::size_t n, double risk, double* out) {
    return guarded([&] { *out = min_safe_headway(results_from(results, n), risk); });
}

// probs_out[m]; thr_out[3*k] = (risk, headway, ttc) by decreasing risk
int ref_build_risk_curve(const void* results, std::size_t n, const double* grid,
                         std::size_t m, const double* levels, std::size_t k,
                         double closing_speed, double* probs_out, double* thr_out) {
    return guarded([&] {
        const RiskCurve c = build_risk_curve(results_from(results, n),
                                             std::vector<double>(grid, grid + m),
                                             std::vector<double>(levels, levels + k),
                                             closing_speed);
        for (std::size_t i = 0; i < m; ++i) probs_out[i] = c.probabilities[i];
        for (std::size_t i = 0; i < c.thresholds.size(); ++i) {
            thr_out[3 * i] = c.thresholds[i].risk;
            thr_out[3 * i + 1] = c.thresholds[i].headway_m;
            thr_out[3 * i + 2] = c.thresholds[i].ttc_s;
        }
    });
}

long ref_headway_grid(double start, double stop, double step, double* out, std::size_t cap) {
    long count = -1;
    const int rc = guarded([&] {
        const std::vector<double> g = headway_grid(start, stop, step);
        count = static_cast<long>(g.size());
        for (std::size_t i = 0; i < g.size() && i < cap; ++i) out[i] = g[i];
    });
    return rc == 0 ? count : rc;
}

// rows_out[5*k] = n, mean, sd, delta_mean, delta_sd
int ref_convergence_from_results(const void* results, std::size_t n, const uint64_t* nvals,
                                 std::size_t k, std::size_t baseline_n, double* rows_out) {
    return guarded([&] {
        const std::vector<std::size_t> nv(nvals, nvals + k);
        const auto rows = convergence_from_results(results_from(results, n), nv, baseline_n);
        for (std::size_t i = 0; i < rows.size(); ++i) {
            rows_out[5 * i] = static_cast<double>(rows[i].n);
            rows_out[5 * i + 1] = rows[i].mean;
            rows_out[5 * i + 2] = rows[i].sd;
            rows_out[5 * i + 3] = rows[i].delta_mean;
            rows_out[5 * i + 4] = rows[i].delta_sd;
        }
    });
}

// out: max_abs_deviation, first_mismatch, bitwise_equal, pass
int ref_verify_consistency(const void* a, const void* b, std::size_t n, double* max_dev,
                           uint64_t* first_mismatch, int* bitwise_equal, int* pass) {
    return guarded([&] {
        ExecutionReport ra, rb;
        ra.results = results_from(a, n);
        rb.results = results_from(b, n);
        const ConsistencyVerdict v = verify_consistency(ra, rb);
        *max_dev = v.max_abs_deviation;
        *first_mismatch = v.first_mismatch;
        *bitwise_equal = v.bitwise_equal ? 1 : 0;
        *pass = v.pass ? 1 : 0;
    });
}

// io.cpp:17-31 -- results.csv text, written verbatim to `path`
int ref_write_results_csv(const void* results, std::size_t n, const char* path) {
    return guarded([&] { write_text_file(path, results_csv(results_from(results, n))); });
}

// io.cpp:94-123 + cli.cpp:96-100 (steps rebuilt from t_stop / dt)
int ref_read_results_csv(const char* path, double dt, void* out, std::size_t cap,
                         std::size_t* n_out) {
    return guarded([&] {
        std::vector<RolloutResult> r = parse_results_csv(read_text_file(path));
        for (RolloutResult& x : r) x.steps = std::llround(x.stop_time / dt);
        *n_out = r.size();
        if (r.size() <= cap && !r.empty()) std::memcpy(out, r.data(), r.size() * sizeof(RolloutResult));
    });
}

// tests/oracles.cpp:44-54 -- the independent fine-step integrator
double ref_oracle_stopping_distance(const double* sample, const double* world, double dt,
                                    double t_limit) {
    const World w = world_from(world);
    oracle::Params p;
    p.v0 = sample[0];
    p.mu = sample[1];
    p.theta = sample[2];
    p.mass = sample[3];
    p.cd = sample[4];
    p.gravity = w.phys.gravity;
    p.rho = w.phys.air_density;
    p.frontal_area = w.phys.frontal_area;
    p.cg_height = w.geo.cg_height;
    p.wheelbase = w.geo.wheelbase;
    p.tau = w.geo.actuator_tau;
    p.brake_cmd = w.sim.brake_cmd;
    return oracle::stopping_distance(p, dt, t_limit);
}

} // extern "C"
