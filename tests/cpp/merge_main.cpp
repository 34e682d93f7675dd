// merge_main.cpp -- C++ CPU test of the statistics merge (no GPU needed).
//
// The fused statistics stage's orchestration (bmc_stats_pipeline.h) runs on
// the host twin (stats_host.cpp) for worlds 1, 2 and 3: one std::thread per
// rank, each over its contiguous shard, merging through an in-process
// FakeCollective that implements brakemc::Collective (include/brakemc/
// cuda_multi.hpp) over host memory -- the same interface the NCCL backend
// implements for devices.  Data and answers come from the UNMODIFIED
// reference (oracle/_ref: draw_batch, run_parallel, summarize,
// collision_probability, min_safe_headway).
//
// Pass: every rank of every world returns the single-rank answer bit for bit
// (exact sums, integer counts), and that answer equals the reference's
// counts / extrema / median / histogram / collision probabilities /
// min_safe_headway exactly, mean/sd/skewness within the reference's own
// summation error.  Also with a tiny candidate capacity (merged exact
// fallback).  Exit status 0 on success.
#include "brakemc/analysis.hpp"
#include "brakemc/backends.hpp"
#include "brakemc/cuda_multi.hpp"
#include "brakemc/sampling.hpp"

#include <barrier>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <thread>
#include <vector>

extern "C" int bmch_stats_run(const double* d, const uint8_t* hz, size_t n, const bmc_stats_req* req,
                              uint64_t cand_cap, const bmc_merge* merge, bmc_stats* out, char* err,
                              size_t errcap);

namespace {

using namespace brakemc;

// In-process ranks over host memory: deposit pointers, meet, each rank
// reduces (or gathers) every rank's words privately, meet, write back.
class FakeCollective : public Collective {
public:
    explicit FakeCollective(int world)
        : world_(world), bar_(world), bufs_(world), sends_(world), calls_(0) {}
    int world() const override { return world_; }
    int allreduce_u64(int rank, std::uint64_t* buf, std::size_t count, int op, void*) override {
        bufs_[rank] = buf;
        if (rank == 0) ++calls_;
        bar_.arrive_and_wait();
        std::vector<std::uint64_t> acc(bufs_[0], bufs_[0] + count);
        for (int r = 1; r < world_; ++r) {
            for (std::size_t i = 0; i < count; ++i) {
                const std::uint64_t v = bufs_[r][i];
                acc[i] = op == BMC_MERGE_SUM ? acc[i] + v
                         : op == BMC_MERGE_MIN ? std::min(acc[i], v) : std::max(acc[i], v);
            }
        }
        bar_.arrive_and_wait();
        std::memcpy(buf, acc.data(), count * 8);
        bar_.arrive_and_wait();
        return 0;
    }
    int allgather_u64(int rank, const std::uint64_t* send, std::uint64_t* recv, std::size_t count,
                      void*) override {
        sends_[rank] = send;
        if (rank == 0) ++calls_;
        bar_.arrive_and_wait();
        for (int r = 0; r < world_; ++r) std::memcpy(recv + r * count, sends_[r], count * 8);
        bar_.arrive_and_wait();
        return 0;
    }
    int calls() const { return calls_; }

private:
    int world_;
    std::barrier<> bar_;
    std::vector<std::uint64_t*> bufs_;
    std::vector<const std::uint64_t*> sends_;
    int calls_;
};

struct Answer {
    bmc_stats s{};
    std::vector<std::uint64_t> exceed, hist;
    std::vector<double> msh;
    bool operator==(const Answer& o) const {
        return s.n == o.s.n && s.horizon_count == o.s.horizon_count &&
               std::memcmp(&s.summary, &o.s.summary, sizeof s.summary) == 0 && exceed == o.exceed &&
               hist == o.hist &&
               std::memcmp(msh.data(), o.msh.data(), msh.size() * 8) == 0;
    }
};

int failures = 0;
#define CHECK(c, ...)                                    \
    do {                                                 \
        if (!(c)) {                                      \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                    \
            std::printf("\n");                           \
            ++failures;                                  \
        }                                                \
    } while (0)

Answer run_world(const std::vector<RolloutResult>& res, const bmc_stats_req& req, int world,
                 uint64_t cand_cap, int* calls) {
    const std::size_t n = res.size();
    std::vector<double> d(n);
    std::vector<uint8_t> hz(n);
    for (std::size_t i = 0; i < n; ++i) {
        d[i] = res[i].stop_distance;
        hz[i] = res[i].hit_horizon ? 1 : 0;
    }
    FakeCollective coll(world);
    std::vector<Answer> ans(world);
    std::vector<int> rcs(world, 0);
    auto rank_main = [&](int r) {
        const std::size_t b = n * r / world, e = n * (r + 1) / world;
        Answer& a = ans[r];
        a.exceed.resize(req.n_headways);
        a.msh.resize(req.n_risk);
        a.hist.assign(1 << 16, 0);
        a.s.exceed = a.exceed.data();
        a.s.min_safe_headway = a.msh.data();
        a.s.histogram = a.hist.data();
        a.s.histogram_cap = a.hist.size();
        const bmc_merge m = coll.merge(r);
        char err[256] = {0};
        rcs[r] = bmch_stats_run(d.data() + b, hz.data() + b, e - b, &req, cand_cap,
                                world > 1 ? &m : nullptr, &a.s, err, sizeof err);
        if (rcs[r]) std::printf("rank %d: %s\n", r, err);
        a.hist.resize(a.s.summary.bins);
    };
    std::vector<std::thread> ts;
    for (int r = 0; r < world; ++r) ts.emplace_back(rank_main, r);
    for (auto& t : ts) t.join();
    for (int r = 0; r < world; ++r) CHECK(rcs[r] == 0, "world %d rank %d rc %d", world, r, rcs[r]);
    for (int r = 1; r < world; ++r) CHECK(ans[r] == ans[0], "world %d: rank %d differs from rank 0", world, r);
    if (calls) *calls = coll.calls();
    return ans[0];
}

void check_reference(const std::vector<RolloutResult>& res, const Answer& a,
                     const std::vector<double>& grid, const std::vector<double>& risks, double bw) {
    const DistributionSummary w = summarize(res, bw);
    const bmc_summary& g = a.s.summary;
    CHECK(g.n == w.n && g.horizon_count == w.horizon_count, "counts");
    CHECK(g.min == w.min && g.max == w.max && g.median == w.median, "extrema/median");
    CHECK(g.origin == w.histogram.origin && g.bins == w.histogram.counts.size(), "hist shape");
    CHECK(std::equal(a.hist.begin(), a.hist.end(), w.histogram.counts.begin()), "hist counts");
    double abs_sum = 0.0;
    for (const auto& r : res) abs_sum += std::fabs(r.stop_distance);
    const double eps = std::ldexp(1.0, -52);
    const double bound = (res.size() - 1) * eps * abs_sum / res.size() + std::fabs(w.mean) * eps;
    CHECK(std::fabs(g.mean - w.mean) <= bound, "mean %.17g vs %.17g", g.mean, w.mean);
    CHECK(std::fabs(g.sd - w.sd) <= 1e-12 * w.sd, "sd");
    CHECK(std::fabs(g.skewness - w.skewness) <= 1e-9 * std::fabs(w.skewness) + 1e-12, "skewness");
    for (std::size_t j = 0; j < grid.size(); ++j) {
        const double p = static_cast<double>(a.exceed[j]) / static_cast<double>(res.size());
        CHECK(p == collision_probability(res, grid[j]), "collision_probability(%g)", grid[j]);
    }
    for (std::size_t k = 0; k < risks.size(); ++k) {
        CHECK(a.msh[k] == min_safe_headway(res, risks[k]), "min_safe_headway(%g)", risks[k]);
    }
}

}  // namespace

int main() {
    const SimConfig config;
    const VehicleGeometry geometry;
    const PhysicalConstants constants;
    UncertaintyModel mixed;
    mixed.seed = 13;
    mixed.friction = NormalSpec{0.45, 0.20};
    mixed.grade = NormalSpec{0.0, std::atan(0.06)};
    for (const auto& [model, n] : {std::pair{UncertaintyModel{}, std::size_t{12000}},
                                   std::pair{mixed, std::size_t{7001}}}) {
        const SampleBatch batch = draw_batch(model, n);
        const auto res = run_parallel(batch, config, geometry, constants, 0).results;
        double lo = 1e300, hi = -1e300;
        for (const auto& r : res) {
            lo = std::min(lo, r.stop_distance);
            hi = std::max(hi, r.stop_distance);
        }
        const std::vector<double> grid = headway_grid(std::floor(lo) - 5.0, std::ceil(hi) + 5.0, 1.0);
        const std::vector<double> risks{0.05, 0.01, 0.001, 0.5};
        for (double bw : {2.0, 0.37}) {
            bmc_stats_req req{};
            req.headways = grid.data();
            req.n_headways = grid.size();
            req.risk_levels = risks.data();
            req.n_risk = risks.size();
            req.summarize = 1;
            req.bin_width = bw;
            const Answer one = run_world(res, req, 1, 0, nullptr);
            check_reference(res, one, grid, risks, bw);
            for (int world : {2, 3}) {
                for (uint64_t cap : {uint64_t{0}, uint64_t{1}}) {
                    int calls = 0;
                    const Answer many = run_world(res, req, world, cap, &calls);
                    CHECK(many == one, "model seed %llu bw %g world %d cap %llu differs from world 1",
                          static_cast<unsigned long long>(model.seed), bw, world,
                          static_cast<unsigned long long>(cap));
                    CHECK(calls >= 5, "world %d: %d merge calls", world, calls);
                    if (cap) CHECK(many.s.fallbacks > 0, "cap %llu took no fallback",
                                   static_cast<unsigned long long>(cap));
                }
            }
        }
    }
    std::printf("%s: statistics merge over FakeCollective, worlds 1/2/3 (%d failures)\n",
                failures ? "FAIL" : "PASS", failures);
    return failures ? 1 : 0;
}
