// bmc_graph.cpp -- real-time mode (C2): one decision batch of fixed size n
// captured once as a CUDA graph {H2D terms -> predict/bin -> rollout -> D2H}
// and replayed per decision, so a decision costs one cudaGraphLaunch plus the
// host staging / unpack (the reference's 530 ms Monte Carlo budget,
// analysis.hpp:108-116).  The graph owns every buffer it captured (terms,
// outputs, scratch, actuator tables), so later context calls cannot move
// them.  g++ -ffp-contract=off.
#include "bmc_ctx.h"

#include <atomic>
#include <chrono>
#include <cstring>
#include <memory>

struct bmc_graph {
    bmc_ctx* ctx = nullptr;
    size_t n = 0;
    bmc_world world{};
    bmc::WorldDerived d{};
    bmc::Plan plan;
    bmc::Scratch sc;
    bmc::DevBuf table, coarse, d_terms, d_out, steps_total;
    bmc::PinBuf h_terms, h_out;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t done = nullptr;
    unsigned threads = 1;
    uint32_t launches = 0;
};

namespace {

void release(bmc_graph* g) {
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    if (g->done) cudaEventDestroy(g->done);
    g->sc.release();
    for (bmc::DevBuf* b : {&g->table, &g->coarse, &g->d_terms, &g->d_out, &g->steps_total}) b->release();
    g->h_terms.release();
    g->h_out.release();
}

int graph_fail(bmc_graph* g, int code, const std::string& msg) {
    return bmc::fail(g ? g->ctx : nullptr, code, msg);
}

#define BMC_GK(g, expr)                                                                  \
    do {                                                                                 \
        const cudaError_t e_ = (expr);                                                   \
        if (e_ != cudaSuccess)                                                           \
            return graph_fail((g), BMC_E_CUDA,                                           \
                              std::string(#expr) + ": " + cudaGetErrorString(e_));       \
    } while (0)

// Replay + unpack; the caller has filled g->h_terms.
int replay(bmc_graph* g, bmc_result* out, bmc_run_info* info,
           std::chrono::steady_clock::time_point t0) {
    bmc_ctx* ctx = g->ctx;
    BMC_GK(g, cudaGraphLaunch(g->exec, ctx->stream));
    BMC_GK(g, cudaEventRecord(g->done, ctx->stream));
    BMC_GK(g, cudaEventSynchronize(g->done));
    const size_t n = g->n;
    const double* dd = g->h_out.as<double>();
    const int32_t* st = reinterpret_cast<const int32_t*>(g->h_out.as<char>() + n * 8);
    const uint8_t* hz = reinterpret_cast<const uint8_t*>(g->h_out.as<char>() + n * 12);
    const double dt = g->d.dt;
    bmc::host_pool().parallel_for(
        n,
        [&](size_t b, size_t e) {
            for (size_t i = b; i < e; ++i) {
                bmc_result r;
                std::memset(&r, 0, sizeof r);
                r.stop_distance = dd[i];
                r.stop_time = static_cast<double>(st[i]) * dt;
                r.steps = st[i];
                r.hit_horizon = hz[i];
                out[i] = r;
            }
        },
        g->threads);
    if (info) {
        std::memset(info, 0, sizeof *info);
        info->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        info->h2d_bytes = n * 32;
        info->d2h_bytes = n * 13;
        info->launches = g->launches;
        info->chunks = 1;
        unsigned long long steps = 0;
        BMC_GK(g, cudaMemcpy(&steps, g->steps_total.p, sizeof steps, cudaMemcpyDeviceToHost));
        info->total_steps = steps;
    }
    return BMC_OK;
}

}  // namespace

extern "C" {

int bmc_cuda_graph_create(bmc_ctx* ctx, size_t n, const bmc_world* world,
                          const bmc_run_opts* opts, bmc_graph** out) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (!out || !world) return bmc::fail(ctx, BMC_E_CONFIG, "bmc_cuda_graph_create: null argument");
    *out = nullptr;
    if (n == 0) return bmc::fail(ctx, BMC_E_CONFIG, "batch: must be non-empty");
    auto g = std::make_unique<bmc_graph>();
    g->ctx = ctx;
    g->n = n;
    g->world = *world;
    std::string err;
    if ((rc = bmc::derive_world(*world, &g->d, &err)) != BMC_OK) return bmc::fail(ctx, rc, err);
    const bmc_run_opts o = opts ? *opts : bmc_run_opts{};
    g->threads = bmc::resolve_threads(o.host_threads);
    if ((rc = bmc::make_plan(ctx, g->d, o, n, &g->plan)) != BMC_OK) return rc;
    // private copies of the world-dependent tables
    if (g->plan.table_len > 0 && g->plan.table) {
        const size_t tb = static_cast<size_t>(g->plan.table_len) * sizeof(bmc::StageA);
        BMC_CK(ctx, g->table.reserve(tb));
        BMC_CK(ctx, cudaMemcpy(g->table.p, g->plan.table, tb, cudaMemcpyDeviceToDevice));
        g->plan.table = g->table.as<bmc::StageA>();
    }
    if (g->plan.coarse_len > 0) {
        const size_t cb = static_cast<size_t>(g->plan.coarse_len) * sizeof(float);
        BMC_CK(ctx, g->coarse.reserve(cb));
        BMC_CK(ctx, cudaMemcpy(g->coarse.p, g->plan.coarse, cb, cudaMemcpyDeviceToDevice));
        g->plan.coarse = g->coarse.as<float>();
    }
    BMC_CK(ctx, g->h_terms.reserve(n * 32));
    BMC_CK(ctx, g->h_out.reserve(n * 13));
    BMC_CK(ctx, g->d_terms.reserve(n * 32));
    BMC_CK(ctx, g->d_out.reserve(n * 13));
    BMC_CK(ctx, g->steps_total.reserve(sizeof(unsigned long long)));
    if ((rc = bmc::reserve_scratch(ctx, g->sc, g->plan, n)) != BMC_OK) return rc;
    BMC_CK(ctx, cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming));
    BMC_CK(ctx, cudaStreamSynchronize(ctx->stream));

    const double* dv0 = g->d_terms.as<double>();
    const bmc_terms terms{dv0, dv0 + n, dv0 + 2 * n, dv0 + 3 * n};
    char* dout = g->d_out.as<char>();
    const bmc_outputs outs{reinterpret_cast<double*>(dout), reinterpret_cast<int32_t*>(dout + n * 8),
                           reinterpret_cast<uint8_t*>(dout + n * 12)};
    cudaStream_t s = ctx->stream;
    BMC_CK(ctx, cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    uint32_t launches = 0;
    bool ok = cudaMemcpyAsync(g->d_terms.p, g->h_terms.p, n * 32, cudaMemcpyHostToDevice, s) == cudaSuccess &&
              cudaMemsetAsync(g->steps_total.p, 0, sizeof(unsigned long long), s) == cudaSuccess;
    if (ok) {
        ok = bmc::enqueue_rollout(ctx, g->plan, g->sc, terms, n, outs,
                                  g->steps_total.as<unsigned long long>(), s, nullptr,
                                  &launches) == BMC_OK;
    }
    if (ok) ok = cudaMemcpyAsync(g->h_out.p, g->d_out.p, n * 13, cudaMemcpyDeviceToHost, s) == cudaSuccess;
    const cudaError_t ec = cudaStreamEndCapture(s, &g->graph);
    if (!ok || ec != cudaSuccess) {
        const std::string why = ctx->err.empty() ? cudaGetErrorString(ec) : ctx->err;
        release(g.get());
        return bmc::fail(ctx, BMC_E_CUDA, "graph capture failed: " + why);
    }
    const cudaError_t ei = cudaGraphInstantiate(&g->exec, g->graph, 0);
    if (ei != cudaSuccess) {
        release(g.get());
        return bmc::fail(ctx, BMC_E_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ei));
    }
    g->launches = launches;
    *out = g.release();
    return BMC_OK;
}

int bmc_cuda_graph_run(bmc_graph* g, const bmc_sample* samples, bmc_result* out,
                       bmc_run_info* info) {
    if (!g || !samples || !out) return bmc::fail(g ? g->ctx : nullptr, BMC_E_CONFIG, "bmc_cuda_graph_run: null argument");
    int rc = bmc::prepare(g->ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g->ctx->mu);
    const auto t0 = std::chrono::steady_clock::now();
    const size_t n = g->n;
    double* h = g->h_terms.as<double>();
    std::atomic<int> status{BMC_OK};
    bmc::host_pool().parallel_for(
        n,
        [&](size_t b, size_t e) {
            const int r = bmc::stage_terms_serial(samples + b, e - b, g->world, h + b, h + n + b,
                                                  h + 2 * n + b, h + 3 * n + b);
            if (r != BMC_OK) status = r;
        },
        g->threads);
    if (status != BMC_OK) return bmc::fail(g->ctx, BMC_E_DOMAIN, "friction_limit: weight-transfer denominator <= 0");
    return replay(g, out, info, t0);
}

int bmc_cuda_graph_run_model(bmc_graph* g, const bmc_model* model, uint64_t first, bmc_result* out,
                             uint64_t* clamp_count, bmc_run_info* info) {
    if (!g || !model || !out) return bmc::fail(g ? g->ctx : nullptr, BMC_E_CONFIG, "bmc_cuda_graph_run_model: null argument");
    int rc = bmc::prepare(g->ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g->ctx->mu);
    const auto t0 = std::chrono::steady_clock::now();
    const size_t n = g->n;
    double* h = g->h_terms.as<double>();
    std::atomic<int> status{BMC_OK};
    std::atomic<uint64_t> clamps{0};
    bmc::host_pool().parallel_for(
        n,
        [&](size_t b, size_t e) {
            uint64_t c = 0;
            const int r = bmc::draw_terms_serial(*model, first + b, e - b, g->world, h + b, h + n + b,
                                                 h + 2 * n + b, h + 3 * n + b, &c);
            clamps += c;
            if (r != BMC_OK) status = r;
        },
        g->threads);
    if (status != BMC_OK) return bmc::fail(g->ctx, BMC_E_DOMAIN, "friction_limit: weight-transfer denominator <= 0");
    if (clamp_count) *clamp_count = clamps.load();
    return replay(g, out, info, t0);
}

void bmc_cuda_graph_destroy(bmc_graph* g) {
    if (!g) return;
    cudaSetDevice(g->ctx->device);
    cudaStreamSynchronize(g->ctx->stream);
    release(g);
    delete g;
}

}  // extern "C"
