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
    // Model-driven decisions on the device sampler: a second graph
    // {H2D draw params, draw kernel, rollout, D2H outputs + draw counters},
    // captured on the first bmc_cuda_graph_run_model call.
    int sampler = 0;  // bmc_run_opts.sampler
    cudaGraph_t mgraph = nullptr;
    cudaGraphExec_t mexec = nullptr;
    bmc::DevBuf d_dyn, d_ctr;
    bmc::PinBuf h_dyn, h_ctr;
    uint32_t mlaunches = 0;
    // Optional statistics stage captured after the rollout (pass 1 fused in
    // its epilogue); its read-back words land in a pinned mirror per replay.
    bmc_stats_stage* st = nullptr;
    bmc::PinBuf h_stats;
    bool replayed = false;
};

namespace {

void release(bmc_graph* g) {
    if (g->st) bmc_stats_destroy(g->st);
    g->st = nullptr;
    g->h_stats.release();
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    if (g->mexec) cudaGraphExecDestroy(g->mexec);
    if (g->mgraph) cudaGraphDestroy(g->mgraph);
    for (bmc::DevBuf* b : {&g->d_dyn, &g->d_ctr}) b->release();
    g->h_dyn.release();
    g->h_ctr.release();
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

// Replay + unpack; the caller has filled g->h_terms (or g->h_dyn).
int replay(bmc_graph* g, bmc_result* out, bmc_run_info* info,
           std::chrono::steady_clock::time_point t0, bool model_graph = false) {
    bmc_ctx* ctx = g->ctx;
    BMC_GK(g, cudaGraphLaunch(model_graph ? g->mexec : g->exec, ctx->stream));
    BMC_GK(g, cudaEventRecord(g->done, ctx->stream));
    BMC_GK(g, cudaEventSynchronize(g->done));
    g->replayed = true;
    const size_t n = g->n;
    const double* dd = g->h_out.as<double>();
    const int32_t* st = reinterpret_cast<const int32_t*>(g->h_out.as<char>() + n * 8);
    const uint8_t* hz = reinterpret_cast<const uint8_t*>(g->h_out.as<char>() + n * 12);
    const double dt = g->d.dt;
    bmc::ctx_pool(g->ctx, g->threads).parallel_for(
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
        info->h2d_bytes = model_graph ? sizeof(bmc::DrawDyn) : n * 32;
        info->d2h_bytes = n * 13 + (model_graph ? 16 : 0);
        info->launches = model_graph ? g->mlaunches : g->launches;
        info->chunks = 1;
        unsigned long long steps = 0;
        BMC_GK(g, cudaMemcpy(&steps, g->steps_total.p, sizeof steps, cudaMemcpyDeviceToHost));
        info->total_steps = steps;
    }
    return BMC_OK;
}

// Inside a capture: the rollout (pass 1 fused when the graph has a stage),
// the stage's device passes, and the D2H of outputs + statistics words.
bool capture_rollout_tail(bmc_graph* g, const bmc_terms& terms, const bmc_outputs& outs,
                          cudaStream_t s, uint32_t* launches) {
    bmc_ctx* ctx = g->ctx;
    const size_t n = g->n;
    bmc::P1Args p1{};
    if (g->st) {
        bmc::stats_p1_args(g->st, &p1);
        if (bmc::stats_begin_enqueue(g->st, s) != BMC_OK) return false;
    }
    if (bmc::enqueue_rollout(ctx, g->plan, g->sc, terms, n, outs, g->steps_total.as<unsigned long long>(),
                             s, nullptr, launches, g->st ? &p1 : nullptr,
                             bmc::direct_outputs_for(n)) != BMC_OK) {
        return false;
    }
    if (g->st) {
        const uint32_t before = bmc::stats_launches(g->st);
        if (bmc::stats_enqueue_device(g->st, outs.stop_distance, outs.hit_horizon, n, s) != BMC_OK) return false;
        *launches += bmc::stats_launches(g->st) - before;
    }
    if (cudaMemcpyAsync(g->h_out.p, g->d_out.p, n * 13, cudaMemcpyDeviceToHost, s) != cudaSuccess) return false;
    if (g->st && bmc::stats_enqueue_readback(g->st, g->h_stats.as<uint64_t>(), s) != BMC_OK) return false;
    return true;
}

// Capture the device-sampler decision graph (lazily, first model decision).
int capture_model_graph(bmc_graph* g) {
    bmc_ctx* ctx = g->ctx;
    const size_t n = g->n;
    BMC_CK(ctx, g->d_dyn.reserve(sizeof(bmc::DrawDyn)));
    BMC_CK(ctx, g->h_dyn.reserve(sizeof(bmc::DrawDyn)));
    BMC_CK(ctx, g->d_ctr.reserve(16));
    BMC_CK(ctx, g->h_ctr.reserve(16));
    BMC_CK(ctx, cudaStreamSynchronize(ctx->stream));
    bmc_model zero{};
    bmc::DrawArgs da = bmc::draw_args(zero, 0, n, g->world);
    double* dv0 = g->d_terms.as<double>();
    da.v0 = dv0;
    da.brake_floor = dv0 + n;
    da.drag = dv0 + 2 * n;
    da.grade = dv0 + 3 * n;
    da.clamps = g->d_ctr.as<unsigned long long>();
    da.flags = reinterpret_cast<unsigned int*>(g->d_ctr.as<char>() + 8);
    da.dyn = g->d_dyn.as<bmc::DrawDyn>();
    const bmc_terms terms{dv0, dv0 + n, dv0 + 2 * n, dv0 + 3 * n};
    char* dout = g->d_out.as<char>();
    const bmc_outputs outs{reinterpret_cast<double*>(dout), reinterpret_cast<int32_t*>(dout + n * 8),
                           reinterpret_cast<uint8_t*>(dout + n * 12)};
    cudaStream_t s = ctx->stream;
    BMC_CK(ctx, cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    uint32_t launches = 1;
    bool ok = cudaMemcpyAsync(g->d_dyn.p, g->h_dyn.p, sizeof(bmc::DrawDyn), cudaMemcpyHostToDevice, s) == cudaSuccess &&
              cudaMemsetAsync(g->d_ctr.p, 0, 16, s) == cudaSuccess &&
              cudaMemsetAsync(g->steps_total.p, 0, sizeof(unsigned long long), s) == cudaSuccess &&
              bmc::launch_draw_terms(da, ctx->sms, s) == cudaSuccess;
    if (ok) ok = capture_rollout_tail(g, terms, outs, s, &launches);
    if (ok) ok = cudaMemcpyAsync(g->h_ctr.p, g->d_ctr.p, 16, cudaMemcpyDeviceToHost, s) == cudaSuccess;
    const cudaError_t ec = cudaStreamEndCapture(s, &g->mgraph);
    if (!ok || ec != cudaSuccess) {
        const std::string why = ctx->err.empty() ? cudaGetErrorString(ec) : ctx->err;
        if (g->mgraph) cudaGraphDestroy(g->mgraph);
        g->mgraph = nullptr;
        return bmc::fail(ctx, BMC_E_CUDA, "graph capture failed: " + why);
    }
    const cudaError_t ei = cudaGraphInstantiate(&g->mexec, g->mgraph, 0);
    if (ei != cudaSuccess) {
        g->mexec = nullptr;
        return bmc::fail(ctx, BMC_E_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ei));
    }
    g->mlaunches = launches;
    return BMC_OK;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

int graph_create(bmc_ctx* ctx, size_t n, const bmc_world* world, const bmc_run_opts* opts,
                 const bmc_stats_req* req, bmc_graph** out) {
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
    g->sampler = o.sampler;
    if ((rc = bmc::make_plan(ctx, g->d, o, n, &g->plan)) != BMC_OK) return rc;
    if (req) {
        if ((rc = bmc::stats_stage_create(ctx, req, n, &g->st)) != BMC_OK) return rc;
        bmc::P1Args p1{};
        if (!bmc::stats_p1_args(g->st, &p1)) {
            release(g.get());
            return bmc::fail(ctx, BMC_E_RANGE, "risk.headways: at most 4096 in a decision graph");
        }
        bmc::fit_stats_plan(&g->plan, p1);
        BMC_CK(ctx, g->h_stats.reserve(bmc::stats_mirror_words(g->st) * 8));
    }
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
    if ((rc = bmc::reserve_scratch(ctx, g->sc, g->plan, n, bmc::direct_outputs_for(n))) != BMC_OK) return rc;
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
    if (ok) ok = capture_rollout_tail(g.get(), terms, outs, s, &launches);
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

}  // namespace

extern "C" {

int bmc_cuda_graph_create(bmc_ctx* ctx, size_t n, const bmc_world* world,
                          const bmc_run_opts* opts, bmc_graph** out) {
    try {
        return graph_create(ctx, n, world, opts, nullptr, out);
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_graph_create_stats(bmc_ctx* ctx, size_t n, const bmc_world* world,
                                const bmc_run_opts* opts, const bmc_stats_req* req,
                                bmc_graph** out) {
    try {
        if (!req) return bmc::fail(ctx, BMC_E_CONFIG, "bmc_cuda_graph_create_stats: null request");
        return graph_create(ctx, n, world, opts, req, out);
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_graph_stats(bmc_graph* g, bmc_stats* out) {
    try {
        if (!g || !out) return bmc::fail(g ? g->ctx : nullptr, BMC_E_CONFIG, "bmc_cuda_graph_stats: null argument");
        if (!g->st) return bmc::fail(g->ctx, BMC_E_CONFIG, "bmc_cuda_graph_stats: graph has no statistics stage");
        if (!g->replayed) return bmc::fail(g->ctx, BMC_E_CONFIG, "bmc_cuda_graph_stats: no decision ran yet");
        int rc = bmc::prepare(g->ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(g->ctx->mu);
        const char* dout = g->d_out.as<char>();
        rc = bmc::stats_compose_mirror(g->st, g->h_stats.as<uint64_t>(), reinterpret_cast<const double*>(dout),
                                       reinterpret_cast<const uint8_t*>(dout + g->n * 12), g->n, out);
        if (rc == BMC_OK) out->launches = g->launches;
        return rc;
    } catch (...) {
        return bmc::abi_exception();
    }
}

int bmc_cuda_graph_run(bmc_graph* g, const bmc_sample* samples, bmc_result* out,
                       bmc_run_info* info) {
    try {
        if (!g || !samples || !out) return bmc::fail(g ? g->ctx : nullptr, BMC_E_CONFIG, "bmc_cuda_graph_run: null argument");
        int rc = bmc::prepare(g->ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(g->ctx->mu);
        const auto t0 = std::chrono::steady_clock::now();
        const size_t n = g->n;
        double* h = g->h_terms.as<double>();
        std::atomic<int> status{BMC_OK};
        bmc::ctx_pool(g->ctx, g->threads).parallel_for(
            n,
            [&](size_t b, size_t e) {
                const int r = bmc::stage_terms_serial(samples + b, e - b, g->world, h + b, h + n + b,
                                                      h + 2 * n + b, h + 3 * n + b);
                if (r != BMC_OK) status = r;
            },
            g->threads);
        if (status != BMC_OK) return bmc::fail(g->ctx, BMC_E_DOMAIN, "friction_limit: weight-transfer denominator <= 0");
        return replay(g, out, info, t0);
    } catch (...) {
        return bmc::abi_exception();
    }
}

int bmc_cuda_graph_run_model(bmc_graph* g, const bmc_model* model, uint64_t first, bmc_result* out,
                             uint64_t* clamp_count, bmc_run_info* info) {
    try {
        if (!g || !model || !out) return bmc::fail(g ? g->ctx : nullptr, BMC_E_CONFIG, "bmc_cuda_graph_run_model: null argument");
        int rc = bmc::prepare(g->ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(g->ctx->mu);
        const auto t0 = std::chrono::steady_clock::now();
        bmc_run_opts o{};
        o.sampler = g->sampler;
        bool dev = false;
        if ((rc = bmc::use_device_sampler(g->ctx, o, &dev)) != BMC_OK) return rc;
        if (dev) {
            if (!g->mexec && (rc = capture_model_graph(g)) != BMC_OK) return rc;
            bmc::DrawDyn* p = g->h_dyn.as<bmc::DrawDyn>();
            p->seed = model->seed;
            p->spec[0] = model->initial_speed;
            p->spec[1] = model->friction;
            p->spec[2] = model->grade;
            p->spec[3] = model->mass;
            p->spec[4] = model->drag_coeff;
            p->first = first;
            if ((rc = replay(g, out, info, t0, true)) != BMC_OK) return rc;
            const unsigned long long* c = g->h_ctr.as<unsigned long long>();
            const unsigned flags = static_cast<unsigned>(c[1]);
            if (flags & bmc::kDrawDomain) {
                return bmc::fail(g->ctx, BMC_E_DOMAIN, "friction_limit: weight-transfer denominator <= 0");
            }
            if (flags & bmc::kDrawUnported) {
                return bmc::fail(g->ctx, BMC_E_RANGE, "device sampler: a libm argument left the ported glibc range");
            }
            if (clamp_count) *clamp_count = c[0];
            return BMC_OK;
        }
        const size_t n = g->n;
        double* h = g->h_terms.as<double>();
        std::atomic<int> status{BMC_OK};
        std::atomic<uint64_t> clamps{0};
        bmc::ctx_pool(g->ctx, g->threads).parallel_for(
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
    } catch (...) {
        return bmc::abi_exception();
    }
}

void bmc_cuda_graph_destroy(bmc_graph* g) {
    if (!g) return;
    cudaSetDevice(g->ctx->device);
    cudaStreamSynchronize(g->ctx->stream);
    release(g);
    delete g;
}

}  // extern "C"
