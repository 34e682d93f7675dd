// bmc_capi.cpp -- the C-ABI (include/brakemc_cuda.h): device contexts, the
// actuator-table cache, the chunked host<->device pipeline behind
// bmc_cuda_run, and the host composition of the statistics kernels.
//
// Compiled by g++ with -ffp-contract=off: the double-double merges and the
// final statistics formulas below must not be contracted into FMAs.
#include "bmc_ctx.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <numeric>

namespace bmc {
namespace {

constexpr size_t kTableCap = size_t{1} << 20;      // 32 MB of stage values
constexpr uint64_t kDefaultChunk = uint64_t{1} << 22;  // 4M samples per pipeline slot
constexpr int kMaxCoarseSteps = 2048;
constexpr int kBucketsTarget = 2000;  // step buckets; x2 clamp classes <= 4096 keys

bool same_key(const WorldDerived& a, const WorldDerived& b) {
    return std::memcmp(&a, &b, sizeof a) == 0;
}

int ensure_table(bmc_ctx* ctx, const WorldDerived& d) {
    if (ctx->have_table && same_key(ctx->tkey, d)) return BMC_OK;
    const ActuatorTable t = build_actuator_table(d, kTableCap);
    ctx->have_table = false;
    // The kernel's crossover form of the clamp needs every stage sequence to
    // be non-increasing in n (true whenever brake_cmd < 0 and the RK4 step is
    // stable); anything else runs the generic inline path.
    bool monotone = true;
    double tmin = t.stages.empty() ? 0.0 : t.stages[0].a0;
    for (size_t k = 0; k < t.stages.size(); ++k) {
        const StageA& e = t.stages[k];
        for (double vv : {e.a0, e.a1, e.a2, e.a3}) {
            if (!(vv == vv)) monotone = false;
            tmin = std::min(tmin, vv);
        }
        if (k > 0) {
            const StageA& p = t.stages[k - 1];
            if (e.a0 > p.a0 || e.a1 > p.a1 || e.a2 > p.a2 || e.a3 > p.a3) monotone = false;
        }
    }
    ctx->t_converged = t.converged && monotone;
    ctx->t_min = tmin;
    ctx->t_len = static_cast<int>(t.stages.size());
    ctx->coarse_len = 0;
    if (ctx->t_converged) {
        const size_t bytes = t.stages.size() * sizeof(StageA);
        BMC_CK(ctx, ctx->d_table.reserve(bytes));
        BMC_CK(ctx, cudaMemcpy(ctx->d_table.p, t.stages.data(), bytes, cudaMemcpyHostToDevice));
        // Coarse brake_accel samples for the stop-step predictor: step
        // h = H*dt with H even, a(t) read at t = k*h/2 from the exact table.
        if (d.max_steps > 0 && d.dt > 0.0) {
            const long long H = std::max<long long>(2, 2 * std::llround(0.025 / d.dt));
            const long long K = (d.max_steps + H - 1) / H;
            if (K <= kMaxCoarseSteps) {
                std::vector<float> coarse(static_cast<size_t>(2 * K + 1));
                for (long long k = 0; k <= 2 * K; ++k) {
                    const long long idx = std::min<long long>(k * (H / 2), ctx->t_len - 1);
                    coarse[static_cast<size_t>(k)] = static_cast<float>(t.stages[idx].a0);
                }
                BMC_CK(ctx, ctx->d_coarse.reserve(coarse.size() * sizeof(float)));
                BMC_CK(ctx, cudaMemcpy(ctx->d_coarse.p, coarse.data(), coarse.size() * sizeof(float),
                                       cudaMemcpyHostToDevice));
                ctx->coarse_len = static_cast<int>(coarse.size());
                ctx->coarse_h = static_cast<float>(static_cast<double>(H) * d.dt);
            }
        }
    }
    ctx->tkey = d;
    ctx->have_table = true;
    return BMC_OK;
}

// Enqueue predictor/binning (optional) + rollout for n samples on `s`.
int enqueue_rollout(bmc_ctx* ctx, const bmc_terms& terms, uint64_t n, const WorldDerived& d,
                    const bmc_run_opts& opts, const bmc_outputs& out,
                    unsigned long long* total_steps_dev, cudaStream_t s, KernelEvents& ev,
                    uint32_t* launches) {
    if (n >= (uint64_t{1} << 32)) {
        return fail(ctx, BMC_E_CONFIG, "batch: at most 2^32-1 samples per device launch");
    }
    int rc = ensure_table(ctx, d);
    if (rc != BMC_OK) return rc;

    int mode = opts.table_mode;
    if (mode == kTableAuto) mode = ctx->t_len <= kSmemTableMax ? kTableShared : kTableGlobal;
    if (mode == kTableShared && ctx->t_len > kSmemTableMax) mode = kTableGlobal;
    if (!ctx->t_converged) mode = kTableNone;

    int sched = opts.schedule;
    if (sched == kScheduleDefault) sched = kScheduleBinned;
    if (ctx->coarse_len == 0 || mode == kTableNone) sched = kScheduleIndex;

    int bt = opts.block_threads;
    if (bt == 0) bt = mode == kTableGlobal ? 256 : 1024;

    uint32_t nl = 0;
    const uint32_t* perm = nullptr;
    ev.predicted = false;
    if (sched == kScheduleBinned && n > 0) {
        const int width = static_cast<int>((d.max_steps + kBucketsTarget) / kBucketsTarget);
        const int buckets = 2 * (static_cast<int>(d.max_steps / width) + 1);
        BMC_CK(ctx, ctx->keys.reserve(n * sizeof(uint16_t)));
        BMC_CK(ctx, ctx->perm.reserve(n * sizeof(uint32_t)));
        BMC_CK(ctx, ctx->hist.reserve(4096 * sizeof(unsigned int)));
        BMC_CK(ctx, cudaEventRecord(ev.p0, s));
        BMC_CK(ctx, cudaMemsetAsync(ctx->hist.p, 0, buckets * sizeof(unsigned int), s));
        PredictArgs pa{};
        pa.v0 = terms.initial_speed;
        pa.brake_floor = terms.brake_floor;
        pa.drag = terms.drag_factor;
        pa.grade = terms.grade_accel;
        pa.n = n;
        pa.coarse_a = ctx->d_coarse.as<float>();
        pa.coarse_len = ctx->coarse_len;
        pa.h = ctx->coarse_h;
        pa.inv_dt = static_cast<float>(1.0 / d.dt);
        pa.max_steps = static_cast<int32_t>(d.max_steps);
        pa.bucket_width = width;
        pa.buckets = buckets;
        pa.table_min = ctx->t_min;
        pa.keys = ctx->keys.as<uint16_t>();
        pa.hist = ctx->hist.as<unsigned int>();
        BMC_CK(ctx, launch_predict(pa, s));
        BMC_CK(ctx, launch_bin_scan(ctx->hist.as<unsigned int>(), buckets, s));
        BMC_CK(ctx, launch_bin_scatter(ctx->keys.as<uint16_t>(), n, ctx->hist.as<unsigned int>(),
                                       ctx->perm.as<uint32_t>(), s));
        BMC_CK(ctx, cudaEventRecord(ev.p1, s));
        nl += 3;
        perm = ctx->perm.as<uint32_t>();
        ev.predicted = true;
    }

    // [0] work counter (u32) | [8] executed steps (u64) | [16] lane slots (u64)
    BMC_CK(ctx, ctx->counter.reserve(64));
    BMC_CK(ctx, cudaMemsetAsync(ctx->counter.p, 0, 24, s));
    RolloutArgs ra{};
    ra.v0 = terms.initial_speed;
    ra.brake_floor = terms.brake_floor;
    ra.drag = terms.drag_factor;
    ra.grade = terms.grade_accel;
    ra.perm = perm;
    ra.n = n;
    ra.dt = d.dt;
    ra.half = d.half;
    ra.sixth = d.sixth;
    ra.brake_cmd = d.brake_cmd;
    ra.inv_tau = d.inv_tau;
    ra.max_steps = static_cast<int32_t>(d.max_steps);
    ra.table = ctx->d_table.as<StageA>();
    ra.table_len = ctx->t_len;
    ra.stop_distance = out.stop_distance;
    ra.steps = out.steps;
    ra.hit_horizon = out.hit_horizon;
    ra.total_steps = total_steps_dev;
    ra.work_counter = ctx->counter.as<unsigned int>();
    ra.counters = reinterpret_cast<unsigned long long*>(ctx->counter.as<char>() + 8);
    BMC_CK(ctx, cudaEventRecord(ev.r0, s));
    if (n > 0) {
        BMC_CK(ctx, launch_rollout(ra, mode, bt, s));
        ++nl;
    }
    BMC_CK(ctx, cudaEventRecord(ev.r1, s));
    if (launches) *launches += nl;
    return BMC_OK;
}

}  // namespace
}  // namespace bmc

using bmc::fail;

extern "C" {

int bmc_device_count(int* out) {
    int c = 0;
    const cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        *out = 0;
        return fail(nullptr, BMC_E_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    }
    *out = c;
    return BMC_OK;
}

int bmc_cuda_init(int device, bmc_ctx** out) {
    if (out == nullptr) return fail(nullptr, BMC_E_CONFIG, "bmc_cuda_init: null output");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        return fail(nullptr, BMC_E_CUDA,
                    std::string("no CUDA device: ") + (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
    }
    if (device < 0 || device >= count) {
        return fail(nullptr, BMC_E_CONFIG, "execution.device: out of range");
    }
    cudaDeviceProp prop{};
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) {
        return fail(nullptr, BMC_E_CUDA, std::string("cudaGetDeviceProperties: ") + cudaGetErrorString(e));
    }
    if (prop.major != 10) {
        return fail(nullptr, BMC_E_CUDA,
                    "device is sm_" + std::to_string(prop.major) + std::to_string(prop.minor) +
                        "; this build targets sm_100a only");
    }
    auto ctx = std::make_unique<bmc_ctx>();
    ctx->device = device;
    ctx->sms = prop.multiProcessorCount;
    if ((e = cudaSetDevice(device)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = ctx->kev.create()) != cudaSuccess) {
        return fail(nullptr, BMC_E_CUDA, std::string("context setup: ") + cudaGetErrorString(e));
    }
    for (auto& s : ctx->slots) {
        if ((e = cudaEventCreateWithFlags(&s.h2d_done, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&s.compute_done, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&s.d2h_done, cudaEventDisableTiming)) != cudaSuccess ||
            (e = s.kev.create()) != cudaSuccess) {
            return fail(nullptr, BMC_E_CUDA, std::string("context events: ") + cudaGetErrorString(e));
        }
    }
    *out = ctx.release();
    return BMC_OK;
}

void bmc_cuda_destroy(bmc_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    for (auto& s : ctx->slots) {
        s.h_terms.release();
        s.h_out.release();
        s.d_terms.release();
        s.d_out.release();
        if (s.h2d_done) cudaEventDestroy(s.h2d_done);
        if (s.compute_done) cudaEventDestroy(s.compute_done);
        if (s.d2h_done) cudaEventDestroy(s.d2h_done);
        s.kev.destroy();
    }
    for (bmc::DevBuf* b : {&ctx->d_table, &ctx->d_coarse, &ctx->keys, &ctx->perm, &ctx->hist,
                           &ctx->counter, &ctx->total_steps, &ctx->partials, &ctx->sel_hist,
                           &ctx->sel_pref, &ctx->sorted_h, &ctx->buckets, &ctx->hist_buf}) {
        b->release();
    }
    ctx->h_small.release();
    ctx->kev.destroy();
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
    if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
    delete ctx;
}

const char* bmc_cuda_last_error(const bmc_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

void* bmc_cuda_stream(bmc_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int bmc_cuda_sync(bmc_ctx* ctx) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    BMC_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return BMC_OK;
}

int bmc_cuda_rollout_device(bmc_ctx* ctx, const bmc_terms* terms, size_t n, const bmc_world* world,
                            const bmc_run_opts* opts, const bmc_outputs* out,
                            unsigned long long* total_steps_dev, void* stream) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (!terms || !world || !out) return fail(ctx, BMC_E_CONFIG, "bmc_cuda_rollout_device: null argument");
    if (n == 0) return fail(ctx, BMC_E_CONFIG, "batch: must be non-empty");
    bmc::WorldDerived d{};
    std::string err;
    if ((rc = bmc::derive_world(*world, &d, &err)) != BMC_OK) return fail(ctx, rc, err);
    const bmc_run_opts o = opts ? *opts : bmc_run_opts{};
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    ctx->last_launches = 0;
    rc = bmc::enqueue_rollout(ctx, *terms, n, d, o, *out, total_steps_dev, s, ctx->kev,
                              &ctx->last_launches);
    return rc;
}

int bmc_cuda_last_kernel_ms(bmc_ctx* ctx, float* rollout_ms, float* predict_ms) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    float r = 0.0f, p = 0.0f;
    BMC_CK(ctx, cudaEventElapsedTime(&r, ctx->kev.r0, ctx->kev.r1));
    if (ctx->kev.predicted) BMC_CK(ctx, cudaEventElapsedTime(&p, ctx->kev.p0, ctx->kev.p1));
    if (rollout_ms) *rollout_ms = r;
    if (predict_ms) *predict_ms = p;
    return BMC_OK;
}

int bmc_cuda_fp64_peak(bmc_ctx* ctx, int reps, double* ops_per_s, double* best_ms) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    BMC_CK(ctx, ctx->counter.reserve(64));
    double best = 1e30;
    uint64_t ops = 0;
    for (int r = 0; r < std::max(1, reps) + 1; ++r) {  // first launch is a warm-up
        BMC_CK(ctx, cudaEventRecord(ctx->kev.r0, ctx->stream));
        BMC_CK(ctx, bmc::launch_fp64_probe(ctx->counter.as<double>(), 4096, &ops, ctx->stream));
        BMC_CK(ctx, cudaEventRecord(ctx->kev.r1, ctx->stream));
        BMC_CK(ctx, cudaEventSynchronize(ctx->kev.r1));
        float ms = 0.0f;
        BMC_CK(ctx, cudaEventElapsedTime(&ms, ctx->kev.r0, ctx->kev.r1));
        if (r > 0) best = std::min(best, static_cast<double>(ms));
    }
    if (ops_per_s) *ops_per_s = static_cast<double>(ops) / (best * 1e-3);
    if (best_ms) *best_ms = best;
    return BMC_OK;
}

int bmc_cuda_last_lane_stats(bmc_ctx* ctx, uint64_t* steps, uint64_t* slots) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    unsigned long long c[2] = {0, 0};
    BMC_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->counter.p) {
        BMC_CK(ctx, cudaMemcpy(c, ctx->counter.as<char>() + 8, sizeof c, cudaMemcpyDeviceToHost));
    }
    if (steps) *steps = c[0];
    if (slots) *slots = c[1];
    return BMC_OK;
}

int bmc_cuda_last_launches(bmc_ctx* ctx, uint32_t* launches) {
    if (!ctx || !launches) return BMC_E_CONFIG;
    *launches = ctx->last_launches;
    return BMC_OK;
}

int bmc_cuda_run(bmc_ctx* ctx, const bmc_sample* samples, size_t n, const bmc_world* world,
                 const bmc_run_opts* opts, bmc_result* out, bmc_run_info* info) {
    using Clock = std::chrono::steady_clock;
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (n == 0) return fail(ctx, BMC_E_CONFIG, "batch: must be non-empty");  // backends.cpp:41-43
    if (!samples || !world || !out) return fail(ctx, BMC_E_CONFIG, "bmc_cuda_run: null argument");
    bmc::WorldDerived d{};
    std::string err;
    if ((rc = bmc::derive_world(*world, &d, &err)) != BMC_OK) return fail(ctx, rc, err);
    const bmc_run_opts o = opts ? *opts : bmc_run_opts{};
    const uint64_t chunk = std::min<uint64_t>(o.chunk_samples ? o.chunk_samples : bmc::kDefaultChunk, n);
    const unsigned threads = bmc::resolve_threads(o.host_threads);

    for (auto& s : ctx->slots) {
        BMC_CK(ctx, s.h_terms.reserve(chunk * 32));
        BMC_CK(ctx, s.h_out.reserve(chunk * 13));
        BMC_CK(ctx, s.d_terms.reserve(chunk * 32));
        BMC_CK(ctx, s.d_out.reserve(chunk * 13));
        s.busy = false;
    }
    BMC_CK(ctx, ctx->total_steps.reserve(sizeof(unsigned long long)));
    BMC_CK(ctx, cudaMemsetAsync(ctx->total_steps.p, 0, sizeof(unsigned long long), ctx->stream));

    double kernel_ms = 0.0, predict_ms = 0.0;
    uint32_t launches = 0;
    const auto t0 = Clock::now();

    auto finish = [&](bmc::Slot& s) -> int {
        if (!s.busy) return BMC_OK;
        BMC_CK(ctx, cudaEventSynchronize(s.d2h_done));
        float ms = 0.0f;
        BMC_CK(ctx, cudaEventElapsedTime(&ms, s.kev.r0, s.kev.r1));
        kernel_ms += ms;
        if (s.kev.predicted) {
            BMC_CK(ctx, cudaEventElapsedTime(&ms, s.kev.p0, s.kev.p1));
            predict_ms += ms;
        }
        const double* dd = s.h_out.as<double>();
        const int32_t* st = reinterpret_cast<const int32_t*>(s.h_out.as<char>() + s.len * 8);
        const uint8_t* hz = reinterpret_cast<const uint8_t*>(s.h_out.as<char>() + s.len * 12);
        bmc_result* dst = out + s.offset;
        const double dt = d.dt;
        bmc::host_pool().parallel_for(
            s.len,
            [&](size_t b, size_t e) {
                for (size_t i = b; i < e; ++i) {
                    bmc_result r;
                    std::memset(&r, 0, sizeof r);
                    r.stop_distance = dd[i];
                    r.stop_time = static_cast<double>(st[i]) * dt;  // integrator.cpp:23,27
                    r.steps = st[i];
                    r.hit_horizon = hz[i];
                    dst[i] = r;
                }
            },
            threads);
        s.busy = false;
        return BMC_OK;
    };

    const uint64_t nchunks = (n + chunk - 1) / chunk;
    for (uint64_t k = 0; k < nchunks; ++k) {
        bmc::Slot& s = ctx->slots[k & 1];
        if ((rc = finish(s)) != BMC_OK) return rc;
        s.offset = k * chunk;
        s.len = std::min<uint64_t>(chunk, n - s.offset);
        double* hv0 = s.h_terms.as<double>();
        double* hfl = hv0 + s.len;
        double* hdr = hfl + s.len;
        double* hgr = hdr + s.len;
        std::atomic<int> status{BMC_OK};
        bmc::host_pool().parallel_for(
            s.len,
            [&](size_t b, size_t e) {
                const int r = bmc::stage_terms_serial(samples + s.offset + b, e - b, *world, hv0 + b,
                                                      hfl + b, hdr + b, hgr + b);
                if (r != BMC_OK) status = r;
            },
            threads);
        if (status != BMC_OK) {
            cudaStreamSynchronize(ctx->stream);
            cudaStreamSynchronize(ctx->d2h);
            return fail(ctx, BMC_E_DOMAIN, "friction_limit: weight-transfer denominator <= 0");
        }
        BMC_CK(ctx, cudaMemcpyAsync(s.d_terms.p, s.h_terms.p, s.len * 32, cudaMemcpyHostToDevice, ctx->h2d));
        BMC_CK(ctx, cudaEventRecord(s.h2d_done, ctx->h2d));
        BMC_CK(ctx, cudaStreamWaitEvent(ctx->stream, s.h2d_done, 0));
        const double* dv0 = s.d_terms.as<double>();
        bmc_terms terms{dv0, dv0 + s.len, dv0 + 2 * s.len, dv0 + 3 * s.len};
        char* dout = s.d_out.as<char>();
        bmc_outputs outs{reinterpret_cast<double*>(dout), reinterpret_cast<int32_t*>(dout + s.len * 8),
                         reinterpret_cast<uint8_t*>(dout + s.len * 12)};
        rc = bmc::enqueue_rollout(ctx, terms, s.len, d, o, outs,
                                  ctx->total_steps.as<unsigned long long>(), ctx->stream, s.kev,
                                  &launches);
        if (rc != BMC_OK) return rc;
        BMC_CK(ctx, cudaEventRecord(s.compute_done, ctx->stream));
        BMC_CK(ctx, cudaStreamWaitEvent(ctx->d2h, s.compute_done, 0));
        // d_out holds d (8B), steps (4B), horizon (1B) blocks contiguously
        BMC_CK(ctx, cudaMemcpyAsync(s.h_out.p, s.d_out.p, s.len * 13, cudaMemcpyDeviceToHost, ctx->d2h));
        BMC_CK(ctx, cudaEventRecord(s.d2h_done, ctx->d2h));
        s.busy = true;
    }
    // drain in submission order
    for (uint64_t k = nchunks > 2 ? nchunks - 2 : 0; k < nchunks; ++k) {
        if ((rc = finish(ctx->slots[k & 1])) != BMC_OK) return rc;
    }
    unsigned long long steps_total = 0;
    BMC_CK(ctx, cudaMemcpy(&steps_total, ctx->total_steps.p, sizeof steps_total, cudaMemcpyDeviceToHost));
    const double wall = std::chrono::duration<double>(Clock::now() - t0).count();
    ctx->last_launches = launches;
    if (info) {
        info->wall_s = wall;
        info->kernel_ms = kernel_ms;
        info->predict_ms = predict_ms;
        info->total_steps = steps_total;
        info->h2d_bytes = static_cast<uint64_t>(n) * 32;
        info->d2h_bytes = static_cast<uint64_t>(n) * 13;
        info->launches = launches;
        info->chunks = static_cast<uint32_t>(nchunks);
    }
    return BMC_OK;
}

}  // extern "C"
