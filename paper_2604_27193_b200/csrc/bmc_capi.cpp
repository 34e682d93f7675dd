// bmc_capi.cpp -- the C-ABI (include/brakemc_cuda.h): device contexts, the
// actuator-table cache, rollout plans, and the chunked host<->device
// pipeline behind bmc_cuda_run / bmc_cuda_run_model.
//
// Compiled by g++ with -ffp-contract=off.
#include "bmc_ctx.h"

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <numeric>

namespace bmc {
namespace {

constexpr size_t kTableCap = size_t{1} << 20;          // 32 MB of stage values
// Pipeline chunk (samples per slot).  Every chunk's rollout costs at least
// the latency of its longest sample (~1.2 ms for the default model) plus
// its launches, while one chunk alone cannot overlap its host staging, H2D,
// D2H and unpack with compute.  Measured on the B200 (tools/chunk_sweep.py,
// profiles/round1_chunk_sweep.txt, and the 1e8 bench; each slot has its own
// compute stream, so a chunk's binning and rollout fill the previous
// chunk's tail): up to 128k samples one chunk, up to 8M two chunks, then
// four chunks capped at 4M samples.
uint64_t default_chunk(uint64_t n) {
    constexpr uint64_t kOne = uint64_t{1} << 17, kTwo = uint64_t{1} << 23, kMax = uint64_t{1} << 22;
    if (n <= kOne) return n;
    if (n <= kTwo) return (n + 1) / 2;
    return std::min(kMax, (n + 3) / 4);
}
constexpr int kMaxCoarseSteps = 2048;
constexpr int kBucketsTarget = 2000;  // step buckets; x2 clamp classes <= 4096 keys
// Two chains per thread (one table-row load feeds both) once a launch has
// enough 64-sample groups to fill the GPU several times; below that the
// latency of each thread's doubled work dominates (tools/kernel_sweep.py
// --ilpcmp, profiles/round1_sweep_ilp.txt: crossover ~1M samples).
constexpr uint64_t kIlp2MinSamples = uint64_t{1} << 20;
constexpr int kDefaultIlp2Block = 640;
constexpr int kDefaultTestBlock = 8;  // profiles/round1_sweep_testblock.txt

bool same_key(const WorldDerived& a, const WorldDerived& b) {
    return std::memcmp(&a, &b, sizeof a) == 0;
}

int bucket_width(const WorldDerived& d) {
    return static_cast<int>((d.max_steps + kBucketsTarget) / kBucketsTarget);
}

int bucket_count(const WorldDerived& d) {
    return 2 * (static_cast<int>(d.max_steps / bucket_width(d)) + 1);
}

}  // namespace

int ensure_table(bmc_ctx* ctx, const WorldDerived& d, TableEntry** out) {
    auto& cache = ctx->tables;
    for (size_t i = 0; i < cache.size(); ++i) {
        if (same_key(cache[i]->key, d)) {
            std::rotate(cache.begin(), cache.begin() + static_cast<std::ptrdiff_t>(i),
                        cache.begin() + static_cast<std::ptrdiff_t>(i) + 1);
            *out = cache.front().get();
            return BMC_OK;
        }
    }
    const ActuatorTable t = build_actuator_table(d, kTableCap);
    auto e = std::make_unique<TableEntry>();
    e->key = d;
    // The kernel's crossover form of the clamp needs every stage sequence to
    // be non-increasing in n (true whenever brake_cmd < 0 and the RK4 step is
    // stable); anything else runs the generic inline path.
    bool monotone = true;
    double tmin = t.stages.empty() ? 0.0 : t.stages[0].a0;
    for (size_t k = 0; k < t.stages.size(); ++k) {
        const StageA& st = t.stages[k];
        for (double vv : {st.a0, st.a1, st.a2, st.a3}) {
            if (!(vv == vv)) monotone = false;
            tmin = std::min(tmin, vv);
        }
        if (k > 0) {
            const StageA& p = t.stages[k - 1];
            if (st.a0 > p.a0 || st.a1 > p.a1 || st.a2 > p.a2 || st.a3 > p.a3) monotone = false;
        }
    }
    e->converged = t.converged && monotone;
    e->t_min = tmin;
    e->t_len = static_cast<int>(t.stages.size());
    e->coarse_len = 0;
    if (e->converged) {
        // fresh buffers, written before any launch can see them
        const size_t bytes = t.stages.size() * sizeof(StageA);
        BMC_CK(ctx, e->table.reserve(bytes));
        BMC_CK(ctx, cudaMemcpy(e->table.p, t.stages.data(), bytes, cudaMemcpyHostToDevice));
        // Coarse brake_accel samples for the stop-step predictor: step
        // h = H*dt with H even, a(t) read at t = k*h/2 from the exact table.
        if (d.max_steps > 0 && d.dt > 0.0) {
            // coarse step ~0.2 s (BMC_COARSE_STEP_S overrides, for tuning):
            // it only orders samples, never changes a result
            double hs = 0.2;
            if (const char* env = std::getenv("BMC_COARSE_STEP_S")) hs = std::max(1e-6, std::atof(env));
            const long long H = std::max<long long>(2, 2 * std::llround(0.5 * hs / d.dt));
            const long long K = (d.max_steps + H - 1) / H;
            if (K <= kMaxCoarseSteps) {
                std::vector<float> coarse(static_cast<size_t>(2 * K + 1));
                for (long long k = 0; k <= 2 * K; ++k) {
                    const long long idx = std::min<long long>(k * (H / 2), e->t_len - 1);
                    coarse[static_cast<size_t>(k)] = static_cast<float>(t.stages[idx].a0);
                }
                BMC_CK(ctx, e->coarse.reserve(coarse.size() * sizeof(float)));
                BMC_CK(ctx, cudaMemcpy(e->coarse.p, coarse.data(), coarse.size() * sizeof(float),
                                       cudaMemcpyHostToDevice));
                e->coarse_len = static_cast<int>(coarse.size());
                e->coarse_h = static_cast<float>(static_cast<double>(H) * d.dt);
                // the transient: coarse steps until brake_accel stays within
                // 1e-6 of its final value (the predictor solves the rest in
                // closed form)
                const float a_inf = coarse.back();
                long long j = 2 * K;
                while (j > 0 && std::fabs(coarse[static_cast<size_t>(j - 1)] - a_inf) <=
                                    1e-6f * std::fabs(a_inf)) {
                    --j;
                }
                e->coarse_steps = static_cast<int>((j + 1) / 2);
                e->coarse_inf = a_inf;
            }
        }
    }
    if (cache.size() >= kTableCacheEntries) {
        // the least recently used world may still be read by a launch in
        // flight on any stream: wait for the device before freeing it
        BMC_CK(ctx, cudaDeviceSynchronize());
        cache.pop_back();
    }
    cache.insert(cache.begin(), std::move(e));
    *out = cache.front().get();
    return BMC_OK;
}

ThreadPool& ctx_pool(bmc_ctx* ctx, unsigned threads) {
    if (!ctx->pool || ctx->pool_threads < threads) {
        ctx->pool.reset();
        ctx->pool = std::make_unique<ThreadPool>(threads);
        ctx->pool_threads = threads;
    }
    return *ctx->pool;
}

int make_plan(bmc_ctx* ctx, const WorldDerived& d, const bmc_run_opts& opts, uint64_t n,
              Plan* plan) {
    TableEntry* te = nullptr;
    const int rc = ensure_table(ctx, d, &te);
    if (rc != BMC_OK) return rc;
    Plan p;
    p.d = d;
    int mode = opts.table_mode;
    if (mode == kTableAuto) mode = te->t_len <= kSmemTableMax ? kTableShared : kTableGlobal;
    if (mode == kTableShared && te->t_len > kSmemTableMax) mode = kTableGlobal;
    if (!te->converged) mode = kTableNone;
    int sched = opts.schedule;
    if (sched == kScheduleDefault) sched = kScheduleBinned;
    if (te->coarse_len == 0 || mode == kTableNone) sched = kScheduleIndex;
    int ilp = opts.ilp != 0 ? opts.ilp : (n >= kIlp2MinSamples ? 2 : 1);
    if (ilp != 1 && ilp != 2) return fail(ctx, BMC_E_CONFIG, "execution.ilp: must be 1 or 2");
    if (mode == kTableNone) ilp = 1;
    int tb = opts.test_block == 0 ? kDefaultTestBlock : opts.test_block;
    if (tb != 1 && tb != 8) return fail(ctx, BMC_E_CONFIG, "execution.test_block: must be 1 or 8");
    if (mode == kTableNone) tb = 1;
    int bt = opts.block_threads;
    if (bt == 0) bt = ilp == 2 ? kDefaultIlp2Block : (mode == kTableGlobal ? 256 : 1024);
    const bool ok_bt = ilp == 2 ? (bt == 512 || bt == 640 || bt == 768)
                                : (bt == 256 || bt == 512 || bt == 768 || bt == 1024);
    if (!ok_bt) {
        return fail(ctx, BMC_E_CONFIG,
                    ilp == 2 ? "execution.block_threads: must be 512, 640 or 768 with ilp 2"
                             : "execution.block_threads: must be 256, 512, 768 or 1024");
    }
    p.mode = mode;
    p.sched = sched;
    p.bt = bt;
    p.ilp = ilp;
    p.test_block = tb;
    p.table = te->table.as<StageA>();
    p.table_len = te->t_len;
    p.table_min = te->t_min;
    p.coarse = te->coarse.as<float>();
    p.coarse_len = te->coarse_len;
    p.coarse_h = te->coarse_h;
    p.coarse_steps = te->coarse_steps;
    p.coarse_inf = te->coarse_inf;
    *plan = p;
    return BMC_OK;
}

// Binned outputs: the rollout writes packed 16-B records in sorted order
// (full sectors, coalesced) and unpermute gathers them into index order --
// measured at 1e8: rollout DRAM traffic 45.8 B/sample + unpermute 73
// B/sample, 942.6 ms/step.  BMC_DIRECT_OUTPUTS=1 instead writes each
// sample's outputs at its own index from the rollout epilogue through a
// forward map (no unpermute pass; 940.6 ms/step, but the scattered partial
// writes cost 226 B/sample of read-modify-write traffic inside the rollout,
// hidden under its FP64 bound).  profiles/round2_summary.md has both.
// The streamed pipeline (run_pipeline) writes directly: its chunk outputs
// (13 B/sample, <= 64 MiB) stay in the 126 MB L2, so the scattered writes
// merge there instead of costing DRAM read-modify-write, and a chunk's D2H
// no longer waits for an unpermute that the next chunk's persistent rollout
// would hold off the SMs.
int env_direct_outputs() {
    static const int v = [] {
        const char* e = std::getenv("BMC_DIRECT_OUTPUTS");
        return (e && (e[0] == '0' || e[0] == '1')) ? e[0] - '0' : -1;
    }();
    return v;
}
bool resolve_direct(int direct) {
    if (env_direct_outputs() >= 0) return env_direct_outputs() == 1;
    return direct == 1;
}
constexpr uint64_t kDirectChunkBytes = uint64_t{64} << 20;

int direct_outputs_for(uint64_t n) { return n * 13 <= kDirectChunkBytes ? 1 : 0; }

int reserve_scratch(bmc_ctx* ctx, Scratch& sc, const Plan& plan, uint64_t n, int direct) {
    // counter: [0] work counter (u32) | [8] executed steps | [16] lane slots
    BMC_CK(ctx, sc.counter.reserve(64));
    if (plan.sched == kScheduleBinned) {
        const uint64_t m = std::max<uint64_t>(n, 1);
        BMC_CK(ctx, sc.keys.reserve(m * sizeof(uint16_t)));
        BMC_CK(ctx, sc.perm.reserve(m * sizeof(uint32_t)));  // forward (or inverse) permutation
        BMC_CK(ctx, sc.hist.reserve(bin_windows(m) * 4096 * sizeof(unsigned int)));
        BMC_CK(ctx, sc.packed_in.reserve(m * sizeof(PackedTerms)));
        if (!resolve_direct(direct)) BMC_CK(ctx, sc.packed_out.reserve(m * sizeof(PackedOut)));
    }
    return BMC_OK;
}

int enqueue_rollout(bmc_ctx* ctx, const Plan& plan, Scratch& sc, const bmc_terms& terms,
                    uint64_t n, const bmc_outputs& out, unsigned long long* total_steps_dev,
                    cudaStream_t s, KernelEvents* ev, uint32_t* launches, const P1Args* p1,
                    int direct) {
    if (n >= (uint64_t{1} << 32)) {
        return fail(ctx, BMC_E_CONFIG, "batch: at most 2^32-1 samples per device launch");
    }
    int rc = reserve_scratch(ctx, sc, plan, n, direct);
    if (rc != BMC_OK) return rc;
    const WorldDerived& d = plan.d;
    uint32_t nl = 0;
    bool packed = false;
    const bool any_out = out.stop_distance || out.steps || out.hit_horizon;
    const bool direct_out = resolve_direct(direct);
    if (ev) ev->predicted = false;
    if (plan.sched == kScheduleBinned && n > 0) {
        const int buckets = bucket_count(d);
        if (ev) BMC_CK(ctx, cudaEventRecord(ev->p0, s));
        BMC_CK(ctx, cudaMemsetAsync(sc.hist.p, 0, bin_windows(n) * buckets * sizeof(unsigned int), s));
        PredictArgs pa{};
        pa.v0 = terms.initial_speed;
        pa.brake_floor = terms.brake_floor;
        pa.drag = terms.drag_factor;
        pa.grade = terms.grade_accel;
        pa.n = n;
        pa.coarse_a = plan.coarse;
        pa.coarse_len = plan.coarse_len;
        pa.h = plan.coarse_h;
        pa.coarse_steps = plan.coarse_steps;
        pa.a_inf = plan.coarse_inf;
        pa.inv_dt = static_cast<float>(1.0 / d.dt);
        pa.max_steps = static_cast<int32_t>(d.max_steps);
        pa.bucket_width = bucket_width(d);
        pa.buckets = buckets;
        pa.table_min = plan.table_min;
        pa.keys = sc.keys.as<uint16_t>();
        pa.hist = sc.hist.as<unsigned int>();
        BMC_CK(ctx, launch_predict(pa, s));
        BMC_CK(ctx, launch_bin_scan(sc.hist.as<unsigned int>(), buckets, n, s));
        BMC_CK(ctx, launch_bin_scatter(sc.keys.as<uint16_t>(), n, sc.hist.as<unsigned int>(),
                                       terms.initial_speed, terms.brake_floor, terms.drag_factor,
                                       terms.grade_accel, sc.packed_in.as<PackedTerms>(),
                                       sc.perm.as<uint32_t>(), direct_out ? 1 : 0, buckets, s));
        if (ev) BMC_CK(ctx, cudaEventRecord(ev->p1, s));
        nl += 3;
        packed = true;
        if (ev) ev->predicted = true;
    }
    BMC_CK(ctx, cudaMemsetAsync(sc.counter.p, 0, 24, s));
    RolloutArgs ra{};
    ra.v0 = terms.initial_speed;
    ra.brake_floor = terms.brake_floor;
    ra.drag = terms.drag_factor;
    ra.grade = terms.grade_accel;
    ra.perm = nullptr;
    ra.packed_in = packed ? sc.packed_in.as<PackedTerms>() : nullptr;
    ra.packed_out = (packed && !direct_out) ? sc.packed_out.as<PackedOut>() : nullptr;
    ra.fwd = (packed && direct_out) ? sc.perm.as<uint32_t>() : nullptr;
    ra.n = n;
    ra.dt = d.dt;
    ra.half = d.half;
    ra.sixth = d.sixth;
    ra.brake_cmd = d.brake_cmd;
    ra.inv_tau = d.inv_tau;
    ra.max_steps = static_cast<int32_t>(d.max_steps);
    ra.table = plan.table;
    ra.table_len = plan.table_len;
    ra.stop_distance = out.stop_distance;
    ra.steps = out.steps;
    ra.hit_horizon = out.hit_horizon;
    ra.total_steps = total_steps_dev;
    ra.work_counter = sc.counter.as<unsigned int>();
    ra.counters = reinterpret_cast<unsigned long long*>(sc.counter.as<char>() + 8);
    if (p1) ra.p1 = *p1;
    // BMC_PER_STEP_TEST=1 (A/B runs): every block folds every step's speed
    static const bool per_step = [] {
        const char* e = std::getenv("BMC_PER_STEP_TEST");
        return e && e[0] == '1';
    }();
    ra.monotone_blocks = per_step ? 0 : 1;
    if (ev) BMC_CK(ctx, cudaEventRecord(ev->r0, s));
    if (n > 0) {
        BMC_CK(ctx, launch_rollout(ra, plan.mode, plan.bt, plan.ilp, plan.test_block, s));
        ++nl;
    }
    if (ev) BMC_CK(ctx, cudaEventRecord(ev->r1, s));
    if (ev) ev->unpermuted = false;
    if (packed && !direct_out && n > 0 && any_out) {
        BMC_CK(ctx, launch_unpermute(sc.packed_out.as<PackedOut>(), sc.perm.as<uint32_t>(), n,
                                     out.stop_distance, out.steps, out.hit_horizon, s));
        ++nl;
        if (ev) {
            BMC_CK(ctx, cudaEventRecord(ev->u1, s));
            ev->unpermuted = true;
        }
    }
    if (launches) *launches += nl;
    return BMC_OK;
}


int use_device_sampler(bmc_ctx* ctx, const bmc_run_opts& o, bool* device) {
    *device = false;
    if (o.sampler < 0 || o.sampler > 2) {
        return fail(ctx, BMC_E_CONFIG, "execution.sampler: must be 0 (auto), 1 (host) or 2 (device)");
    }
    if (o.sampler == 1) return BMC_OK;
    std::string why;
    const bool ok = device_sampler_supported(&why);
    if (!ok && o.sampler == 2) return fail(ctx, BMC_E_CONFIG, "execution.sampler: " + why);
    *device = ok;
    return BMC_OK;
}

DrawArgs draw_args(const bmc_model& m, uint64_t first, uint64_t n, const bmc_world& w) {
    DrawArgs a{};
    a.seed = m.seed;
    a.spec[0] = m.initial_speed;
    a.spec[1] = m.friction;
    a.spec[2] = m.grade;
    a.spec[3] = m.mass;
    a.spec[4] = m.drag_coeff;
    a.first = first;
    a.n = n;
    a.cg_height = w.cg_height;
    a.wheelbase = w.wheelbase;
    a.gravity = w.gravity;
    a.air_density = w.air_density;
    a.frontal_area = w.frontal_area;
    return a;
}

int finish_draw(bmc_ctx* ctx, const DevBuf& ctr, uint64_t* clamps) {
    unsigned long long c[2] = {0, 0};
    BMC_CK(ctx, cudaMemcpyAsync(c, ctr.p, sizeof c, cudaMemcpyDeviceToHost, ctx->stream));
    BMC_CK(ctx, cudaStreamSynchronize(ctx->stream));
    const unsigned flags = static_cast<unsigned>(c[1]);
    if (flags & kDrawDomain) {
        return fail(ctx, BMC_E_DOMAIN, "friction_limit: weight-transfer denominator <= 0");
    }
    if (flags & kDrawUnported) {
        return fail(ctx, BMC_E_RANGE,
                    "device sampler: a libm argument left the ported glibc range (log of x <= 0 "
                    "or subnormal, |x| >= 105414350 or non-finite for sin/cos)");
    }
    if (clamps) *clamps = c[0];
    return BMC_OK;
}

namespace {

int trace_level() {
    static const int v = [] {
        const char* e = std::getenv("BMC_PIPE_TRACE");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

// Chunked host<->device pipeline (3 slots): per chunk the host pool fills
// pinned SoA terms (from AoS samples, or straight from the sampler), the
// h2d stream copies them, the compute stream bins + rolls out, and either
// the d2h stream returns the compact outputs for the host unpack, or the
// kernel writes straight into caller-owned device outputs.
// The persistent rollout of chunk k+1 takes every SM during the tail of
// chunk k's rollout, so any kernel after chunk k's rollout (an unpermute)
// waited for the whole of chunk k+1, its D2H and host unpack came late, and
// with two slots the host -- which unpacks chunk k before staging chunk k+2
// into the same slot -- left the device idle ~9.5 ms every second chunk
// (BMC_PIPE_TRACE=2 timeline, profiles/round2_pipeline_trace.txt).  Chunks
// therefore write their outputs directly (direct_outputs_for), and a third
// slot gives the host a whole chunk of slack: 1040 -> 940 ms at 1e8.
int run_pipeline(bmc_ctx* ctx, const bmc_world& w, const WorldDerived& d, const bmc_run_opts& o,
                 uint64_t n, const bmc_sample* samples, const bmc_model* model, uint64_t first,
                 bmc_result* host_out, const bmc_outputs* dev_out, bmc_run_info* info,
                 uint64_t* clamp_count, const P1Args* p1 = nullptr) {
    using Clock = std::chrono::steady_clock;
    const uint64_t chunk = std::min<uint64_t>(o.chunk_samples ? o.chunk_samples : default_chunk(n), n);
    const unsigned threads = resolve_threads(o.host_threads);
    Plan plan;
    int rc = make_plan(ctx, d, o, chunk, &plan);
    if (rc != BMC_OK) return rc;
    if (p1) fit_stats_plan(&plan, *p1);
    bool dev_draw = false;
    if (model && (rc = use_device_sampler(ctx, o, &dev_draw)) != BMC_OK) return rc;
    if (dev_draw) {
        BMC_CK(ctx, ctx->draw_ctr.reserve(16));
        BMC_CK(ctx, cudaMemsetAsync(ctx->draw_ctr.p, 0, 16, ctx->stream));
    }
    static const uint64_t kSlots = [] {  // BMC_PIPE_SLOTS=2 (A/B runs)
        const char* e = std::getenv("BMC_PIPE_SLOTS");
        return (e && e[0] == '2') ? uint64_t{2} : uint64_t{sizeof(bmc_ctx::slots) / sizeof(Slot)};
    }();
    // Chunk schedule: fixed chunks; long automatic schedules (>= 8 chunks)
    // start with a chunk/4 piece so less host staging and H2D is exposed
    // before the device starts: 1e8 host -> host 932.0 -> 929.3 ms (3 slots,
    // profiles/round2_pipeline_trace.txt; BMC_PIPE_HEAD=d sets the divisor,
    // 1 = off).  Ramping both edges down lost 7 ms with two slots.
    static const uint64_t head_div = [] {
        const char* e = std::getenv("BMC_PIPE_HEAD");
        const long v = e ? std::atol(e) : 4;
        return static_cast<uint64_t>(v >= 1 && v <= 64 ? v : 4);
    }();
    std::vector<std::pair<uint64_t, uint64_t>> sched;
    {
        uint64_t off = 0;
        if (head_div > 1 && o.chunk_samples == 0 && n >= 8 * chunk) {
            const uint64_t h = std::max<uint64_t>(1, chunk / head_div);
            sched.emplace_back(0, h);
            off = h;
        }
        for (; off < n; off += chunk) sched.emplace_back(off, std::min(chunk, n - off));
    }
    const uint64_t nchunks = sched.size();
    const uint64_t used_slots = std::min(kSlots, nchunks);
    const int direct = direct_outputs_for(chunk);
    for (uint64_t q = 0; q < used_slots; ++q) {
        Slot& s = ctx->slots[q];
        if (!dev_draw) BMC_CK(ctx, s.h_terms.reserve(chunk * 32));
        BMC_CK(ctx, s.d_terms.reserve(chunk * 32));
        if (host_out) {
            BMC_CK(ctx, s.h_out.reserve(chunk * 13));
            BMC_CK(ctx, s.d_out.reserve(chunk * 13));
        }
        s.busy = false;
    }
    BMC_CK(ctx, ctx->total_steps.reserve(sizeof(unsigned long long)));
    BMC_CK(ctx, cudaMemsetAsync(ctx->total_steps.p, 0, sizeof(unsigned long long), ctx->stream));
    for (uint64_t q = 0; q < used_slots; ++q) {
        if ((rc = reserve_scratch(ctx, ctx->slots[q].sc, plan, chunk, direct)) != BMC_OK) return rc;
    }
    // the slot streams start after the counters above are cleared
    BMC_CK(ctx, cudaStreamSynchronize(ctx->stream));

    double kernel_ms = 0.0, predict_ms = 0.0;
    uint32_t launches = 0;
    std::atomic<uint64_t> clamps{0};
    const auto t0 = Clock::now();
    // BMC_PIPE_TRACE=1: host-side phase totals of this call on stderr
    // (waiting on the device, unpack, staging) -- diagnostics only
    const bool trace = trace_level() >= 1;
    double t_wait = 0.0, t_unpack = 0.0, t_stage = 0.0;
    // BMC_PIPE_TRACE=2 adds the device timeline of every chunk (ms from the
    // call's start): binning start/end, rollout start/end, unpermute end
    cudaEvent_t base = nullptr;
    std::vector<std::array<float, 6>> tl;
    if (trace_level() >= 2) {
        BMC_CK(ctx, cudaEventCreate(&base));
        BMC_CK(ctx, cudaEventRecord(base, ctx->stream));
    }
    auto since = [](Clock::time_point a) { return std::chrono::duration<double>(Clock::now() - a).count(); };

    auto finish = [&](Slot& s) -> int {
        if (!s.busy) return BMC_OK;
        auto tw = Clock::now();
        BMC_CK(ctx, cudaEventSynchronize(s.d2h_done));
        t_wait += since(tw);
        if (base) {
            std::array<float, 6> r{};
            r[0] = static_cast<float>(s.offset / chunk);
            cudaEvent_t evs[5] = {s.kev.p0, s.kev.p1, s.kev.r0, s.kev.r1, s.kev.u1};
            for (int q = 0; q < 5; ++q) {
                const bool have = (q >= 2 || s.kev.predicted) && (q < 4 || s.kev.unpermuted);
                r[q + 1] = -1.0f;
                if (have) BMC_CK(ctx, cudaEventElapsedTime(&r[q + 1], base, evs[q]));
            }
            tl.push_back(r);
        }
        tw = Clock::now();
        float ms = 0.0f;
        BMC_CK(ctx, cudaEventElapsedTime(&ms, s.kev.r0, s.kev.r1));
        kernel_ms += ms;
        if (s.kev.predicted) {
            BMC_CK(ctx, cudaEventElapsedTime(&ms, s.kev.p0, s.kev.p1));
            predict_ms += ms;
        }
        if (host_out) {
            const double* dd = s.h_out.as<double>();
            const int32_t* st = reinterpret_cast<const int32_t*>(s.h_out.as<char>() + s.len * 8);
            const uint8_t* hz = reinterpret_cast<const uint8_t*>(s.h_out.as<char>() + s.len * 12);
            bmc_result* dst = host_out + s.offset;
            const double dt = d.dt;
            ctx_pool(ctx, threads).parallel_for(
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
        }
        t_unpack += since(tw);
        s.busy = false;
        return BMC_OK;
    };

    for (uint64_t k = 0; k < nchunks; ++k) {
        Slot& s = ctx->slots[k % kSlots];
        if ((rc = finish(s)) != BMC_OK) return rc;
        s.offset = sched[k].first;
        s.len = sched[k].second;
        if (dev_draw) {
            // samples drawn on the device straight into this slot's terms
            DrawArgs da = draw_args(*model, first + s.offset, s.len, w);
            double* dt0 = s.d_terms.as<double>();
            da.v0 = dt0;
            da.brake_floor = dt0 + s.len;
            da.drag = dt0 + 2 * s.len;
            da.grade = dt0 + 3 * s.len;
            da.clamps = ctx->draw_ctr.as<unsigned long long>();
            da.flags = reinterpret_cast<unsigned int*>(ctx->draw_ctr.as<char>() + 8);
            BMC_CK(ctx, launch_draw_terms(da, ctx->sms, s.compute));
            ++launches;
        } else {
            double* hv0 = s.h_terms.as<double>();
            double* hfl = hv0 + s.len;
            double* hdr = hfl + s.len;
            double* hgr = hdr + s.len;
            const auto ts = Clock::now();
            std::atomic<int> status{BMC_OK};
            ctx_pool(ctx, threads).parallel_for(
                s.len,
                [&](size_t b, size_t e) {
                    int r;
                    if (samples) {
                        r = stage_terms_serial(samples + s.offset + b, e - b, w, hv0 + b, hfl + b,
                                               hdr + b, hgr + b);
                    } else {
                        uint64_t c = 0;
                        r = draw_terms_serial(*model, first + s.offset + b, e - b, w, hv0 + b, hfl + b,
                                              hdr + b, hgr + b, &c);
                        clamps += c;
                    }
                    if (r != BMC_OK) status = r;
                },
                threads);
            t_stage += since(ts);
            if (status != BMC_OK) {
                for (auto& q : ctx->slots) cudaStreamSynchronize(q.compute);
                cudaStreamSynchronize(ctx->d2h);
                return fail(ctx, BMC_E_DOMAIN, "friction_limit: weight-transfer denominator <= 0");
            }
            BMC_CK(ctx, cudaMemcpyAsync(s.d_terms.p, s.h_terms.p, s.len * 32, cudaMemcpyHostToDevice, ctx->h2d));
            BMC_CK(ctx, cudaEventRecord(s.h2d_done, ctx->h2d));
            BMC_CK(ctx, cudaStreamWaitEvent(s.compute, s.h2d_done, 0));
        }
        const double* dv0 = s.d_terms.as<double>();
        const bmc_terms terms{dv0, dv0 + s.len, dv0 + 2 * s.len, dv0 + 3 * s.len};
        bmc_outputs outs;
        if (host_out) {
            char* dout = s.d_out.as<char>();
            outs = bmc_outputs{reinterpret_cast<double*>(dout),
                               reinterpret_cast<int32_t*>(dout + s.len * 8),
                               reinterpret_cast<uint8_t*>(dout + s.len * 12)};
        } else {
            outs = bmc_outputs{dev_out->stop_distance ? dev_out->stop_distance + s.offset : nullptr,
                               dev_out->steps ? dev_out->steps + s.offset : nullptr,
                               dev_out->hit_horizon ? dev_out->hit_horizon + s.offset : nullptr};
        }
        rc = enqueue_rollout(ctx, plan, s.sc, terms, s.len, outs,
                             ctx->total_steps.as<unsigned long long>(), s.compute, &s.kev,
                             &launches, p1, direct);
        if (rc != BMC_OK) return rc;
        BMC_CK(ctx, cudaEventRecord(s.compute_done, s.compute));
        BMC_CK(ctx, cudaStreamWaitEvent(ctx->d2h, s.compute_done, 0));
        if (host_out) {
            // d_out holds d (8B), steps (4B), horizon (1B) blocks contiguously
            BMC_CK(ctx, cudaMemcpyAsync(s.h_out.p, s.d_out.p, s.len * 13, cudaMemcpyDeviceToHost, ctx->d2h));
        }
        BMC_CK(ctx, cudaEventRecord(s.d2h_done, ctx->d2h));
        s.busy = true;
    }
    for (uint64_t k = nchunks > kSlots ? nchunks - kSlots : 0; k < nchunks; ++k) {
        if ((rc = finish(ctx->slots[k % kSlots])) != BMC_OK) return rc;
    }
    unsigned long long steps_total = 0;
    BMC_CK(ctx, cudaMemcpy(&steps_total, ctx->total_steps.p, sizeof steps_total, cudaMemcpyDeviceToHost));
    uint64_t dev_clamps = 0;
    if (dev_draw && (rc = finish_draw(ctx, ctx->draw_ctr, &dev_clamps)) != BMC_OK) return rc;
    const double wall = std::chrono::duration<double>(Clock::now() - t0).count();
    if (trace) {
        std::fprintf(stderr,
                     "bmc pipe: n %llu chunks %llu threads %u wall %.2f ms | host: wait %.2f "
                     "unpack %.2f stage %.2f ms | device: kernel %.2f predict %.2f ms\n",
                     static_cast<unsigned long long>(n), static_cast<unsigned long long>(nchunks),
                     threads, wall * 1e3, t_wait * 1e3, t_unpack * 1e3, t_stage * 1e3, kernel_ms,
                     predict_ms);
        for (const auto& r : tl) {
            std::fprintf(stderr,
                         "  chunk %3d  bin %8.2f..%8.2f  rollout %8.2f..%8.2f (%6.2f)  unpermute ..%8.2f\n",
                         static_cast<int>(r[0]), r[1], r[2], r[3], r[4], r[4] - r[3], r[5]);
        }
    }
    if (base) cudaEventDestroy(base);
    ctx->last_launches = launches;
    if (clamp_count) *clamp_count = dev_draw ? dev_clamps : clamps.load();
    if (info) {
        info->wall_s = wall;
        info->kernel_ms = kernel_ms;
        info->predict_ms = predict_ms;
        info->total_steps = steps_total;
        info->h2d_bytes = dev_draw ? 0 : n * 32;
        info->d2h_bytes = host_out ? n * 13 : 0;
        info->launches = launches;
        info->chunks = static_cast<uint32_t>(nchunks);
    }
    return BMC_OK;
}

}  // namespace
}  // namespace bmc

using bmc::fail;

extern "C" {

int bmc_device_count(int* out) {
    try {
        int c = 0;
        const cudaError_t e = cudaGetDeviceCount(&c);
        if (e != cudaSuccess) {
            *out = 0;
            return fail(nullptr, BMC_E_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
        }
        *out = c;
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception();
    }
}

int bmc_cuda_init(int device, bmc_ctx** out) {
    try {
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
            (e = ctx->kev.create()) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&ctx->scratch_done, cudaEventDisableTiming)) != cudaSuccess) {
            return fail(nullptr, BMC_E_CUDA, std::string("context setup: ") + cudaGetErrorString(e));
        }
        for (auto& s : ctx->slots) {
            if ((e = cudaStreamCreateWithFlags(&s.compute, cudaStreamNonBlocking)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&s.h2d_done, cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&s.compute_done, cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&s.d2h_done, cudaEventDisableTiming)) != cudaSuccess ||
                (e = s.kev.create()) != cudaSuccess) {
                return fail(nullptr, BMC_E_CUDA, std::string("context events: ") + cudaGetErrorString(e));
            }
        }
        *out = ctx.release();
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception();
    }
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
        s.sc.release();
        if (s.compute) cudaStreamDestroy(s.compute);
    }
    if (ctx->stats_cache) bmc_stats_destroy(ctx->stats_cache);
    ctx->stats_cache = nullptr;
    ctx->tables.clear();
    ctx->pool.reset();
    if (ctx->scratch_done) cudaEventDestroy(ctx->scratch_done);
    for (bmc::DevBuf* b : {&ctx->total_steps, &ctx->draw_ctr, &ctx->partials,
                           &ctx->sel_hist, &ctx->sel_pref, &ctx->sorted_h, &ctx->buckets,
                           &ctx->hist_buf}) {
        b->release();
    }
    ctx->scratch.release();
    ctx->kev.destroy();
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
    if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
    delete ctx;
}

const char* bmc_cuda_last_error(const bmc_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

void* bmc_cuda_stream(bmc_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int bmc_cuda_sync(bmc_ctx* ctx) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        BMC_CK(ctx, cudaStreamSynchronize(ctx->stream));
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_rollout_device(bmc_ctx* ctx, const bmc_terms* terms, size_t n, const bmc_world* world,
                            const bmc_run_opts* opts, const bmc_outputs* out,
                            unsigned long long* total_steps_dev, void* stream) {
    try {
        return bmc_cuda_rollout_stats(ctx, terms, n, world, opts, out, total_steps_dev, nullptr, stream);
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_last_kernel_ms(bmc_ctx* ctx, float* rollout_ms, float* predict_ms) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        float r = 0.0f, p = 0.0f;
        BMC_CK(ctx, cudaEventSynchronize(ctx->kev.r1));
        BMC_CK(ctx, cudaEventElapsedTime(&r, ctx->kev.r0, ctx->kev.r1));
        if (ctx->kev.predicted) BMC_CK(ctx, cudaEventElapsedTime(&p, ctx->kev.p0, ctx->kev.p1));
        if (rollout_ms) *rollout_ms = r;
        if (predict_ms) *predict_ms = p;
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_last_stage_ms(bmc_ctx* ctx, float* bin_ms, float* rollout_ms, float* unpermute_ms) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        float b = 0.0f, r = 0.0f, u = 0.0f;
        BMC_CK(ctx, cudaEventSynchronize(ctx->kev.r1));
        BMC_CK(ctx, cudaEventElapsedTime(&r, ctx->kev.r0, ctx->kev.r1));
        if (ctx->kev.predicted) BMC_CK(ctx, cudaEventElapsedTime(&b, ctx->kev.p0, ctx->kev.p1));
        if (ctx->kev.unpermuted) {
            BMC_CK(ctx, cudaEventSynchronize(ctx->kev.u1));
            BMC_CK(ctx, cudaEventElapsedTime(&u, ctx->kev.r1, ctx->kev.u1));
        }
        if (bin_ms) *bin_ms = b;
        if (rollout_ms) *rollout_ms = r;
        if (unpermute_ms) *unpermute_ms = u;
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_last_lane_stats(bmc_ctx* ctx, uint64_t* steps, uint64_t* slots) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        unsigned long long c[2] = {0, 0};
        BMC_CK(ctx, cudaStreamSynchronize(ctx->stream));
        if (ctx->scratch.counter.p) {
            BMC_CK(ctx, cudaMemcpy(c, ctx->scratch.counter.as<char>() + 8, sizeof c, cudaMemcpyDeviceToHost));
        }
        if (steps) *steps = c[0];
        if (slots) *slots = c[1];
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_fp64_peak(bmc_ctx* ctx, int reps, double* ops_per_s, double* best_ms) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        BMC_CK(ctx, ctx->scratch.counter.reserve(64));
        double best = 1e30;
        uint64_t ops = 0;
        for (int r = 0; r < std::max(1, reps) + 1; ++r) {  // first launch is a warm-up
            BMC_CK(ctx, cudaEventRecord(ctx->kev.r0, ctx->stream));
            BMC_CK(ctx, bmc::launch_fp64_probe(ctx->scratch.counter.as<double>(), 4096, &ops, ctx->stream));
            BMC_CK(ctx, cudaEventRecord(ctx->kev.r1, ctx->stream));
            BMC_CK(ctx, cudaEventSynchronize(ctx->kev.r1));
            float ms = 0.0f;
            BMC_CK(ctx, cudaEventElapsedTime(&ms, ctx->kev.r0, ctx->kev.r1));
            if (r > 0) best = std::min(best, static_cast<double>(ms));
        }
        if (ops_per_s) *ops_per_s = static_cast<double>(ops) / (best * 1e-3);
        if (best_ms) *best_ms = best;
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_alloc(bmc_ctx* ctx, size_t bytes, void** out) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        if (!out) return fail(ctx, BMC_E_CONFIG, "bmc_cuda_alloc: null output");
        *out = nullptr;
        const cudaError_t e = cudaMalloc(out, bytes ? bytes : 1);
        if (e != cudaSuccess) return fail(ctx, BMC_E_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_free(bmc_ctx* ctx, void* ptr) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        if (ptr) BMC_CK(ctx, cudaFree(ptr));
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_copy_to_host(bmc_ctx* ctx, void* host, const void* dev, size_t bytes) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (bytes == 0) return BMC_OK;
        BMC_CK(ctx, cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        BMC_CK(ctx, cudaStreamSynchronize(ctx->stream));
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_copy_to_device(bmc_ctx* ctx, void* dev, const void* host, size_t bytes) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (bytes == 0) return BMC_OK;
        BMC_CK(ctx, cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
        BMC_CK(ctx, cudaStreamSynchronize(ctx->stream));
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_draw_device(bmc_ctx* ctx, const bmc_model* model, uint64_t first, size_t n,
                         const bmc_world* world, double* terms, bmc_sample* samples,
                         uint64_t* clamp_count) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (n == 0) return fail(ctx, BMC_E_CONFIG, "samples: must be >= 1");  // sampling.cpp:68-70
        if (!model || !world) return fail(ctx, BMC_E_CONFIG, "bmc_cuda_draw_device: null argument");
        bmc_run_opts o{};
        o.sampler = 2;
        bool dev = false;
        if ((rc = bmc::use_device_sampler(ctx, o, &dev)) != BMC_OK) return rc;
        bmc::DrawArgs a = bmc::draw_args(*model, first, n, *world);
        if (terms) {
            a.v0 = terms;
            a.brake_floor = terms + n;
            a.drag = terms + 2 * n;
            a.grade = terms + 3 * n;
        }
        a.samples = reinterpret_cast<double*>(samples);
        BMC_CK(ctx, ctx->draw_ctr.reserve(16));
        BMC_CK(ctx, cudaMemsetAsync(ctx->draw_ctr.p, 0, 16, ctx->stream));
        a.clamps = ctx->draw_ctr.as<unsigned long long>();
        a.flags = reinterpret_cast<unsigned int*>(ctx->draw_ctr.as<char>() + 8);
        BMC_CK(ctx, bmc::launch_draw_terms(a, ctx->sms, ctx->stream));
        ctx->last_launches = 1;
        return bmc::finish_draw(ctx, ctx->draw_ctr, clamp_count);
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_last_launches(bmc_ctx* ctx, uint32_t* launches) {
    try {
        if (!ctx || !launches) return BMC_E_CONFIG;
        *launches = ctx->last_launches;
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_run(bmc_ctx* ctx, const bmc_sample* samples, size_t n, const bmc_world* world,
                 const bmc_run_opts* opts, bmc_result* out, bmc_run_info* info) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (n == 0) return fail(ctx, BMC_E_CONFIG, "batch: must be non-empty");  // backends.cpp:41-43
        if (!samples || !world || !out) return fail(ctx, BMC_E_CONFIG, "bmc_cuda_run: null argument");
        bmc::WorldDerived d{};
        std::string err;
        if ((rc = bmc::derive_world(*world, &d, &err)) != BMC_OK) return fail(ctx, rc, err);
        const bmc_run_opts o = opts ? *opts : bmc_run_opts{};
        return bmc::run_pipeline(ctx, *world, d, o, n, samples, nullptr, 0, out, nullptr, info, nullptr);
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_run_model(bmc_ctx* ctx, const bmc_model* model, uint64_t first, size_t n,
                       const bmc_world* world, const bmc_run_opts* opts, bmc_result* host_out,
                       const bmc_outputs* dev_out, uint64_t* clamp_count, bmc_run_info* info) {
    try {
        return bmc_cuda_run_model_stats(ctx, model, first, n, world, opts, host_out, dev_out,
                                        clamp_count, info, nullptr);
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_run_model_stats(bmc_ctx* ctx, const bmc_model* model, uint64_t first, size_t n,
                             const bmc_world* world, const bmc_run_opts* opts, bmc_result* host_out,
                             const bmc_outputs* dev_out, uint64_t* clamp_count, bmc_run_info* info,
                             bmc_stats_stage* st) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (n == 0) return fail(ctx, BMC_E_CONFIG, "samples: must be >= 1");  // sampling.cpp:68-70
        if (!model || !world) return fail(ctx, BMC_E_CONFIG, "bmc_cuda_run_model: null argument");
        if ((host_out == nullptr) == (dev_out == nullptr)) {
            return fail(ctx, BMC_E_CONFIG, "bmc_cuda_run_model: exactly one of host_out / dev_out");
        }
        bmc::WorldDerived d{};
        std::string err;
        if ((rc = bmc::derive_world(*world, &d, &err)) != BMC_OK) return fail(ctx, rc, err);
        const bmc_run_opts o = opts ? *opts : bmc_run_opts{};
        bmc::P1Args p1{};
        if (st) {
            if (!bmc::stats_p1_args(st, &p1)) {
                return fail(ctx, BMC_E_RANGE, "risk.headways: at most 4096 when fused into a streamed run");
            }
            if (bmc::stats_max_n(st) < n) {
                return fail(ctx, BMC_E_CONFIG, "stats: more results than the stage was sized for");
            }
        }
        // chunks run on the slot streams; the stage was begun on ctx->stream,
        // which run_pipeline synchronises before the first chunk
        return bmc::run_pipeline(ctx, *world, d, o, n, nullptr, model, first, host_out, dev_out, info,
                                 clamp_count, st ? &p1 : nullptr);
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

}  // extern "C"
