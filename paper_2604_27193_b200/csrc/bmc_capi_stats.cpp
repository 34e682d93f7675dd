// bmc_capi_stats.cpp -- C-ABI of the on-device statistics (brakemc_cuda.h).
//
// The fused statistics stage (bmc_stats_stage): the DeviceBackend below runs
// the stages of bmc_stats_pipeline.h as sm_100a kernels (bmc_fused_stats.cu)
// on one stream; pass 1 is fused into the rollout epilogue
// (bmc_cuda_rollout_stats).  The legacy building blocks (exceedance, order
// statistics by 8-bit radix select, partials, moments, histogram) stay for
// callers that want one quantity.  The O(#blocks) / O(#bins) host
// composition uses the reference's own formulas (analysis.cpp:13-76,
// 145-194).  g++ -ffp-contract=off.
#include "bmc_ctx.h"
#include "bmc_stats_pipeline.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <vector>

namespace bmc {
namespace {

struct DDh {
    double hi = 0.0, lo = 0.0;
};

DDh dd_merge_h(DDh a, double b_hi, double b_lo) {
    const double s = a.hi + b_hi;
    const double bb = s - a.hi;
    const double err = (a.hi - (s - bb)) + (b_hi - bb);
    return DDh{s, a.lo + err + b_lo};
}


double value_of_key(uint64_t k) {
    const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    double v;
    std::memcpy(&v, &b, 8);
    return v;
}

// Exact k-th smallest (1-based ranks) by 8 passes of 8-bit radix select.
int select_ranks(bmc_ctx* ctx, const double* d, const uint8_t* hz, uint64_t n, int exclude,
                 const uint64_t* ranks, size_t m, double* out, uint64_t* count_out) {
    cudaStream_t s = ctx->stream;
    std::vector<uint64_t> prefix(m, 0), residual(ranks, ranks + m);
    std::vector<char> valid(m, 1);
    std::vector<unsigned long long> hist(m * 256);
    uint64_t count = 0;
    BMC_CK(ctx, ctx->sel_pref.reserve(kMaxSelectTargets * sizeof(uint64_t)));
    BMC_CK(ctx, ctx->sel_hist.reserve(kMaxSelectTargets * 256 * sizeof(unsigned long long)));
    for (size_t t0 = 0; t0 < m; t0 += kMaxSelectTargets) {
        const size_t tm = std::min<size_t>(kMaxSelectTargets, m - t0);
        for (int shift = 56; shift >= 0; shift -= 8) {
            BMC_CK(ctx, cudaMemcpyAsync(ctx->sel_pref.p, prefix.data() + t0, tm * sizeof(uint64_t),
                                        cudaMemcpyHostToDevice, s));
            BMC_CK(ctx, cudaMemsetAsync(ctx->sel_hist.p, 0, tm * 256 * sizeof(unsigned long long), s));
            BMC_CK(ctx, launch_select(d, hz, n, exclude, shift, ctx->sel_pref.as<uint64_t>(),
                                      static_cast<int>(tm), ctx->sel_hist.as<unsigned long long>(), s));
            BMC_CK(ctx, cudaMemcpyAsync(hist.data(), ctx->sel_hist.p, tm * 256 * sizeof(unsigned long long),
                                        cudaMemcpyDeviceToHost, s));
            BMC_CK(ctx, cudaStreamSynchronize(s));
            ctx->last_launches += 1;
            if (shift == 56) {
                count = 0;
                for (int b = 0; b < 256; ++b) count += hist[b];
                for (size_t t = 0; t < tm; ++t) {
                    if (residual[t0 + t] < 1 || residual[t0 + t] > count) valid[t0 + t] = 0;
                }
            }
            for (size_t t = 0; t < tm; ++t) {
                if (!valid[t0 + t]) continue;
                uint64_t cum = 0;
                int digit = 255;
                for (int b = 0; b < 256; ++b) {
                    const uint64_t c = hist[t * 256 + b];
                    if (cum + c >= residual[t0 + t]) {
                        digit = b;
                        break;
                    }
                    cum += c;
                }
                residual[t0 + t] -= cum;
                prefix[t0 + t] |= static_cast<uint64_t>(digit) << shift;
            }
        }
    }
    for (size_t t = 0; t < m; ++t) {
        out[t] = valid[t] ? value_of_key(prefix[t]) : std::numeric_limits<double>::quiet_NaN();
    }
    if (count_out) *count_out = count;
    return BMC_OK;
}

}  // namespace
}  // namespace bmc

using bmc::fail;

// ====================================================================
// Fused statistics stage
// ====================================================================

struct bmc_stats_stage {
    bmc_ctx* ctx = nullptr;
    bmc::StatsConfig cfg;
    bmc::StatsLayout L{};
    bmc::DevBuf mem, gather;
    bmc::PinBuf mirror;  // host copy of the stage words the composition reads
    size_t max_n = 0;
    bool exceed_pending = false;  // headways not accumulated by the last P1 producer
    uint32_t launches = 0;

    bmc::StageDev dev() const {
        bmc::StageDev g{};
        g.w = mem.as<unsigned long long>();
        g.p1_min = L.p1_min;
        g.p1_sum = L.p1_sum;
        g.p2_sum = L.p2_sum;
        g.cand_count = L.cand_count;
        g.scal = L.scal;
        g.targets = L.targets;
        g.risks = L.risks;
        g.cand = L.cand;
        g.m = cfg.m();
        g.n_risk = cfg.n_risk();
        g.n_targets = cfg.n_targets();
        g.summary = cfg.summary ? 1 : 0;
        g.hist_cap = cfg.hist_cap;
        g.cand_cap = cfg.cand_cap;
        g.bin_width = cfg.bin_width;
        return g;
    }
    // pass-1 words for a producer; exceedance fused when the headways fit
    bmc::P1Args p1(bool with_exceed) const {
        bmc::P1Args a{};
        a.sum = mem.as<unsigned long long>() + L.p1_sum;
        a.minw = mem.as<unsigned long long>() + L.p1_min;
        a.H = reinterpret_cast<const double*>(mem.as<unsigned long long>() + L.headways);
        a.m = with_exceed ? cfg.m() : 0;
        return a;
    }
};

namespace bmc {
namespace {

constexpr size_t kSmemOptin = 232448;  // 227 KB per CTA (sm_100)

struct DeviceBackend {
    bmc_stats_stage* st;
    cudaStream_t s;

    bmc_ctx* ctx() const { return st->ctx; }
    uint64_t* words(size_t off) {
        if (off >= st->L.gather) return st->gather.as<uint64_t>() + (off - st->L.gather);
        return st->mem.as<uint64_t>() + off;
    }
    int ensure_gather(size_t w) {
        BMC_CK(ctx(), st->gather.reserve(std::max<size_t>(w, 16) * 8));
        return BMC_OK;
    }
    int normalize(size_t off, int accs) {
        BMC_CK(ctx(), launch_normalize(st->dev(), off, accs, s));
        ++st->launches;
        return BMC_OK;
    }
    int finalize1() {
        BMC_CK(ctx(), launch_finalize1(st->dev(), s));
        ++st->launches;
        return BMC_OK;
    }
    int pass2(const double* d, const uint8_t* hz, uint64_t n) {
        if (n == 0) return BMC_OK;
        BMC_CK(ctx(), launch_pass2(d, hz, n, st->dev(), ctx()->sms, s));
        ++st->launches;
        return BMC_OK;
    }
    int targets() {
        BMC_CK(ctx(), launch_targets(st->dev(), s));
        ++st->launches;
        return BMC_OK;
    }
    int compact(const double* d, const uint8_t* hz, uint64_t n) {
        if (n == 0) return BMC_OK;
        BMC_CK(ctx(), launch_compact(d, hz, n, st->dev(), ctx()->sms, s));
        ++st->launches;
        return BMC_OK;
    }
    int pack(const uint64_t* P, const uint64_t* off, uint64_t total) {
        PackArgs p{};
        for (int t = 0; t < sc::kMaxTargets; ++t) p.off[t] = t < st->cfg.n_targets() ? off[t] : total;
        p.total = total;
        (void)P;
        if (total == 0) return BMC_OK;
        BMC_CK(ctx(), launch_pack(st->dev(), p, st->gather.as<unsigned long long>(), ctx()->sms, s));
        ++st->launches;
        return BMC_OK;
    }
    int mark_overflow(const bool* over) {
        sc::Target tg[sc::kMaxTargets];
        int rc = read(tg, st->L.targets, sizeof tg / 8);
        if (rc != BMC_OK) return rc;
        bool any = false;
        for (int t = 0; t < st->cfg.n_targets(); ++t) {
            if (over[t]) {
                tg[t].overflow = 1;
                any = true;
            }
        }
        return any ? write(st->L.targets, tg, sizeof tg / 8) : BMC_OK;
    }
    int select(const SelectSegments& seg) {
        const unsigned long long* keys =
            seg.in_gather ? st->gather.as<unsigned long long>() : st->mem.as<unsigned long long>();
        BMC_CK(ctx(), launch_select_targets(st->dev(), seg, keys, s));
        ++st->launches;
        return BMC_OK;
    }
    int read(void* host, size_t off, size_t w) {
        if (w == 0) return BMC_OK;
        BMC_CK(ctx(), cudaMemcpyAsync(host, words(off), w * 8, cudaMemcpyDeviceToHost, s));
        BMC_CK(ctx(), cudaStreamSynchronize(s));
        return BMC_OK;
    }
    int write(size_t off, const void* host, size_t w) {
        if (w == 0) return BMC_OK;
        BMC_CK(ctx(), cudaMemcpyAsync(words(off), host, w * 8, cudaMemcpyHostToDevice, s));
        BMC_CK(ctx(), cudaStreamSynchronize(s));
        return BMC_OK;
    }
    int snapshot(size_t w, const uint64_t** host) {
        BMC_CK(ctx(), st->mirror.reserve(w * 8));
        BMC_CK(ctx(), cudaMemcpyAsync(st->mirror.p, st->mem.p, w * 8, cudaMemcpyDeviceToHost, s));
        BMC_CK(ctx(), cudaStreamSynchronize(s));
        *host = st->mirror.as<uint64_t>();
        return BMC_OK;
    }
    // exact fallbacks (degenerate data only)
    int hist_full(const double* d, uint64_t n, double lo, double bw, uint64_t bins, uint64_t* out) {
        bmc_ctx* c = ctx();
        BMC_CK(c, c->hist_buf.reserve(bins * sizeof(unsigned long long)));
        BMC_CK(c, cudaMemsetAsync(c->hist_buf.p, 0, bins * sizeof(unsigned long long), s));
        if (n) {
            BMC_CK(c, launch_hist(d, n, lo, bw, bins, c->hist_buf.as<unsigned long long>(), s));
            ++st->launches;
        }
        BMC_CK(c, cudaMemcpyAsync(out, c->hist_buf.p, bins * 8, cudaMemcpyDeviceToHost, s));
        BMC_CK(c, cudaStreamSynchronize(s));
        return BMC_OK;
    }
    int select_pass(const double* d, const uint8_t* hz, uint64_t n, int exclude, int shift,
                    const uint64_t* prefixes, size_t m, uint64_t* hist) {
        bmc_ctx* c = ctx();
        BMC_CK(c, c->sel_pref.reserve(kMaxSelectTargets * sizeof(uint64_t)));
        BMC_CK(c, c->sel_hist.reserve(kMaxSelectTargets * 256 * sizeof(unsigned long long)));
        BMC_CK(c, cudaMemcpyAsync(c->sel_pref.p, prefixes, m * 8, cudaMemcpyHostToDevice, s));
        BMC_CK(c, cudaMemsetAsync(c->sel_hist.p, 0, m * 256 * 8, s));
        if (n) {
            BMC_CK(c, launch_select(d, hz, n, exclude, shift, c->sel_pref.as<uint64_t>(),
                                    static_cast<int>(m), c->sel_hist.as<unsigned long long>(), s));
            ++st->launches;
        }
        BMC_CK(c, cudaMemcpyAsync(hist, c->sel_hist.p, m * 256 * 8, cudaMemcpyDeviceToHost, s));
        BMC_CK(c, cudaStreamSynchronize(s));
        return BMC_OK;
    }
};

cudaStream_t stream_of(bmc_stats_stage* st, void* stream) {
    return stream ? static_cast<cudaStream_t>(stream) : st->ctx->stream;
}

int stage_begin(bmc_stats_stage* st, cudaStream_t s) {
    bmc_ctx* ctx = st->ctx;
    unsigned long long* w = st->mem.as<unsigned long long>();
    BMC_CK(ctx, cudaMemsetAsync(w + st->L.p1_min, 0xFF, sc::kP1MinWords * 8, s));
    BMC_CK(ctx, cudaMemsetAsync(w + st->L.zero_begin, 0,
                                (st->L.zero_end - st->L.zero_begin) * 8, s));
    st->exceed_pending = false;
    st->launches = 0;
    return BMC_OK;
}

int stage_accumulate(bmc_stats_stage* st, const double* d, const uint8_t* hz, uint64_t n,
                     cudaStream_t s) {
    bmc_ctx* ctx = st->ctx;
    if (n == 0) return BMC_OK;
    const bool fuse_exceed = static_cast<size_t>(st->cfg.m()) <= kMaxFusedHeadways;
    BMC_CK(ctx, launch_pass1(d, hz, n, st->p1(fuse_exceed), ctx->sms, s));
    ++st->launches;
    if (!fuse_exceed) {
        BMC_CK(ctx, launch_exceed(d, hz, n, st->p1(true).H, st->cfg.m(),
                                  st->mem.as<unsigned long long>() + st->L.p1_sum + sc::kP1Exceed, s));
        ++st->launches;
    }
    return BMC_OK;
}

int stage_finish(bmc_stats_stage* st, const double* d, const uint8_t* hz, uint64_t n,
                 const bmc_merge* merge, bmc_stats* out, cudaStream_t s) {
    bmc_ctx* ctx = st->ctx;
    if (st->exceed_pending) {
        if (!d) return fail(ctx, BMC_E_CONFIG, "stats: headway grid too large to fuse; needs outputs");
        if (n) {
            BMC_CK(ctx, launch_exceed(d, hz, n, st->p1(true).H, st->cfg.m(),
                                      st->mem.as<unsigned long long>() + st->L.p1_sum + sc::kP1Exceed, s));
            ++st->launches;
        }
        st->exceed_pending = false;
    }
    if (merge && (!merge->allreduce_u64 || !merge->allgather_u64 || merge->world < 1)) {
        return fail(ctx, BMC_E_CONFIG, "stats: merge needs allreduce_u64, allgather_u64 and world >= 1");
    }
    DeviceBackend be{st, s};
    std::string err;
    uint32_t launches = 0;
    const int rc = stats_finish(be, st->cfg, st->L, d, hz, n, merge, out, s, &launches, &err);
    if (rc != BMC_OK) return fail(ctx, rc, err.empty() ? ctx->err : err);
    out->launches = st->launches;
    ctx->last_launches = st->launches;
    return BMC_OK;
}

bool same_config(const StatsConfig& a, const StatsConfig& b) {
    return a.headways == b.headways && a.order == b.order && a.risks == b.risks &&
           a.summary == b.summary && a.bin_width == b.bin_width && a.hist_cap == b.hist_cap &&
           a.cand_cap == b.cand_cap;
}

int stage_create(bmc_ctx* ctx, const bmc_stats_req* req, size_t max_n, bmc_stats_stage** out) {
    auto st = std::make_unique<bmc_stats_stage>();
    st->ctx = ctx;
    std::string err;
    int rc = resolve_request(req, max_n, &st->cfg, &err);
    if (rc != BMC_OK) return fail(ctx, rc, err);
    st->L = make_layout(st->cfg);
    st->max_n = max_n;
    BMC_CK(ctx, st->mem.reserve(st->L.total * 8));
    // every word defined (the read-back snapshot copies whole regions)
    BMC_CK(ctx, cudaMemsetAsync(st->mem.p, 0, st->L.total * 8, ctx->stream));
    std::vector<uint64_t> consts(st->L.cand - st->L.headways, 0);
    if (st->cfg.m()) std::memcpy(consts.data(), st->cfg.headways.data(), st->cfg.headways.size() * 8);
    if (st->cfg.n_risk()) {
        std::memcpy(consts.data() + (st->L.risks - st->L.headways), st->cfg.risks.data(),
                    st->cfg.risks.size() * 8);
    }
    BMC_CK(ctx, cudaMemcpyAsync(st->mem.as<uint64_t>() + st->L.headways, consts.data(),
                                consts.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    BMC_CK(ctx, cudaStreamSynchronize(ctx->stream));
    *out = st.release();
    return BMC_OK;
}

}  // namespace

// ---- pieces a CUDA graph captures (bmc_graph.cpp)
int stats_stage_create(bmc_ctx* ctx, const bmc_stats_req* req, size_t max_n, bmc_stats_stage** out) {
    return stage_create(ctx, req, max_n, out);
}
int stats_begin_enqueue(bmc_stats_stage* st, cudaStream_t s) { return stage_begin(st, s); }
bool stats_p1_args(bmc_stats_stage* st, P1Args* p1) {
    const bool fuse = static_cast<size_t>(st->cfg.m()) <= kMaxFusedHeadways;
    *p1 = st->p1(fuse);
    return fuse;
}
void fit_stats_plan(Plan* plan, const P1Args& p1) {
    // the table and the partials share the CTA's shared memory
    if (plan->mode == kTableShared &&
        static_cast<size_t>(plan->table_len) * sizeof(StageA) + p1_smem_bytes(p1.m) > kSmemOptin) {
        plan->mode = kTableGlobal;
    }
}
int stats_enqueue_device(bmc_stats_stage* st, const double* d, const uint8_t* hz, uint64_t n,
                         cudaStream_t s) {
    DeviceBackend be{st, s};
    std::string err;
    const int rc = stats_device_stages(be, st->cfg, st->L, d, hz, n, nullptr, s, &err);
    return rc == BMC_OK ? rc : fail(st->ctx, rc, err.empty() ? st->ctx->err : err);
}
size_t stats_mirror_words(const bmc_stats_stage* st) { return st->L.cand; }
int stats_enqueue_readback(bmc_stats_stage* st, uint64_t* mirror, cudaStream_t s) {
    for (const ReadRegion& r : readback_regions(st->cfg, st->L)) {
        BMC_CK(st->ctx, cudaMemcpyAsync(mirror + r.off, st->mem.as<uint64_t>() + r.off, r.words * 8,
                                        cudaMemcpyDeviceToHost, s));
    }
    return BMC_OK;
}
int stats_compose_mirror(bmc_stats_stage* st, const uint64_t* mirror, const double* d,
                         const uint8_t* hz, uint64_t n, bmc_stats* out) {
    StatsReadback rb;
    int rc = stats_read(
        [&](void* h, size_t off, size_t w) {
            std::memcpy(h, mirror + off, w * 8);
            return BMC_OK;
        },
        st->cfg, st->L, &rb);
    if (rc != BMC_OK) return rc;
    DeviceBackend be{st, st->ctx->stream};
    std::string err;
    rc = stats_compose(be, st->cfg, st->L, rb, d, hz, n, nullptr, out, st->ctx->stream, &err);
    if (rc != BMC_OK) return fail(st->ctx, rc, err);
    return BMC_OK;
}
uint32_t stats_launches(const bmc_stats_stage* st) { return st->launches; }
size_t stats_max_n(const bmc_stats_stage* st) { return st->max_n; }

}  // namespace bmc

extern "C" {

int bmc_stats_create(bmc_ctx* ctx, const bmc_stats_req* req, size_t max_n, bmc_stats_stage** out) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (!out) return fail(ctx, BMC_E_CONFIG, "bmc_stats_create: null output");
        *out = nullptr;
        return bmc::stage_create(ctx, req, max_n, out);
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

void bmc_stats_destroy(bmc_stats_stage* st) {
    if (!st) return;
    cudaSetDevice(st->ctx->device);
    cudaDeviceSynchronize();
    st->mem.release();
    st->gather.release();
    st->mirror.release();
    delete st;
}

int bmc_stats_begin(bmc_stats_stage* st, void* stream) {
    try {
        if (!st) return fail(nullptr, BMC_E_CONFIG, "bmc_stats_begin: null stage");
        int rc = bmc::prepare(st->ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(st->ctx->mu);
        return bmc::stage_begin(st, bmc::stream_of(st, stream));
    } catch (...) {
        return bmc::abi_exception();
    }
}

int bmc_stats_accumulate(bmc_stats_stage* st, const double* d, const uint8_t* hz, size_t n,
                         void* stream) {
    try {
        if (!st) return fail(nullptr, BMC_E_CONFIG, "bmc_stats_accumulate: null stage");
        int rc = bmc::prepare(st->ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(st->ctx->mu);
        if (n && !d) return fail(st->ctx, BMC_E_CONFIG, "bmc_stats_accumulate: null outputs");
        if (n > st->max_n) return fail(st->ctx, BMC_E_CONFIG, "stats: more results than the stage was sized for");
        return bmc::stage_accumulate(st, d, hz, n, bmc::stream_of(st, stream));
    } catch (...) {
        return bmc::abi_exception();
    }
}

int bmc_stats_finish(bmc_stats_stage* st, const double* d, const uint8_t* hz, size_t n,
                     const bmc_merge* merge, bmc_stats* out, void* stream) {
    try {
        if (!st || !out) return fail(st ? st->ctx : nullptr, BMC_E_CONFIG, "bmc_stats_finish: null argument");
        int rc = bmc::prepare(st->ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(st->ctx->mu);
        if (n && !d) return fail(st->ctx, BMC_E_CONFIG, "bmc_stats_finish: null outputs");
        if (n > st->max_n) return fail(st->ctx, BMC_E_CONFIG, "stats: more results than the stage was sized for");
        return bmc::stage_finish(st, d, hz, n, merge, out, bmc::stream_of(st, stream));
    } catch (...) {
        return bmc::abi_exception();
    }
}

int bmc_cuda_stats(bmc_ctx* ctx, const double* d, const uint8_t* hz, size_t n,
                   const bmc_stats_req* req, bmc_stats* out) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        if (!out) return fail(ctx, BMC_E_CONFIG, "bmc_cuda_stats: null output");
        if (n == 0) {
            return fail(ctx, BMC_E_CONFIG, req && req->summarize ? "summarize: needs at least one result"
                                                                 : "risk: needs at least one result");
        }
        if (!d) return fail(ctx, BMC_E_CONFIG, "bmc_cuda_stats: null outputs");
        std::lock_guard<std::mutex> lk(ctx->mu);
        // reuse the context's cached stage when the resolved request (and so the
        // layout and candidate capacity) is the same; the stage's memory is
        // allocated once per request shape, not per call
        bmc::StatsConfig cfg;
        std::string err;
        if ((rc = bmc::resolve_request(req, n, &cfg, &err)) != BMC_OK) return fail(ctx, rc, err);
        bmc_stats_stage* st = ctx->stats_cache;
        if (!st || !bmc::same_config(st->cfg, cfg) || st->max_n < n) {
            if (st) bmc_stats_destroy(st);
            ctx->stats_cache = nullptr;
            if ((rc = bmc::stage_create(ctx, req, n, &st)) != BMC_OK) return rc;
            ctx->stats_cache = st;
        }
        cudaStream_t s = ctx->stream;
        if (ctx->scratch_used) BMC_CK(ctx, cudaStreamWaitEvent(s, ctx->scratch_done, 0));
        if ((rc = bmc::stage_begin(st, s)) != BMC_OK) return rc;
        if ((rc = bmc::stage_accumulate(st, d, hz, n, s)) != BMC_OK) return rc;
        return bmc::stage_finish(st, d, hz, n, nullptr, out, s);
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_rollout_stats(bmc_ctx* ctx, const bmc_terms* terms, size_t n, const bmc_world* world,
                           const bmc_run_opts* opts, const bmc_outputs* out,
                           unsigned long long* total_steps_dev, bmc_stats_stage* st, void* stream) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (!terms || !world || !out) return fail(ctx, BMC_E_CONFIG, "bmc_cuda_rollout_device: null argument");
        if (n == 0) return fail(ctx, BMC_E_CONFIG, "batch: must be non-empty");
        if (st && st->ctx != ctx) return fail(ctx, BMC_E_CONFIG, "stats: stage belongs to another context");
        if (st && n > st->max_n) return fail(ctx, BMC_E_CONFIG, "stats: more results than the stage was sized for");
        bmc::WorldDerived d{};
        std::string err;
        if ((rc = bmc::derive_world(*world, &d, &err)) != BMC_OK) return fail(ctx, rc, err);
        const bmc_run_opts o = opts ? *opts : bmc_run_opts{};
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
        bmc::Plan plan;
        if ((rc = bmc::make_plan(ctx, d, o, n, &plan)) != BMC_OK) return rc;
        bmc::P1Args p1{};
        if (st) {
            st->exceed_pending = !bmc::stats_p1_args(st, &p1);
            bmc::fit_stats_plan(&plan, p1);
        }
        ctx->last_launches = 0;
        if (ctx->scratch_used) BMC_CK(ctx, cudaStreamWaitEvent(s, ctx->scratch_done, 0));
        rc = bmc::enqueue_rollout(ctx, plan, ctx->scratch, *terms, n, *out, total_steps_dev, s, &ctx->kev,
                                  &ctx->last_launches, st ? &p1 : nullptr);
        BMC_CK(ctx, cudaEventRecord(ctx->scratch_done, s));
        ctx->scratch_used = true;
        return rc;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

}  // extern "C"

extern "C" {

int bmc_cuda_order_stats(bmc_ctx* ctx, const double* d, const uint8_t* hz, size_t n,
                         int exclude_horizon, const uint64_t* ranks, size_t m, double* out,
                         uint64_t* count_out) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if ((rc = bmc::order_after_rollouts(ctx)) != BMC_OK) return rc;
        if (!d || (m && (!ranks || !out))) return fail(ctx, BMC_E_CONFIG, "order_stats: null argument");
        if (exclude_horizon && !hz) return fail(ctx, BMC_E_CONFIG, "order_stats: horizon flags required");
        ctx->last_launches = 0;
        if (n == 0) return fail(ctx, BMC_E_CONFIG, "risk: needs at least one result");
        return bmc::select_ranks(ctx, d, hz, n, exclude_horizon, ranks, m, out, count_out);
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_summarize(bmc_ctx* ctx, const double* d, const uint8_t* hz, size_t n, double bin_width,
                       bmc_summary* out, uint64_t* hist, size_t hist_cap) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        // analysis.cpp:14-19
        if (n == 0) return fail(ctx, BMC_E_CONFIG, "summarize: needs at least one result");
        if (!(bin_width > 0.0)) return fail(ctx, BMC_E_CONFIG, "outputs.bin_width: must be > 0");
        if (!d || !out) return fail(ctx, BMC_E_CONFIG, "summarize: null argument");
        bmc_stats_req req{};
        req.summarize = 1;
        req.bin_width = bin_width;
        bmc_stats st{};
        st.histogram = hist;
        st.histogram_cap = hist ? hist_cap : 0;
        rc = bmc_cuda_stats(ctx, d, hz, n, &req, &st);
        if (rc == BMC_OK || rc == BMC_E_RANGE) *out = st.summary;
        return rc;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_exceedance_ttc_noise(bmc_ctx* ctx, const double* d, const uint8_t* hz, size_t n,
                                  uint64_t first, uint64_t noise_seed, double sigma,
                                  const double* ttc, size_t m, double closing_speed,
                                  uint64_t* counts) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if ((rc = bmc::order_after_rollouts(ctx)) != BMC_OK) return rc;
        if (n == 0) return fail(ctx, BMC_E_CONFIG, "risk: needs at least one result");
        if (m == 0) return BMC_OK;
        if (!d || !ttc || !counts) return fail(ctx, BMC_E_CONFIG, "exceedance: null argument");
        if (!(closing_speed > 0.0)) return fail(ctx, BMC_E_CONFIG, "risk.closing_speed: must be > 0");
        if (!(sigma >= 0.0) || !std::isfinite(sigma)) {
            return fail(ctx, BMC_E_CONFIG, "risk.sensor_noise: must be finite and >= 0");
        }
        if (m > static_cast<size_t>(bmc::kNoiseMaxThresholds)) {
            return fail(ctx, BMC_E_RANGE, "risk.ttc: at most 1024 thresholds");
        }
        for (size_t j = 0; j < m; ++j) {
            if (!std::isfinite(ttc[j])) return fail(ctx, BMC_E_CONFIG, "risk.ttc: must be finite");
        }
        std::string why;
        if (!bmc::device_sampler_supported(&why)) {
            return fail(ctx, BMC_E_CONFIG, "risk.sensor_noise: " + why);
        }
        ctx->last_launches = 0;
        std::vector<size_t> order(m);
        std::iota(order.begin(), order.end(), size_t{0});
        std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return ttc[a] < ttc[b]; });
        std::vector<double> sorted(m);
        for (size_t j = 0; j < m; ++j) sorted[j] = ttc[order[j]];
        cudaStream_t s = ctx->stream;
        BMC_CK(ctx, ctx->sorted_h.reserve(m * sizeof(double)));
        BMC_CK(ctx, ctx->buckets.reserve((m + 1) * sizeof(unsigned long long)));
        BMC_CK(ctx, ctx->draw_ctr.reserve(16));
        BMC_CK(ctx, cudaMemcpyAsync(ctx->sorted_h.p, sorted.data(), m * sizeof(double), cudaMemcpyHostToDevice, s));
        BMC_CK(ctx, cudaMemsetAsync(ctx->buckets.p, 0, (m + 1) * sizeof(unsigned long long), s));
        BMC_CK(ctx, cudaMemsetAsync(ctx->draw_ctr.p, 0, 16, s));
        bmc::NoiseExceedArgs a{};
        a.d = d;
        a.hz = hz;
        a.n = n;
        a.first = first;
        a.seed = noise_seed;
        a.sigma = sigma;
        a.closing = closing_speed;
        a.ttc = ctx->sorted_h.as<double>();
        a.m = static_cast<int>(m);
        a.buckets = ctx->buckets.as<unsigned long long>();
        a.flags = reinterpret_cast<unsigned int*>(ctx->draw_ctr.as<char>() + 8);
        BMC_CK(ctx, bmc::launch_noise_exceed(a, ctx->sms, s));
        std::vector<unsigned long long> b(m + 1);
        BMC_CK(ctx, cudaMemcpyAsync(b.data(), ctx->buckets.p, (m + 1) * sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, s));
        if ((rc = bmc::finish_draw(ctx, ctx->draw_ctr, nullptr)) != BMC_OK) return rc;  // syncs s
        ctx->last_launches = 1;
        uint64_t suffix = 0;
        std::vector<uint64_t> ex(m);
        for (size_t j = m; j-- > 0;) {
            suffix += b[j + 1];
            ex[j] = suffix;
        }
        for (size_t j = 0; j < m; ++j) counts[order[j]] = ex[j];
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_exceedance(bmc_ctx* ctx, const double* d, const uint8_t* hz, size_t n,
                        const double* headways, size_t m, uint64_t* counts) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if ((rc = bmc::order_after_rollouts(ctx)) != BMC_OK) return rc;
        if (n == 0) return fail(ctx, BMC_E_CONFIG, "risk: needs at least one result");
        if (m == 0) return BMC_OK;
        if (!d || !headways || !counts) return fail(ctx, BMC_E_CONFIG, "exceedance: null argument");
        for (size_t j = 0; j < m; ++j) {
            if (!(headways[j] >= 0.0)) return fail(ctx, BMC_E_CONFIG, "risk.headway: must be >= 0");
        }
        if (m > (size_t{1} << 30)) return fail(ctx, BMC_E_RANGE, "exceedance: too many headways");
        ctx->last_launches = 0;
        std::vector<size_t> order(m);
        std::iota(order.begin(), order.end(), size_t{0});
        std::stable_sort(order.begin(), order.end(),
                         [&](size_t a, size_t b) { return headways[a] < headways[b]; });
        std::vector<double> sorted(m);
        for (size_t j = 0; j < m; ++j) sorted[j] = headways[order[j]];
        cudaStream_t s = ctx->stream;
        BMC_CK(ctx, ctx->sorted_h.reserve(m * sizeof(double)));
        BMC_CK(ctx, ctx->buckets.reserve((m + 1) * sizeof(unsigned long long)));
        BMC_CK(ctx, cudaMemcpyAsync(ctx->sorted_h.p, sorted.data(), m * sizeof(double), cudaMemcpyHostToDevice, s));
        BMC_CK(ctx, cudaMemsetAsync(ctx->buckets.p, 0, (m + 1) * sizeof(unsigned long long), s));
        BMC_CK(ctx, bmc::launch_exceed(d, hz, n, ctx->sorted_h.as<double>(), static_cast<int>(m),
                                       ctx->buckets.as<unsigned long long>(), s));
        std::vector<unsigned long long> b(m + 1);
        BMC_CK(ctx, cudaMemcpyAsync(b.data(), ctx->buckets.p, (m + 1) * sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, s));
        BMC_CK(ctx, cudaStreamSynchronize(s));
        ctx->last_launches = 1;
        // exceed(sorted j) = #{p > j} = suffix sum of buckets (j+1 .. m)
        uint64_t suffix = 0;
        std::vector<uint64_t> ex(m);
        for (size_t j = m; j-- > 0;) {
            suffix += b[j + 1];
            ex[j] = suffix;
        }
        for (size_t j = 0; j < m; ++j) counts[order[j]] = ex[j];
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

// ----------------------------------------------------------------------
// Mergeable building blocks: every output below is exactly additive (counts)
// or exactly mergeable (min/max, double-double sums) across shards, so a
// multi-GPU run combines them with one allreduce per quantity.

int bmc_cuda_partials(bmc_ctx* ctx, const double* d, const uint8_t* hz, size_t n,
                      bmc_partials* out) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if ((rc = bmc::order_after_rollouts(ctx)) != BMC_OK) return rc;
        if (!d || !out) return fail(ctx, BMC_E_CONFIG, "partials: null argument");
        bmc_partials p;
        std::memset(&p, 0, sizeof p);
        p.min = std::numeric_limits<double>::infinity();
        p.max = -std::numeric_limits<double>::infinity();
        ctx->last_launches = 0;
        if (n > 0) {
            cudaStream_t s = ctx->stream;
            const int P = bmc::stats_partials(n);
            BMC_CK(ctx, ctx->partials.reserve(static_cast<size_t>(P) * sizeof(bmc::BlockPartial)));
            std::vector<bmc::BlockPartial> parts(P);
            BMC_CK(ctx, bmc::launch_reduce(d, hz, n, ctx->partials.as<bmc::BlockPartial>(), s));
            BMC_CK(ctx, cudaMemcpyAsync(parts.data(), ctx->partials.p, P * sizeof(bmc::BlockPartial),
                                        cudaMemcpyDeviceToHost, s));
            BMC_CK(ctx, cudaStreamSynchronize(s));
            ctx->last_launches = 1;
            bmc::DDh sum;
            for (const auto& q : parts) {
                p.min = std::fmin(p.min, q.min);
                p.max = std::fmax(p.max, q.max);
                sum = bmc::dd_merge_h(sum, q.sum_hi, q.sum_lo);
                p.horizon_count += q.horizon;
                p.count += q.count;
                p.any_nan |= q.nan;
            }
            p.sum_hi = sum.hi;
            p.sum_lo = sum.lo;
        }
        *out = p;
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_moments(bmc_ctx* ctx, const double* d, size_t n, double mean, double* m2m3) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if ((rc = bmc::order_after_rollouts(ctx)) != BMC_OK) return rc;
        if (!d || !m2m3) return fail(ctx, BMC_E_CONFIG, "moments: null argument");
        ctx->last_launches = 0;
        bmc::DDh m2, m3;
        if (n > 0) {
            cudaStream_t s = ctx->stream;
            const int P = bmc::stats_partials(n);
            BMC_CK(ctx, ctx->partials.reserve(static_cast<size_t>(P) * sizeof(bmc::MomentPartial)));
            std::vector<bmc::MomentPartial> mom(P);
            BMC_CK(ctx, bmc::launch_moments(d, n, mean, ctx->partials.as<bmc::MomentPartial>(), s));
            BMC_CK(ctx, cudaMemcpyAsync(mom.data(), ctx->partials.p, P * sizeof(bmc::MomentPartial),
                                        cudaMemcpyDeviceToHost, s));
            BMC_CK(ctx, cudaStreamSynchronize(s));
            ctx->last_launches = 1;
            for (const auto& q : mom) {
                m2 = bmc::dd_merge_h(m2, q.m2_hi, q.m2_lo);
                m3 = bmc::dd_merge_h(m3, q.m3_hi, q.m3_lo);
            }
        }
        m2m3[0] = m2.hi;
        m2m3[1] = m2.lo;
        m2m3[2] = m3.hi;
        m2m3[3] = m3.lo;
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_histogram(bmc_ctx* ctx, const double* d, size_t n, double origin, double bin_width,
                       uint64_t bins, uint64_t* counts) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if ((rc = bmc::order_after_rollouts(ctx)) != BMC_OK) return rc;
        if (!d || !counts) return fail(ctx, BMC_E_CONFIG, "histogram: null argument");
        if (!(bin_width > 0.0)) return fail(ctx, BMC_E_CONFIG, "outputs.bin_width: must be > 0");
        if (bins == 0 || bins > (uint64_t{1} << 28)) return fail(ctx, BMC_E_RANGE, "histogram: bins out of range");
        ctx->last_launches = 0;
        cudaStream_t s = ctx->stream;
        BMC_CK(ctx, ctx->hist_buf.reserve(bins * sizeof(unsigned long long)));
        BMC_CK(ctx, cudaMemsetAsync(ctx->hist_buf.p, 0, bins * sizeof(unsigned long long), s));
        if (n > 0) {
            BMC_CK(ctx, bmc::launch_hist(d, n, origin, bin_width, bins, ctx->hist_buf.as<unsigned long long>(), s));
            ctx->last_launches = 1;
        }
        BMC_CK(ctx, cudaMemcpyAsync(counts, ctx->hist_buf.p, bins * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        BMC_CK(ctx, cudaStreamSynchronize(s));
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

int bmc_cuda_select_pass(bmc_ctx* ctx, const double* d, const uint8_t* hz, size_t n,
                         int exclude_horizon, int shift, const uint64_t* prefixes, size_t m,
                         uint64_t* hist) {
    try {
        int rc = bmc::prepare(ctx);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if ((rc = bmc::order_after_rollouts(ctx)) != BMC_OK) return rc;
        if (!d || !prefixes || !hist) return fail(ctx, BMC_E_CONFIG, "select_pass: null argument");
        if (m < 1 || m > static_cast<size_t>(bmc::kMaxSelectTargets)) {
            return fail(ctx, BMC_E_RANGE, "select_pass: 1..16 targets per pass");
        }
        if (shift < 0 || shift > 56 || shift % 8 != 0) return fail(ctx, BMC_E_CONFIG, "select_pass: shift must be 0, 8, ..., 56");
        ctx->last_launches = 0;
        cudaStream_t s = ctx->stream;
        BMC_CK(ctx, ctx->sel_pref.reserve(bmc::kMaxSelectTargets * sizeof(uint64_t)));
        BMC_CK(ctx, ctx->sel_hist.reserve(bmc::kMaxSelectTargets * 256 * sizeof(unsigned long long)));
        BMC_CK(ctx, cudaMemcpyAsync(ctx->sel_pref.p, prefixes, m * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
        BMC_CK(ctx, cudaMemsetAsync(ctx->sel_hist.p, 0, m * 256 * sizeof(unsigned long long), s));
        if (n > 0) {
            BMC_CK(ctx, bmc::launch_select(d, hz, n, exclude_horizon, shift, ctx->sel_pref.as<uint64_t>(),
                                           static_cast<int>(m), ctx->sel_hist.as<unsigned long long>(), s));
            ctx->last_launches = 1;
        }
        BMC_CK(ctx, cudaMemcpyAsync(hist, ctx->sel_hist.p, m * 256 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        BMC_CK(ctx, cudaStreamSynchronize(s));
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception(ctx);
    }
}

}  // extern "C"
