// bmc_stats_pipeline.h -- orchestration of the fused statistics stage.
//
// One template drives both backends:
//   * DeviceBackend (bmc_capi_stats.cpp): sm_100a kernels enqueued on one
//     stream; with no merge the whole stage is device-side (no host round
//     trip until the final read), so a CUDA graph can capture it;
//   * HostBackend (tests/cpp/stats_host.cpp, test infrastructure only): the
//     same stages as plain loops over host arrays, so the merge logic is
//     exercised on CPU with fake collectives (worlds 2 and 3).
//
// Stages (reference: /root/reference/proj/src/analysis.cpp):
//   P1   counts, horizon, extrema keys, exact sum, exceedance buckets
//        (fused into the rollout epilogue, or a standalone pass)
//   [merge A: SUM p1_sum, MIN p1_min]
//   finalize_p1 -> mean, min, max, histogram origin/bins, bucket map
//   P2   exact m2/m3, summary histogram, level-1 order-statistic histograms
//   [merge B: SUM p2_sum]
//   targets -> bucket + residual rank of each order statistic
//   compact  -> the values of each target bucket
//   [merge C: allgather of the candidates]
//   select   -> exact order statistic per target
//   read back + host composition (sd, skewness with glibc pow, median, ...)
#pragma once

#include "bmc_stats_core.h"
#include "brakemc_cuda.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

namespace bmc {

// Default capacities (results never depend on them; overflow falls back to
// exact multi-pass selection).
constexpr uint64_t kDefaultHistCap = 8192;
constexpr size_t kMaxFusedHeadways = 4096;

struct StatsConfig {
    std::vector<double> headways;   // sorted ascending
    std::vector<size_t> order;      // order[j] = caller index of headways[j]
    std::vector<double> risks;      // caller order
    bool summary = false;
    double bin_width = 0.0;
    uint64_t hist_cap = kDefaultHistCap;
    uint64_t cand_cap = 0;
    int m() const { return static_cast<int>(headways.size()); }
    int n_risk() const { return static_cast<int>(risks.size()); }
    int n_targets() const { return 2 + n_risk(); }
    bool need_p2() const { return summary || !risks.empty(); }
};

// Word offsets of one stage's memory (identical on both backends).
struct StatsLayout {
    size_t p1_min, p1_sum, p2_sum, cand_count, scal, targets, headways, risks, cand, gather;
    size_t zero_begin, zero_end;  // [p1_sum, cand_count + targets) is zeroed per run
    size_t total;
    int p1_words = 0, p2_words = 0, n_targets = 0;
};

inline int resolve_request(const bmc_stats_req* req, uint64_t max_n, StatsConfig* cfg,
                           std::string* err) {
    StatsConfig c;
    if (req) {
        if (req->n_headways && !req->headways) {
            *err = "stats: null headways";
            return BMC_E_CONFIG;
        }
        if (req->n_risk && !req->risk_levels) {
            *err = "stats: null risk levels";
            return BMC_E_CONFIG;
        }
        for (size_t j = 0; j < req->n_headways; ++j) {
            if (!(req->headways[j] >= 0.0)) {  // analysis.cpp:146-148
                *err = "risk.headway: must be >= 0";
                return BMC_E_CONFIG;
            }
        }
        if (req->n_risk > static_cast<size_t>(sc::kMaxRisk)) {
            *err = "risk.levels: at most 16 per stage";
            return BMC_E_RANGE;
        }
        for (size_t k = 0; k < req->n_risk; ++k) {
            const double r = req->risk_levels[k];
            if (!(r > 0.0 && r < 1.0)) {  // analysis.cpp:162-164
                *err = "risk.level: must be strictly between 0 and 1";
                return BMC_E_CONFIG;
            }
            c.risks.push_back(r);
        }
        if (req->summarize) {
            if (!(req->bin_width > 0.0)) {  // analysis.cpp:17-19
                *err = "outputs.bin_width: must be > 0";
                return BMC_E_CONFIG;
            }
            c.summary = true;
            c.bin_width = req->bin_width;
        }
        if (req->hist_cap) c.hist_cap = req->hist_cap;
        const size_t m = req->n_headways;
        if (m > (size_t{1} << 24)) {
            *err = "risk.headways: at most 2^24 per stage";
            return BMC_E_RANGE;
        }
        c.order.resize(m);
        std::iota(c.order.begin(), c.order.end(), size_t{0});
        std::stable_sort(c.order.begin(), c.order.end(),
                         [&](size_t a, size_t b) { return req->headways[a] < req->headways[b]; });
        for (size_t j = 0; j < m; ++j) c.headways.push_back(req->headways[c.order[j]]);
    }
    // candidate capacity per target: the level-1 bucket holding a rank keeps
    // about 1e-3 of the values for smooth distributions (n/256 leaves margin);
    // batches up to 64k never overflow
    const uint64_t n = std::max<uint64_t>(max_n, 1);
    c.cand_cap = std::min<uint64_t>(n, std::max<uint64_t>(uint64_t{1} << 16, n >> 8));
    if (req && req->cand_cap) c.cand_cap = req->cand_cap;
    *cfg = c;
    return BMC_OK;
}

inline StatsLayout make_layout(const StatsConfig& c) {
    StatsLayout L{};
    L.p1_words = sc::p1_sum_words(c.m());
    L.p2_words = c.need_p2() ? sc::p2_sum_words(c.summary ? c.hist_cap : 0) : 0;
    L.n_targets = c.n_targets();
    size_t o = 0;
    auto take = [&](size_t words) {
        const size_t at = o;
        o += (words + 1) & ~size_t{1};  // 16-byte alignment
        return at;
    };
    L.p1_min = take(sc::kP1MinWords);
    L.p1_sum = take(static_cast<size_t>(L.p1_words));
    L.zero_begin = L.p1_sum;
    L.p2_sum = take(static_cast<size_t>(L.p2_words));
    L.cand_count = take(sc::kMaxTargets);
    L.targets = take(sc::kMaxTargets * sizeof(sc::Target) / 8);
    L.zero_end = o;
    L.scal = take(sizeof(sc::Scalars) / 8);
    L.headways = take(static_cast<size_t>(c.m()));
    L.risks = take(sc::kMaxRisk);
    L.cand = take(static_cast<size_t>(L.n_targets) * c.cand_cap);
    L.gather = o;  // merge scratch follows (sized per run)
    L.total = o;
    return L;
}


// Host composition of the read-back partials into the caller's bmc_stats
// (analysis.cpp:13-76, 145-194; the few scalar ops that use libm -- pow --
// run here, on the host, exactly as the reference does).
struct StatsReadback {
    std::vector<uint64_t> p1_sum;
    uint64_t p1_min[2];
    sc::Scalars scal;
    std::vector<uint64_t> p2_head;  // m2 + m3 accumulators (2 * kAccWords)
    std::vector<uint64_t> hist;     // first min(bins, hist_cap) words
    sc::Target targets[sc::kMaxTargets];
};

inline double round_acc(const uint64_t* acc) {
    uint64_t w[2 * sc::kLimbs];
    for (int i = 0; i < 2 * sc::kLimbs; ++i) w[i] = acc[i];
    sc::normalize(w);
    sc::normalize(w + sc::kLimbs);
    return sc::sum_value(w, w + sc::kLimbs, acc + 2 * sc::kLimbs);
}

// Merge callbacks (one call per merge point; buffers are backend memory).
inline int merge_reduce(const bmc_merge* mg, uint64_t* buf, size_t count, int op, void* stream,
                        std::string* err) {
    if (count == 0) return BMC_OK;
    const int rc = mg->allreduce_u64(mg->user, buf, count, op, stream);
    if (rc != 0) {
        *err = "stats merge: allreduce failed (" + std::to_string(rc) + ")";
        return BMC_E_CUDA;
    }
    return BMC_OK;
}

inline int merge_gather(const bmc_merge* mg, const uint64_t* send, uint64_t* recv, size_t count,
                        void* stream, std::string* err) {
    const int rc = mg->allgather_u64(mg->user, send, recv, count, stream);
    if (rc != 0) {
        *err = "stats merge: allgather failed (" + std::to_string(rc) + ")";
        return BMC_E_CUDA;
    }
    return BMC_OK;
}

// The stage after P1 has been accumulated on every rank.  `d`/`hz` are this
// rank's outputs (backend memory), n its count.  Backend contract (all
// operations ordered on `stream`):
//   uint64_t* words(size_t offset)             backend pointer into the stage memory
//   int ensure_gather(size_t words)            merge scratch of that many words
//   int normalize(size_t offset, int accs)     carry-normalise `accs` exact sums in place
//   int finalize1(), pass2(d,hz,n), targets(), compact(d,hz,n)
//   int pack(P, off, total)                    padded local candidates -> scratch
//   int mark_overflow(const bool* over)        targets whose candidates overflowed a rank
//   int select(const SelectSegments&)
//   int hist_full(d, n, lo, bw, bins, uint64_t* host_out)   histogram fallback (local)
//   int select_pass(d, hz, n, exclude, shift, prefixes, m, uint64_t* host_hist)
//   int read(void* host, size_t offset, size_t words)   synchronising copy
//   int snapshot(size_t words, const uint64_t** host)   stage words [0, words) on the host
//   int write(size_t offset, const void* host, size_t words)
//
// Part 1: every device stage up to the selected order statistics.  With no
// merge nothing here reads back, so a CUDA graph can capture it.
template <class B>
int stats_device_stages(B& be, const StatsConfig& cfg, const StatsLayout& L, const double* d,
                        const uint8_t* hz, uint64_t n, const bmc_merge* mg, void* stream,
                        std::string* err) {
    int rc;
    const bool merging = mg != nullptr;
    const int T = cfg.n_targets();
    // ---- merge A
    if (merging) {
        if ((rc = be.normalize(L.p1_sum + sc::kP1Acc, 1)) != BMC_OK) return rc;
        if ((rc = merge_reduce(mg, be.words(L.p1_sum), L.p1_words, BMC_MERGE_SUM, stream, err)) != BMC_OK) return rc;
        if ((rc = merge_reduce(mg, be.words(L.p1_min), 2, BMC_MERGE_MIN, stream, err)) != BMC_OK) return rc;
    }
    if ((rc = be.finalize1()) != BMC_OK) return rc;
    if (!cfg.need_p2()) return BMC_OK;
    // ---- P2 + merge B
    if ((rc = be.pass2(d, hz, n)) != BMC_OK) return rc;
    if (merging) {
        if ((rc = be.normalize(L.p2_sum, 2)) != BMC_OK) return rc;
        if ((rc = merge_reduce(mg, be.words(L.p2_sum), L.p2_words, BMC_MERGE_SUM, stream, err)) != BMC_OK) return rc;
    }
    if ((rc = be.targets()) != BMC_OK) return rc;
    if ((rc = be.compact(d, hz, n)) != BMC_OK) return rc;
    SelectSegments seg{};
    seg.world = 1;
    if (!merging) {
        for (int t = 0; t < T; ++t) {
            seg.base[t] = L.cand + static_cast<uint64_t>(t) * cfg.cand_cap;
            seg.len[t] = cfg.cand_cap;
        }
        seg.use_counts = 1;
        return be.select(seg);
    }
    // ---- merge C: every rank's counts, then the padded candidate lists
    const int G = mg->world;
    if ((rc = be.ensure_gather(static_cast<size_t>(G) * sc::kMaxTargets)) != BMC_OK) return rc;
    if ((rc = merge_gather(mg, be.words(L.cand_count), be.words(L.gather), sc::kMaxTargets, stream,
                           err)) != BMC_OK) return rc;
    std::vector<uint64_t> counts(static_cast<size_t>(G) * sc::kMaxTargets);
    if ((rc = be.read(counts.data(), L.gather, counts.size())) != BMC_OK) return rc;
    uint64_t P[sc::kMaxTargets] = {0};
    bool over[sc::kMaxTargets] = {false};
    for (int r = 0; r < G; ++r) {
        for (int t = 0; t < T; ++t) {
            const uint64_t c = counts[static_cast<size_t>(r) * sc::kMaxTargets + t];
            if (c > cfg.cand_cap) over[t] = true;
            P[t] = std::max(P[t], std::min<uint64_t>(c, cfg.cand_cap));
        }
    }
    uint64_t S = 0, off[sc::kMaxTargets] = {0};
    for (int t = 0; t < T; ++t) {
        if (over[t]) P[t] = 0;  // exact fallback after the read back
        off[t] = S;
        S += P[t];
    }
    // local padded block [t0: P0 keys][t1: P1 keys]... at the scratch start,
    // every rank's block gathered right after it
    if ((rc = be.ensure_gather(S * (static_cast<size_t>(G) + 1))) != BMC_OK) return rc;
    if ((rc = be.pack(P, off, S)) != BMC_OK) return rc;
    if (S) {
        if ((rc = merge_gather(mg, be.words(L.gather), be.words(L.gather + S), S, stream, err)) != BMC_OK) return rc;
    }
    for (int t = 0; t < T; ++t) {
        seg.base[t] = S + off[t];  // relative to the merge scratch
        seg.len[t] = P[t];
    }
    seg.rank_stride = S;
    seg.world = G;
    seg.use_counts = 0;
    seg.in_gather = 1;
    if ((rc = be.mark_overflow(over)) != BMC_OK) return rc;
    return be.select(seg);
}

// The words the host composition needs, as (offset, count) regions of the
// stage memory: P1 (both sections), scalars, m2/m3 + histogram, targets.
struct ReadRegion {
    size_t off, words;
};
inline std::vector<ReadRegion> readback_regions(const StatsConfig& cfg, const StatsLayout& L) {
    std::vector<ReadRegion> r;
    r.push_back({L.p1_min, L.p1_sum + static_cast<size_t>(L.p1_words) - L.p1_min});
    r.push_back({L.scal, sizeof(sc::Scalars) / 8});
    if (cfg.need_p2()) {
        r.push_back({L.p2_sum, 2 * static_cast<size_t>(sc::kAccWords) +
                                   (cfg.summary ? static_cast<size_t>(cfg.hist_cap) : 0)});
        r.push_back({L.targets, sc::kMaxTargets * sizeof(sc::Target) / 8});
    }
    return r;
}

// Part 2: read back.  `read(host, off, words)` copies stage words.
template <class Read>
int stats_read(Read&& read, const StatsConfig& cfg, const StatsLayout& L, StatsReadback* rb) {
    int rc;
    rb->p1_sum.resize(static_cast<size_t>(L.p1_words));
    if ((rc = read(rb->p1_sum.data(), L.p1_sum, rb->p1_sum.size())) != BMC_OK) return rc;
    if ((rc = read(rb->p1_min, L.p1_min, 2)) != BMC_OK) return rc;
    if ((rc = read(&rb->scal, L.scal, sizeof(sc::Scalars) / 8)) != BMC_OK) return rc;
    if (cfg.need_p2()) {
        rb->p2_head.resize(2 * sc::kAccWords);
        if ((rc = read(rb->p2_head.data(), L.p2_sum, rb->p2_head.size())) != BMC_OK) return rc;
        if ((rc = read(rb->targets, L.targets, sc::kMaxTargets * sizeof(sc::Target) / 8)) != BMC_OK) return rc;
        if (cfg.summary && !rb->scal.hist_overflow) {
            rb->hist.resize(rb->scal.bins);
            if ((rc = read(rb->hist.data(), L.p2_sum + sc::kP2Hist, rb->hist.size())) != BMC_OK) return rc;
        }
    }
    return BMC_OK;
}

// Part 3: exact fallbacks (degenerate data only) and the host composition.
template <class B>
int stats_compose(B& be, const StatsConfig& cfg, const StatsLayout& L, StatsReadback& rb,
                  const double* d, const uint8_t* hz, uint64_t n, const bmc_merge* mg,
                  bmc_stats* out, void* stream, std::string* err) {
    int rc;
    const bool merging = mg != nullptr;
    const int T = cfg.n_targets();
    const sc::Scalars& s = rb.scal;
    if (s.n == 0) {
        *err = cfg.summary ? "summarize: needs at least one result" : "risk: needs at least one result";
        return BMC_E_CONFIG;
    }
    if (cfg.summary && s.hist_overflow) {
        // the reference sizes counts with (size_t)ceil((hi - lo) / bw) (analysis.cpp:61-63):
        // a non-finite or extreme range has no usable histogram there either
        if (s.bins > (uint64_t{1} << 30)) {
            *err = "summarize: histogram of " + std::to_string(s.bins) +
                   " bins (non-finite or extreme stop-distance range)";
            return BMC_E_RANGE;
        }
        rb.hist.assign(s.bins, 0);
        if ((rc = be.hist_full(d, n, s.lo, s.bin_width, s.bins, rb.hist.data())) != BMC_OK) return rc;
        if (merging) {
            if ((rc = be.ensure_gather(s.bins)) != BMC_OK) return rc;
            if ((rc = be.write(L.gather, rb.hist.data(), s.bins)) != BMC_OK) return rc;
            if ((rc = merge_reduce(mg, be.words(L.gather), s.bins, BMC_MERGE_SUM, stream, err)) != BMC_OK) return rc;
            if ((rc = be.read(rb.hist.data(), L.gather, s.bins)) != BMC_OK) return rc;
        }
    }
    uint32_t fallbacks = 0;
    if (cfg.need_p2()) {
        // exact 8 x 8-bit radix select over the whole shard for targets whose
        // bucket overflowed the candidate capacity (SUM-merged digit counts)
        for (int pop = 0; pop < 2; ++pop) {
            std::vector<int> which;
            for (int t = 0; t < T; ++t) {
                const sc::Target& g = rb.targets[t];
                if (g.rank && g.valid && g.overflow && g.population == pop) which.push_back(t);
            }
            for (size_t w0 = 0; w0 < which.size(); w0 += 16) {
                const size_t tm = std::min<size_t>(16, which.size() - w0);
                std::vector<uint64_t> prefix(tm, 0), resid(tm);
                for (size_t k = 0; k < tm; ++k) resid[k] = rb.targets[which[w0 + k]].rank;
                std::vector<uint64_t> hist(tm * 256);
                if (merging && (rc = be.ensure_gather(tm * 256 + 16)) != BMC_OK) return rc;
                for (int shift = 56; shift >= 0; shift -= 8) {
                    if ((rc = be.select_pass(d, hz, n, pop, shift, prefix.data(), tm, hist.data())) != BMC_OK) return rc;
                    if (merging) {
                        if ((rc = be.write(L.gather, hist.data(), hist.size())) != BMC_OK) return rc;
                        if ((rc = merge_reduce(mg, be.words(L.gather), hist.size(), BMC_MERGE_SUM, stream, err)) != BMC_OK) return rc;
                        if ((rc = be.read(hist.data(), L.gather, hist.size())) != BMC_OK) return rc;
                    }
                    for (size_t k = 0; k < tm; ++k) {
                        uint64_t cum = 0;
                        int digit = 255;
                        for (int b = 0; b < 256; ++b) {
                            const uint64_t c = hist[k * 256 + b];
                            if (cum + c >= resid[k]) {
                                digit = b;
                                break;
                            }
                            cum += c;
                        }
                        resid[k] -= cum;
                        prefix[k] |= static_cast<uint64_t>(digit) << shift;
                    }
                }
                for (size_t k = 0; k < tm; ++k) {
                    rb.targets[which[w0 + k]].key = prefix[k];
                    rb.targets[which[w0 + k]].overflow = 0;
                    ++fallbacks;
                }
            }
        }
    }
    out->n = s.n;
    out->horizon_count = s.horizon;
    const int m = cfg.m();
    if (out->exceed && m) {
        // exceed(sorted j) = #{p > j} = suffix sum of buckets j+1 .. m
        const uint64_t* b = rb.p1_sum.data() + sc::kP1Exceed;
        uint64_t suffix = 0;
        for (int j = m; j-- > 0;) {
            suffix += b[j + 1];
            out->exceed[cfg.order[static_cast<size_t>(j)]] = suffix;
        }
    }
    auto target_value = [&](int t) {
        const sc::Target& g = rb.targets[t];
        return g.valid ? sc::key_value(g.key) : std::numeric_limits<double>::quiet_NaN();
    };
    if (out->min_safe_headway) {
        for (int k = 0; k < cfg.n_risk(); ++k) {
            const sc::Target& g = rb.targets[2 + k];
            // analysis.cpp:186-189: a rank inside the never-stopping tail
            out->min_safe_headway[k] =
                g.valid ? sc::key_value(g.key) : std::numeric_limits<double>::infinity();
        }
    }
    if (cfg.summary) {
        bmc_summary sm;
        std::memset(&sm, 0, sizeof sm);
        sm.n = s.n;
        sm.horizon_count = s.horizon;
        sm.mean = s.mean;
        const double dn = static_cast<double>(s.n);
        const double M2 = round_acc(rb.p2_head.data());
        const double M3 = round_acc(rb.p2_head.data() + sc::kAccWords);
        // analysis.cpp:47-50
        sm.sd = s.n > 1 ? std::sqrt(M2 / (dn - 1.0)) : 0.0;
        const double var_pop = M2 / dn;
        sm.skewness = var_pop > 0.0 ? (M3 / dn) / std::pow(var_pop, 1.5) : 0.0;
        sm.min = s.min;
        sm.max = s.max;
        // analysis.cpp:51-57
        sm.median = (s.n % 2 == 1) ? target_value(1) : 0.5 * (target_value(0) + target_value(1));
        sm.right_skewed = sm.mean > sm.median ? 1 : 0;
        sm.origin = s.lo;
        sm.bin_width = s.bin_width;
        sm.bins = s.bins;
        out->summary = sm;
        if (out->histogram) {
            if (out->histogram_cap < s.bins) {
                *err = "summarize: histogram buffer smaller than bin count";
                return BMC_E_RANGE;
            }
            std::memcpy(out->histogram, rb.hist.data(), s.bins * sizeof(uint64_t));
        }
    }
    out->fallbacks = fallbacks;
    return BMC_OK;
}

template <class B>
int stats_finish(B& be, const StatsConfig& cfg, const StatsLayout& L, const double* d,
                 const uint8_t* hz, uint64_t n, const bmc_merge* mg, bmc_stats* out,
                 void* stream, uint32_t* launches, std::string* err) {
    int rc = stats_device_stages(be, cfg, L, d, hz, n, mg, stream, err);
    if (rc != BMC_OK) return rc;
    // one synchronising copy of the stage words [0, L.cand) (~140 KB), then
    // the composition reads host memory
    const uint64_t* snap = nullptr;
    if ((rc = be.snapshot(L.cand, &snap)) != BMC_OK) return rc;
    StatsReadback rb;
    rc = stats_read(
        [&](void* h, size_t off, size_t w) {
            std::memcpy(h, snap + off, w * 8);
            return BMC_OK;
        },
        cfg, L, &rb);
    if (rc != BMC_OK) return rc;
    rc = stats_compose(be, cfg, L, rb, d, hz, n, mg, out, stream, err);
    if (launches) *launches = 0;
    return rc;
}

}  // namespace bmc
