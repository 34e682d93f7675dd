// stats_host.cpp -- TEST INFRASTRUCTURE: the fused statistics stage of the
// product library (paper_2604_27193_b200/csrc/bmc_stats_pipeline.h) driven
// by a host backend, so its merge logic -- the three merge points, padded
// candidate exchange, overflow fallbacks -- runs on CPU under fake
// collectives (tests/test_stats_merge.py over gloo, tests/cpp/merge_main.cpp
// with in-process ranks).  Every stage is the same arithmetic as the kernels
// (bmc_stats_core.h compiled by g++ -ffp-contract=off); GPU tests compare the
// two backends bit for bit.  Never linked into the product.
#include "bmc_stats_pipeline.h"

#include <cstdio>
#include <cstring>
#include <vector>

namespace bmc {
namespace {

struct HostStage {
    StatsConfig cfg;
    StatsLayout L{};
    std::vector<uint64_t> mem, gather;
};

struct HostBackend {
    HostStage* st;
    uint32_t launches = 0;

    uint64_t* words(size_t off) {
        if (off >= st->L.gather) return st->gather.data() + (off - st->L.gather);
        return st->mem.data() + off;
    }
    sc::Scalars& scal() { return *reinterpret_cast<sc::Scalars*>(words(st->L.scal)); }
    sc::Target* tgt() { return reinterpret_cast<sc::Target*>(words(st->L.targets)); }
    int ensure_gather(size_t w) {
        if (st->gather.size() < w) st->gather.resize(w);
        return BMC_OK;
    }
    int normalize(size_t off, int accs) {
        for (int k = 0; k < 2 * accs; ++k) {
            sc::normalize(words(off) + static_cast<size_t>(k / 2) * sc::kAccWords +
                          static_cast<size_t>(k % 2) * sc::kLimbs);
        }
        ++launches;
        return BMC_OK;
    }
    int finalize1() {
        uint64_t work[2 * sc::kLimbs];
        sc::finalize_p1(words(st->L.p1_sum), words(st->L.p1_min), st->cfg.bin_width,
                        st->cfg.hist_cap, work, &scal());
        ++launches;
        return BMC_OK;
    }
    int pass2(const double* d, const uint8_t* hz, uint64_t n) {
        const sc::Scalars s = scal();
        const uint64_t hc = st->cfg.summary ? st->cfg.hist_cap : 0;
        uint64_t* p2 = words(st->L.p2_sum);
        const bool hist_on = st->cfg.summary && !s.hist_overflow;
        for (uint64_t i = 0; i < n; ++i) {
            const double v = d[i];
            const bool h = hz && hz[i];
            if (st->cfg.summary) {
                const double dev = v - s.mean;
                const double sq = dev * dev;
                uint64_t* m2 = p2 + sc::kP2M2;
                uint64_t* m3 = p2 + sc::kP2M3;
                sc::acc_add(m2, m2 + sc::kLimbs, m2 + 2 * sc::kLimbs, sq);
                sc::acc_add(m3, m3 + sc::kLimbs, m3 + 2 * sc::kLimbs, sq * dev);
            }
            if (sc::is_nan(v)) continue;
            if (hist_on) p2[sc::kP2Hist + sc::hist_index(v, s.lo, s.bin_width, s.bins)] += 1;
            const int b = sc::sel_bucket(v, s.sel_lo, s.sel_scale);
            p2[sc::p2_sel_all(hc) + b] += 1;
            if (h) p2[sc::p2_sel_hz(hc) + b] += 1;
        }
        ++launches;
        return BMC_OK;
    }
    int targets() {
        const sc::Scalars s = scal();
        const uint64_t hc = st->cfg.summary ? st->cfg.hist_cap : 0;
        const uint64_t* p2 = words(st->L.p2_sum);
        sc::Target* tg = tgt();
        for (int t = 0; t < sc::kMaxTargets; ++t) {
            sc::Target x{};
            x.bucket = -1;
            if (t < 2) {
                x.population = 0;
                if (st->cfg.summary && s.n) x.rank = t == 0 ? (s.n % 2 == 0 ? s.n / 2 : 0) : s.n / 2 + 1;
                x.valid = x.rank >= 1 && x.rank <= s.n - s.nan_count;
            } else if (t < 2 + st->cfg.n_risk()) {
                x.population = 1;
                x.rank = sc::risk_rank(st->cfg.risks[static_cast<size_t>(t - 2)], s.n);
                x.valid = x.rank >= 1 && x.rank <= s.stopped;
            }
            if (x.valid && x.rank) {
                const uint64_t* all = p2 + sc::p2_sel_all(hc);
                const uint64_t* hzb = p2 + sc::p2_sel_hz(hc);
                uint64_t cum = 0;
                for (int b = 0; b < sc::kB1; ++b) {
                    const uint64_t c = x.population ? all[b] - hzb[b] : all[b];  // stoppers
                    if (cum + c >= x.rank) {
                        x.bucket = b;
                        x.residual = x.rank - cum;
                        break;
                    }
                    cum += c;
                }
                if (x.bucket < 0) x.valid = 0;
            }
            tg[t] = x;
        }
        ++launches;
        return BMC_OK;
    }
    int compact(const double* d, const uint8_t* hz, uint64_t n) {
        const sc::Scalars s = scal();
        const sc::Target* tg = tgt();
        uint64_t* cnt = words(st->L.cand_count);
        uint64_t* cand = words(st->L.cand);
        const uint64_t cap = st->cfg.cand_cap;
        for (uint64_t i = 0; i < n; ++i) {
            const double v = d[i];
            if (sc::is_nan(v)) continue;
            const int b = sc::sel_bucket(v, s.sel_lo, s.sel_scale);
            const bool h = hz && hz[i];
            for (int t = 0; t < st->cfg.n_targets(); ++t) {
                if (!tg[t].valid || !tg[t].rank || tg[t].bucket != b || (tg[t].population == 1 && h)) continue;
                const uint64_t pos = cnt[t]++;
                if (pos < cap) cand[static_cast<uint64_t>(t) * cap + pos] = sc::order_key(v);
            }
        }
        ++launches;
        return BMC_OK;
    }
    int pack(const uint64_t* P, const uint64_t* off, uint64_t total) {
        const uint64_t* cnt = words(st->L.cand_count);
        const uint64_t* cand = words(st->L.cand);
        const uint64_t cap = st->cfg.cand_cap;
        for (int t = 0; t < st->cfg.n_targets(); ++t) {
            const uint64_t c = std::min(cnt[t], cap);
            for (uint64_t k = 0; k < P[t]; ++k) {
                st->gather[off[t] + k] = k < c ? cand[static_cast<uint64_t>(t) * cap + k] : ~0ull;
            }
        }
        (void)total;
        ++launches;
        return BMC_OK;
    }
    int mark_overflow(const bool* over) {
        for (int t = 0; t < st->cfg.n_targets(); ++t) {
            if (over[t]) tgt()[t].overflow = 1;
        }
        return BMC_OK;
    }
    int select(const SelectSegments& seg) {
        sc::Target* tg = tgt();
        const uint64_t* keys = seg.in_gather ? st->gather.data() : st->mem.data();
        for (int t = 0; t < st->cfg.n_targets(); ++t) {
            sc::Target& x = tg[t];
            if (!x.valid || !x.rank || x.overflow) continue;
            uint64_t len = seg.len[t];
            if (seg.use_counts) {
                const uint64_t c = words(st->L.cand_count)[t];
                if (c > st->cfg.cand_cap) {
                    x.overflow = 1;
                    continue;
                }
                len = c;
            }
            std::vector<uint64_t> v;
            for (int r = 0; r < seg.world; ++r) {
                const uint64_t* k = keys + seg.base[t] + static_cast<uint64_t>(r) * seg.rank_stride;
                for (uint64_t i = 0; i < len; ++i)
                    if (k[i] != ~0ull) v.push_back(k[i]);
            }
            if (x.residual < 1 || x.residual > v.size()) {
                x.valid = 0;
                continue;
            }
            std::nth_element(v.begin(), v.begin() + static_cast<std::ptrdiff_t>(x.residual - 1), v.end());
            x.key = v[x.residual - 1];
        }
        ++launches;
        return BMC_OK;
    }
    int read(void* host, size_t off, size_t w) {
        std::memcpy(host, words(off), w * 8);
        return BMC_OK;
    }
    int write(size_t off, const void* host, size_t w) {
        std::memcpy(words(off), host, w * 8);
        return BMC_OK;
    }
    int snapshot(size_t w, const uint64_t** host) {
        (void)w;
        *host = st->mem.data();
        return BMC_OK;
    }
    int hist_full(const double* d, uint64_t n, double lo, double bw, uint64_t bins, uint64_t* out) {
        for (uint64_t i = 0; i < n; ++i) {
            if (!sc::is_nan(d[i])) out[sc::hist_index(d[i], lo, bw, bins)] += 1;
        }
        return BMC_OK;
    }
    int select_pass(const double* d, const uint8_t* hz, uint64_t n, int exclude, int shift,
                    const uint64_t* prefixes, size_t m, uint64_t* hist) {
        std::fill(hist, hist + m * 256, 0);
        const uint64_t mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
        for (uint64_t i = 0; i < n; ++i) {
            if (exclude && hz && hz[i]) continue;
            const uint64_t key = sc::order_key(d[i]);
            const unsigned digit = static_cast<unsigned>((key >> shift) & 0xFFu);
            for (size_t t = 0; t < m; ++t)
                if ((key & mask) == prefixes[t]) hist[t * 256 + digit] += 1;
        }
        return BMC_OK;
    }
};

}  // namespace
}  // namespace bmc

extern "C" {

// Pass 1 + finish on host arrays; cand_cap > 0 overrides the candidate
// capacity (tests force the overflow fallback with it).
int bmch_stats_run(const double* d, const uint8_t* hz, size_t n, const bmc_stats_req* req,
                   uint64_t cand_cap, const bmc_merge* merge, bmc_stats* out, char* err,
                   size_t errcap) {
    using namespace bmc;
    HostStage st;
    std::string e;
    int rc = resolve_request(req, n, &st.cfg, &e);
    if (rc == BMC_OK) {
        if (cand_cap) st.cfg.cand_cap = cand_cap;
        st.L = make_layout(st.cfg);
        st.mem.assign(st.L.total, 0);
        uint64_t* w = st.mem.data();
        w[st.L.p1_min] = ~0ull;
        w[st.L.p1_min + 1] = ~0ull;
        // pass 1
        uint64_t* p1 = w + st.L.p1_sum;
        uint64_t* acc = p1 + sc::kP1Acc;
        for (size_t i = 0; i < n; ++i) {
            const double v = d[i];
            const bool h = hz && hz[i];
            p1[sc::kP1Count] += 1;
            if (h) p1[sc::kP1Horizon] += 1;
            sc::acc_add(acc, acc + sc::kLimbs, acc + 2 * sc::kLimbs, v);
            if (sc::special_of(v) != sc::kNaN) {
                const uint64_t k = sc::order_key(v);
                w[st.L.p1_min] = std::min(w[st.L.p1_min], k);
                w[st.L.p1_min + 1] = std::min(w[st.L.p1_min + 1], ~k);
            }
            if (st.cfg.m()) p1[sc::kP1Exceed + sc::exceed_bucket(st.cfg.headways.data(), st.cfg.m(), v, h)] += 1;
        }
        HostBackend be{&st};
        uint32_t launches = 0;
        rc = stats_finish(be, st.cfg, st.L, d, hz, n, merge, out, nullptr, &launches, &e);
        out->launches = be.launches;
    }
    if (rc != BMC_OK && err && errcap) std::snprintf(err, errcap, "%s", e.c_str());
    return rc;
}

// hist_index_fast (the kernels' division-free path) against the exact
// hist_index on caller-chosen values; returns the number of disagreements.
uint64_t bmch_hist_index_mismatches(const double* v, size_t n, double lo, double bw,
                                    uint64_t bins) {
    using namespace bmc;
    const double inv = 1.0 / bw;
    uint64_t bad = 0;
    for (size_t i = 0; i < n; ++i) {
        if (sc::hist_index_fast(v[i], lo, bw, inv, bins) != sc::hist_index(v[i], lo, bw, bins)) ++bad;
    }
    return bad;
}

// The exact sum of the stage's arithmetic, for unit tests of the
// superaccumulator against math.fsum.
double bmch_exact_sum(const double* v, size_t n) {
    using namespace bmc;
    uint64_t a[sc::kAccWords] = {0};
    for (size_t i = 0; i < n; ++i) sc::acc_add(a, a + sc::kLimbs, a + 2 * sc::kLimbs, v[i]);
    return round_acc(a);
}

}  // extern "C"
