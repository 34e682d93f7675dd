// bmc_stats_core.h -- arithmetic of the fused statistics stage, shared
// verbatim by the sm_100a kernels (nvcc -fmad=false) and the host code
// (g++ -ffp-contract=off): every FP operation is one IEEE op spelled with
// BMC_ADD/SUB/MUL/DIV, so both builds give identical bits.
//
// What the reference computes (/root/reference/proj/src/analysis.cpp) and how
// it is re-expressed here so that it streams, fuses and merges exactly:
//
//   * counts (horizon :25-30, exceedance :152-157, histogram :67-75): u64
//     integers -- exact and additive across CTAs, chunks and GPUs.
//   * min / max (:54-55): order keys (a monotone double -> u64 map) under
//     MIN; the max is carried as the MIN of the complemented key.
//   * sums (mean :34-38, m2/m3 :41-46): EXACT sums in a fixed-point
//     superaccumulator of 67 x 32-bit limbs covering every finite binary64
//     (LSB 2^-1074), one array per sign.  A value adds its 53-bit significand
//     to three limbs; a limb is a u64 counter, so up to 2^32 values accumulate
//     without normalisation.  Rounding the exact sum once gives the correctly
//     rounded sum -- independent of order, chunking and GPU count, so every
//     shard split yields the same bits.  (The reference's sequential sum is
//     within (n-1) eps sum|d| of it; tests/test_gpu_stats.py states the bound.)
//   * order statistics (median :51-57, min_safe_headway :161-194): a
//     level-1 histogram over B1 buckets linear in value between the exact min
//     and max (monotone map, so bucket order = value order), then the values
//     of the bucket holding the target rank are compacted and selected
//     exactly.  Exact for every input; the bucket only bounds the work.
#pragma once

#include <math.h>
#include <stddef.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define BMC_HD __host__ __device__ __forceinline__
#else
#define BMC_HD inline
#endif

#if defined(__CUDA_ARCH__)
#define BMC_ADD(a, b) __dadd_rn((a), (b))
#define BMC_SUB(a, b) __dsub_rn((a), (b))
#define BMC_MUL(a, b) __dmul_rn((a), (b))
#define BMC_DIV(a, b) __ddiv_rn((a), (b))
#else
#define BMC_ADD(a, b) ((a) + (b))
#define BMC_SUB(a, b) ((a) - (b))
#define BMC_MUL(a, b) ((a) * (b))
#define BMC_DIV(a, b) ((a) / (b))
#endif

namespace bmc {
namespace sc {

// ------------------------------------------------------------ bit casts
BMC_HD uint64_t bits_of(double v) {
#if defined(__CUDA_ARCH__)
    return static_cast<uint64_t>(__double_as_longlong(v));
#else
    uint64_t b;
    __builtin_memcpy(&b, &v, 8);
    return b;
#endif
}

BMC_HD double double_of(uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double(static_cast<long long>(b));
#else
    double v;
    __builtin_memcpy(&v, &b, 8);
    return v;
#endif
}

// Order-preserving map binary64 -> u64 (total order on non-NaN values; -0 <
// +0 is harmless: both keys decode to the value they came from).
BMC_HD uint64_t order_key(double v) {
    const uint64_t b = bits_of(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

BMC_HD double key_value(uint64_t k) {
    return double_of((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k);
}

BMC_HD bool is_nan(double v) {
    const uint64_t b = bits_of(v) & 0x7FFFFFFFFFFFFFFFull;
    return b > 0x7FF0000000000000ull;
}

// ------------------------------------------------------ superaccumulator
constexpr int kLimbs = 67;  // 67 x 32 bits >= 2^-1074 .. 2^1024 + 32 carry bits

// Split |v| (finite) into its three 32-bit limb contributions starting at
// limb *L: |v| = (w0 + w1 2^32 + w2 2^64) 2^(32 L - 1074).
BMC_HD void split(double v, int* L, uint32_t* w0, uint32_t* w1, uint32_t* w2) {
    const uint64_t b = bits_of(v);
    const uint32_t e = static_cast<uint32_t>((b >> 52) & 0x7FFu);
    uint64_t m = b & 0x000FFFFFFFFFFFFFull;
    if (e) m |= 0x0010000000000000ull;
    const uint32_t p = e ? e - 1u : 0u;  // bit position of the significand's LSB
    const uint32_t sh = p & 31u;
    *L = static_cast<int>(p >> 5);
    *w0 = static_cast<uint32_t>(m << sh);
    *w1 = static_cast<uint32_t>(sh ? (m >> (32u - sh)) : (m >> 32));
    *w2 = sh ? static_cast<uint32_t>(m >> (64u - sh)) : 0u;
}

// Special-value classes a sum can meet (counted, never accumulated).
enum Special : int { kFinite = 0, kNaN = 1, kPosInf = 2, kNegInf = 3 };

BMC_HD int special_of(double v) {
    const uint64_t b = bits_of(v);
    if (((b >> 52) & 0x7FFu) != 0x7FFu) return kFinite;
    if (b & 0x000FFFFFFFFFFFFFull) return kNaN;
    return (b >> 63) ? kNegInf : kPosInf;
}

// Host-side scalar accumulation (device code uses atomics on the same words).
BMC_HD void acc_add(uint64_t* pos, uint64_t* neg, uint64_t* special, double v) {
    const int s = special_of(v);
    if (s != kFinite) {
        special[s - 1] += 1;
        return;
    }
    int L;
    uint32_t w0, w1, w2;
    split(v, &L, &w0, &w1, &w2);
    uint64_t* a = (bits_of(v) >> 63) ? neg : pos;
    a[L] += w0;
    a[L + 1] += w1;
    a[L + 2] += w2;
}

// Carry-normalise limb counters into 32-bit digits (in place).  Each input
// limb must be < 2^64 - 2^33 (any sum of < 2^32 - 1 contributions is).
BMC_HD void normalize(uint64_t* a) {
    uint64_t carry = 0;
    for (int i = 0; i < kLimbs; ++i) {
        const uint64_t t = a[i] + carry;
        a[i] = t & 0xFFFFFFFFull;
        carry = t >> 32;
    }
}

// bit q of a normalised digit array
BMC_HD uint32_t digit_bit(const uint64_t* d, int q) {
    return static_cast<uint32_t>((d[q >> 5] >> (q & 31)) & 1u);
}

// any set bit strictly below position q
BMC_HD bool any_below(const uint64_t* d, int q) {
    const int L = q >> 5;
    for (int i = 0; i < L; ++i)
        if (d[i]) return true;
    const uint64_t mask = (uint64_t{1} << (q & 31)) - 1u;
    return (d[L] & mask) != 0;
}

// Correctly rounded (ties to even) binary64 of pos - neg, both normalised.
// Returns +/-inf past DBL_MAX; +0.0 for an exactly zero difference.
BMC_HD double round_diff(const uint64_t* pos_in, const uint64_t* neg_in) {
    // compare magnitudes from the top digit
    int cmp = 0;
    for (int i = kLimbs - 1; i >= 0 && cmp == 0; --i) {
        if (pos_in[i] != neg_in[i]) cmp = pos_in[i] > neg_in[i] ? 1 : -1;
    }
    if (cmp == 0) return 0.0;
    const uint64_t* big = cmp > 0 ? pos_in : neg_in;
    const uint64_t* small = cmp > 0 ? neg_in : pos_in;
    uint64_t d[kLimbs];
    uint64_t borrow = 0;
    for (int i = 0; i < kLimbs; ++i) {
        const uint64_t sub = small[i] + borrow;
        if (big[i] >= sub) {
            d[i] = big[i] - sub;
            borrow = 0;
        } else {
            d[i] = (big[i] + 0x100000000ull) - sub;
            borrow = 1;
        }
    }
    int top = kLimbs - 1;
    while (top > 0 && d[top] == 0) --top;
    int t = top * 32 + 31;  // bit index of the most significant set bit
    while (((d[top] >> (t & 31)) & 1u) == 0) --t;
    uint64_t bits;
    if (t <= 52) {
        // < 2^53 units of 2^-1074: exactly representable; the bit pattern is
        // the integer itself (subnormal, or exponent field 1 at 2^52)
        bits = d[0] | (d[1] << 32);
    } else {
        // top 53 bits [t-52, t]
        uint64_t M = 0;
        for (int q = t; q >= t - 52; --q) M = (M << 1) | digit_bit(d, q);
        const uint32_t rbit = digit_bit(d, t - 53);
        const bool sticky = (t - 53) > 0 ? any_below(d, t - 53) : false;
        if (rbit && (sticky || (M & 1u))) {
            M += 1;
            if (M == (uint64_t{1} << 53)) {
                M >>= 1;
                t += 1;
            }
        }
        const int biased = t - 51;  // MSB at 2^(t-1074) -> exponent field t - 1074 + 1023
        if (biased >= 0x7FF) {
            bits = 0x7FF0000000000000ull;
        } else {
            bits = (static_cast<uint64_t>(biased) << 52) | (M & 0x000FFFFFFFFFFFFFull);
        }
    }
    if (cmp < 0) bits |= 0x8000000000000000ull;
    return double_of(bits);
}

// The sum a finite reduction of the specials + exact part rounds to.
BMC_HD double sum_value(const uint64_t* pos, const uint64_t* neg, const uint64_t* special) {
    const bool nan = special[kNaN - 1] != 0, pinf = special[kPosInf - 1] != 0,
               ninf = special[kNegInf - 1] != 0;
    if (nan || (pinf && ninf)) return double_of(0x7FF8000000000000ull);
    if (pinf) return double_of(0x7FF0000000000000ull);
    if (ninf) return double_of(0xFFF0000000000000ull);
    return round_diff(pos, neg);
}

// ----------------------------------------------------- word layouts
// Partials are flat u64 arrays so that a merge across CTAs, chunks or GPUs
// is one element-wise op per section: SUM for counts / limbs / histograms,
// MIN for the two extrema keys.  Superaccumulator limbs are exported
// NORMALISED (digits < 2^32) before a cross-GPU merge, so any world size
// sums without overflow.

// One exact sum: pos limbs, neg limbs, special counts {nan, +inf, -inf}.
constexpr int kAccWords = 2 * kLimbs + 3;

// P1 (pass 1 / rollout epilogue): SUM section
constexpr int kP1Count = 0;        // values accumulated
constexpr int kP1Horizon = 1;      // hit_horizon flags set
constexpr int kP1Acc = 2;          // exact sum of d (kAccWords)
constexpr int kP1Exceed = kP1Acc + kAccWords;  // m + 1 exceedance buckets
BMC_HD int p1_sum_words(int m) { return kP1Exceed + m + 1; }
// P1 MIN section: {order_key(min), ~order_key(max)}
constexpr int kP1MinWords = 2;

// P2 (pass 2 over the outputs, after the P1 scalars are known): SUM section
constexpr int kP2M2 = 0;               // exact sum of (d-mean)^2   (kAccWords)
constexpr int kP2M3 = kAccWords;       // exact sum of (d-mean)^3   (kAccWords)
constexpr int kP2Hist = 2 * kAccWords; // summary histogram (hist_cap words)
constexpr int kB1 = 4096;              // level-1 order-statistic buckets
BMC_HD int p2_sel_all(uint64_t hist_cap) { return kP2Hist + static_cast<int>(hist_cap); }
// level-1 counts of the horizon hits (rare): stoppers per bucket = all - hz
BMC_HD int p2_sel_hz(uint64_t hist_cap) { return p2_sel_all(hist_cap) + kB1; }
BMC_HD int p2_sum_words(uint64_t hist_cap) { return p2_sel_hz(hist_cap) + kB1; }

// Scalars derived from the merged P1 (finalize_p1), stored as u64 words.
struct Scalars {
    uint64_t n;            // merged count
    uint64_t horizon;      // merged horizon count
    uint64_t stopped;      // n - horizon
    double sum, mean, min, max;
    double lo, hi;         // histogram origin floor(min), ceil(max)
    uint64_t bins;         // summary histogram bins (analysis.cpp:61-63)
    uint64_t hist_overflow;// bins > hist_cap: histogram left to a follow-up pass
    double sel_lo, sel_scale;  // level-1 bucket = (d - sel_lo) * sel_scale
    double bin_width;
    uint64_t nan_count;    // NaN stop distances seen (order statistics exclude them)
};

// Exact order-statistic targets: the median ranks over all results and the
// min_safe_headway ranks over the stoppers.
constexpr int kMaxRisk = 16;
constexpr int kMaxTargets = 2 + kMaxRisk;
struct Target {
    uint64_t rank;       // 1-based rank in its population (0 = unused)
    uint64_t residual;   // rank within the level-1 bucket
    int32_t bucket;      // level-1 bucket holding the rank
    int32_t population;  // 0: all results, 1: stoppers (hit_horizon == 0)
    int32_t valid;       // 0: rank outside [1, population size]
    int32_t overflow;    // candidates exceeded capacity -> exact fallback
    uint64_t key;        // selected order key (valid && !overflow)
};

// ------------------------------------------------------------ helpers
// summarize's histogram index (analysis.cpp:67-71):
// (size_t)((d - lo) / bin_width) clamped to bins - 1.
BMC_HD uint64_t hist_index(double d, double lo, double bw, uint64_t bins) {
    const double q = BMC_DIV(BMC_SUB(d, lo), bw);
    // C++ double -> size_t truncates toward zero; values past the last bin
    // (and the +inf of a horizon-free overflow) clamp
    uint64_t idx;
    if (!(q < 18446744073709551616.0)) {
        idx = bins - 1;
    } else if (!(q >= 0.0)) {
        idx = 0;
    } else {
        idx = static_cast<uint64_t>(q);
    }
    return idx >= bins ? bins - 1 : idx;
}

// hist_index without the FP64 division on almost every value: the product
// with the rounded reciprocal is within 1.5 * 2^-52 relative of the exact
// quotient q = fl((d - lo) / bw), so floor(q) equals floor of the product
// unless an integer lies within 2^-48 relative of it; those values (and any
// out-of-range or NaN quotient) take the exact division.  Same bins, bit
// for bit, as hist_index (tests: tests/test_stats_stage.py edge batches and
// the device/host-twin comparisons).
BMC_HD uint64_t hist_index_fast(double d, double lo, double bw, double inv_bw, uint64_t bins) {
    const double x = BMC_SUB(d, lo);
    const double qa = BMC_MUL(x, inv_bw);
    if (qa >= 0.0 && qa < 4503599627370496.0) {  // below 2^52: ulp(qa) < 1
        const double fa = floor(qa);
        const double margin = BMC_MUL(qa, 3.552713678800501e-15);  // qa * 2^-48
        if (BMC_SUB(qa, fa) > margin && BMC_SUB(BMC_ADD(fa, 1.0), qa) > margin) {
            const uint64_t idx = static_cast<uint64_t>(fa);
            return idx >= bins ? bins - 1 : idx;
        }
    }
    return hist_index(d, lo, bw, bins);
}

// Level-1 order-statistic bucket: monotone non-decreasing in d.
BMC_HD int sel_bucket(double d, double lo, double scale) {
    const double q = BMC_MUL(BMC_SUB(d, lo), scale);
    if (!(q < static_cast<double>(kB1))) return kB1 - 1;
    if (!(q >= 0.0)) return 0;
    return static_cast<int>(q);
}

// Sorted-threshold bucket p = #{H_j < d}, or m for a horizon hit; count_j =
// #{p > j} is collision_probability's numerator at H_j (analysis.cpp:152-157).
BMC_HD int exceed_bucket(const double* H, int m, double d, bool horizon) {
    if (horizon) return m;
    int lo = 0, hi = m;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (H[mid] < d) {
            lo = mid + 1;
        } else {
            hi = mid;
        }
    }
    return lo;
}

// min_safe_headway's nudged rank (analysis.cpp:182-185):
// ceil(raw - raw * 1e-12), raw = (1 - risk) * n.
BMC_HD uint64_t risk_rank(double risk, uint64_t n) {
    const double raw = BMC_MUL(BMC_SUB(1.0, risk), static_cast<double>(n));
    const double r = ceil(BMC_SUB(raw, BMC_MUL(raw, 1e-12)));
    return r <= 0.0 ? 0 : static_cast<uint64_t>(r);
}

// Scalars from the merged P1 (all IEEE ops: identical on host and device).
BMC_HD void finalize_p1(const uint64_t* p1_sum, const uint64_t* p1_min, double bin_width,
                        uint64_t hist_cap, uint64_t* work /* 2*kLimbs scratch */,
                        Scalars* s) {
    s->n = p1_sum[kP1Count];
    s->horizon = p1_sum[kP1Horizon];
    s->stopped = s->n - s->horizon;
    s->bin_width = bin_width;
    const uint64_t* acc = p1_sum + kP1Acc;
    for (int i = 0; i < kLimbs; ++i) {
        work[i] = acc[i];
        work[kLimbs + i] = acc[kLimbs + i];
    }
    normalize(work);
    normalize(work + kLimbs);
    const uint64_t* special = acc + 2 * kLimbs;
    s->nan_count = special[kNaN - 1];
    s->sum = sum_value(work, work + kLimbs, special);
    const double dn = static_cast<double>(s->n);
    s->mean = s->n ? BMC_DIV(s->sum, dn) : 0.0;  // analysis.cpp:38
    s->min = key_value(p1_min[0]);
    s->max = key_value(~p1_min[1]);
    // analysis.cpp:59-63
    s->lo = floor(s->min);
    s->hi = ceil(s->max);
    s->bins = 0;
    s->hist_overflow = 0;
    if (bin_width > 0.0 && s->n) {
        const double nb = ceil(BMC_DIV(BMC_SUB(s->hi, s->lo), bin_width));
        uint64_t bins;
        if (!(nb < 18446744073709551616.0)) {
            bins = ~uint64_t{0};
        } else {
            bins = nb >= 1.0 ? static_cast<uint64_t>(nb) : 0;
        }
        s->bins = bins < 1 ? 1 : bins;
        s->hist_overflow = s->bins > hist_cap ? 1 : 0;
    }
    s->sel_lo = s->min;
    const double span = BMC_SUB(s->max, s->min);
    const double scale = span > 0.0 ? BMC_DIV(static_cast<double>(kB1), span) : 0.0;
    // an infinite span (or scale) puts everything in one bucket: still exact
    s->sel_scale = (scale < 1.7976931348623157e308) ? scale : 0.0;
}

}  // namespace sc
// ------------------------------------------------- device stage views
// (plain structs passed by value to the stage kernels; word offsets into
// one u64 allocation laid out by make_layout in bmc_stats_pipeline.h)
struct StageDev {
    unsigned long long* w;
    size_t p1_min, p1_sum, p2_sum, cand_count, scal, targets, risks, cand;
    int m, n_risk, n_targets, summary;
    uint64_t hist_cap, cand_cap;
    double bin_width;
};

// Where the select stage finds each target's candidates: G segments (one per
// rank) of len[t] keys at base[t] + r * rank_stride; UINT64_MAX keys are pads.
struct SelectSegments {
    uint64_t base[sc::kMaxTargets];
    uint64_t len[sc::kMaxTargets];
    uint64_t rank_stride;
    int world;
    int use_counts;  // clamp len[t] by the local candidate count (single-rank layout)
    int in_gather;   // base[] is relative to the merge scratch, not the stage memory
};

// Local candidates -> one padded block: target t's P_t keys at off[t]
// (UINT64_MAX pads after the local count); total = sum of P_t.
struct PackArgs {
    uint64_t off[sc::kMaxTargets];
    uint64_t total;
};

}  // namespace bmc
