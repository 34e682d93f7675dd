// bmc_fused_stats.cu -- kernels of the fused statistics stage (orchestrated
// by bmc_stats_pipeline.h; arithmetic in bmc_stats_core.h).  Replaces the
// host passes of /root/reference/proj/src/analysis.cpp:13-228.
//
// HBM traffic per result: pass 1 is free when fused into the rollout
// epilogue (else 9 B); pass 2 reads d + hit_horizon once (9 B); compaction
// reads them once more (9 B) and writes only the ~1e-3 of values in the
// buckets holding a target rank.  Everything else touches O(buckets) words.
// Bound: HBM (3 x 9 B/result at most), not arithmetic.
#include "bmc_stats.h"
#include "bmc_stats_dev.cuh"

#include <cub/block/block_scan.cuh>

namespace bmc {
namespace {

constexpr int kPassThreads = 1024;
constexpr int kSmemHistBins = 8192;

int grid_for(uint64_t n, int sms, int per_sm, int threads) {
    const uint64_t need = (n + threads - 1) / threads;
    const uint64_t cap = static_cast<uint64_t>(sms > 0 ? sms : 148) * per_sm;
    return static_cast<int>(need < 1 ? 1 : (need < cap ? need : cap));
}

// Streaming loop over (d[i], hz[i]): when d is 16-B and hz 4-B aligned, each
// thread takes groups of 4 consecutive results (two 16-B loads + one 4-B
// load), kGroups groups in flight, consecutive threads on consecutive groups
// -- a warp reads 1 KB of d contiguously (ncu: the strided 8-B form left
// pass 2 at 0.83 TB/s and compaction at 1.35 TB/s).  f(i, v, h) per result;
// LOAD_HZ false passes h = 0 and leaves hz to f.
#ifndef BMC_STREAM_LD
#define BMC_STREAM_LD 0
#endif
template <class T>
__device__ __forceinline__ T stream_ld(const T* p) {
    if (BMC_STREAM_LD == 1) return __ldg(p);
    if (BMC_STREAM_LD == 2) return *p;
    return __ldcs(p);
}
// Software-pipelined: the next group's loads are issued before the current
// group is processed (the per-result work ends in atomics / stores the
// compiler cannot hoist later loads above).
template <bool LOAD_HZ, class F>
__device__ __forceinline__ void stream_results(const double* d, const uint8_t* hz, uint64_t n, F&& f) {
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const bool vec = (reinterpret_cast<uintptr_t>(d) & 15u) == 0 &&
                     (!LOAD_HZ || hz == nullptr || (reinterpret_cast<uintptr_t>(hz) & 3u) == 0);
    if (!vec) {
        for (uint64_t i = tid; i < n; i += stride) f(i, d[i], LOAD_HZ && hz != nullptr ? hz[i] : 0);
        return;
    }
    const uint64_t ng = n / 4;
    const double2* d2 = reinterpret_cast<const double2*>(d);
    const uint32_t* h4 = reinterpret_cast<const uint32_t*>(hz);
    uint64_t g = tid;
    double2 a = make_double2(0.0, 0.0), b = a;
    uint32_t h = 0u;
    if (g < ng) {
        a = stream_ld(d2 + 2 * g);
        b = stream_ld(d2 + 2 * g + 1);
        if (LOAD_HZ && hz != nullptr) h = stream_ld(h4 + g);
    }
    for (; g < ng; g += stride) {
        const double2 ca = a, cb = b;
        const uint32_t ch = h;
        const uint64_t gn = g + stride;
        if (gn < ng) {
            a = stream_ld(d2 + 2 * gn);
            b = stream_ld(d2 + 2 * gn + 1);
            if (LOAD_HZ && hz != nullptr) h = stream_ld(h4 + gn);
        }
        f(4 * g, ca.x, ch & 0xffu);
        f(4 * g + 1, ca.y, (ch >> 8) & 0xffu);
        f(4 * g + 2, cb.x, (ch >> 16) & 0xffu);
        f(4 * g + 3, cb.y, ch >> 24);
    }
    for (uint64_t i = 4 * ng + tid; i < n; i += stride) f(i, d[i], LOAD_HZ && hz != nullptr ? hz[i] : 0);
}

// Per-thread register window over kWin consecutive limbs of one exact sum
// (one sign).  A value whose three limb contributions fall inside the
// window adds to registers; otherwise the window is flushed to the CTA's
// shared-memory limbs and re-based.  Stop distances (and their deviations)
// span a few binades, i.e. one or two 32-bit limb positions, so the streaming
// passes do no shared-memory atomics per value -- same-address u64 atomics
// from 32 lanes would serialise (measured 0.65 ms per 2e6 values).
constexpr int kWin = 4;
struct RegWin {
    int L0;
    unsigned long long w[kWin];
};

__device__ __forceinline__ void win_init(RegWin& r) {
    r.L0 = -1000;  // empty: every first add re-bases
#pragma unroll
    for (int k = 0; k < kWin; ++k) r.w[k] = 0ull;
}

__device__ __forceinline__ void win_flush(RegWin& r, unsigned long long* limbs) {
    if (r.L0 >= 0) {
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            if (r.w[k]) atomicAdd(&limbs[r.L0 + k], r.w[k]);
            r.w[k] = 0ull;
        }
    }
}

__device__ __forceinline__ void win_add(RegWin& r, unsigned long long* limbs, int L, uint32_t w0,
                                        uint32_t w1, uint32_t w2) {
    // a re-based window sits one limb below the value (L0 = L - 1), so the
    // common offsets are 1 and 0: straight-line adds, no dynamic indexing
    int off = L - r.L0;
    if (off != 1 && off != 0) {
        win_flush(r, limbs);
        r.L0 = min(max(L - 1, 0), sc::kLimbs - kWin);
        off = L - r.L0;
    }
    const bool hi = off == 1;
    r.w[0] += hi ? 0u : w0;
    r.w[1] += hi ? w0 : w1;
    r.w[2] += hi ? w1 : w2;
    r.w[3] += hi ? w2 : 0u;
}

// One exact sum's per-thread state: a window per sign + special counts.
struct RegAcc {
    RegWin pos, neg;
    unsigned long long nan, pinf, ninf;
};

__device__ __forceinline__ void racc_init(RegAcc& a) {
    win_init(a.pos);
    win_init(a.neg);
    a.nan = a.pinf = a.ninf = 0ull;
}

__device__ __forceinline__ void racc_add(RegAcc& a, unsigned long long* acc, double v) {
    const int sp = sc::special_of(v);
    if (sp != sc::kFinite) {
        a.nan += sp == sc::kNaN ? 1ull : 0ull;
        a.pinf += sp == sc::kPosInf ? 1ull : 0ull;
        a.ninf += sp == sc::kNegInf ? 1ull : 0ull;
        return;
    }
    int L;
    uint32_t w0, w1, w2;
    sc::split(v, &L, &w0, &w1, &w2);
    if (sc::bits_of(v) >> 63) {
        win_add(a.neg, acc + sc::kLimbs, L, w0, w1, w2);
    } else {
        win_add(a.pos, acc, L, w0, w1, w2);
    }
}

// A signed sum (m3: (dev*dev)*dev) in ONE window of signed limbs: a negative
// term subtracts its limb words, so the sign never splits the warp (two
// windows, one per sign, ran both paths for ~half the lanes each: ncu
// showed the m3 update at 16 active threads).  At the flush a positive
// limb adds to the CTA's positive limbs and a negative one to the negative
// limbs -- the same exact value.  int64 limbs: < 2^31 terms per thread.
struct RegWinS {
    int L0;
    long long w[kWin];
};
struct RegAccS {
    RegWinS win;
    unsigned long long nan, pinf, ninf;
};

__device__ __forceinline__ void wins_flush(RegWinS& r, unsigned long long* acc) {
    if (r.L0 >= 0) {
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            const long long v = r.w[k];
            if (v > 0) atomicAdd(&acc[r.L0 + k], static_cast<unsigned long long>(v));
            if (v < 0) atomicAdd(&acc[sc::kLimbs + r.L0 + k], static_cast<unsigned long long>(-v));
            r.w[k] = 0;
        }
    }
}

__device__ __forceinline__ void racc_init(RegAccS& a) {
    a.win.L0 = -1000;
#pragma unroll
    for (int k = 0; k < kWin; ++k) a.win.w[k] = 0;
    a.nan = a.pinf = a.ninf = 0ull;
}

__device__ __forceinline__ void racc_add(RegAccS& a, unsigned long long* acc, double v) {
    const int sp = sc::special_of(v);
    if (sp != sc::kFinite) {
        a.nan += sp == sc::kNaN ? 1ull : 0ull;
        a.pinf += sp == sc::kPosInf ? 1ull : 0ull;
        a.ninf += sp == sc::kNegInf ? 1ull : 0ull;
        return;
    }
    int L;
    uint32_t w0, w1, w2;
    sc::split(v, &L, &w0, &w1, &w2);
    const bool neg = (sc::bits_of(v) >> 63) != 0;
    const long long s0 = neg ? -static_cast<long long>(w0) : static_cast<long long>(w0);
    const long long s1 = neg ? -static_cast<long long>(w1) : static_cast<long long>(w1);
    const long long s2 = neg ? -static_cast<long long>(w2) : static_cast<long long>(w2);
    RegWinS& r = a.win;
    int off = L - r.L0;
    if (off != 1 && off != 0) {
        wins_flush(r, acc);
        r.L0 = min(max(L - 1, 0), sc::kLimbs - kWin);
        off = L - r.L0;
    }
    const bool hi = off == 1;  // straight-line: both offsets as selects
    r.w[0] += hi ? 0 : s0;
    r.w[1] += hi ? s0 : s1;
    r.w[2] += hi ? s1 : s2;
    r.w[3] += hi ? s2 : 0;
}

__device__ __forceinline__ void racc_flush(RegAccS& a, unsigned long long* acc) {
    wins_flush(a.win, acc);
    if (a.nan) atomicAdd(&acc[2 * sc::kLimbs + sc::kNaN - 1], a.nan);
    if (a.pinf) atomicAdd(&acc[2 * sc::kLimbs + sc::kPosInf - 1], a.pinf);
    if (a.ninf) atomicAdd(&acc[2 * sc::kLimbs + sc::kNegInf - 1], a.ninf);
}

// A sum of non-negative terms (m2: dev*dev >= +0): one window, no sign test.
struct RegAccPos {
    RegWin pos;
    unsigned long long nan, pinf;
};

__device__ __forceinline__ void racc_init(RegAccPos& a) {
    win_init(a.pos);
    a.nan = a.pinf = 0ull;
}

__device__ __forceinline__ void racc_add(RegAccPos& a, unsigned long long* acc, double v) {
    const int sp = sc::special_of(v);
    if (sp != sc::kFinite) {
        a.nan += sp == sc::kNaN ? 1ull : 0ull;
        a.pinf += sp == sc::kPosInf ? 1ull : 0ull;
        return;
    }
    int L;
    uint32_t w0, w1, w2;
    sc::split(v, &L, &w0, &w1, &w2);
    win_add(a.pos, acc, L, w0, w1, w2);
}

__device__ __forceinline__ void racc_flush(RegAccPos& a, unsigned long long* acc) {
    win_flush(a.pos, acc);
    if (a.nan) atomicAdd(&acc[2 * sc::kLimbs + sc::kNaN - 1], a.nan);
    if (a.pinf) atomicAdd(&acc[2 * sc::kLimbs + sc::kPosInf - 1], a.pinf);
}

__device__ __forceinline__ void racc_flush(RegAcc& a, unsigned long long* acc) {
    win_flush(a.pos, acc);
    win_flush(a.neg, acc + sc::kLimbs);
    if (a.nan) atomicAdd(&acc[2 * sc::kLimbs + sc::kNaN - 1], a.nan);
    if (a.pinf) atomicAdd(&acc[2 * sc::kLimbs + sc::kPosInf - 1], a.pinf);
    if (a.ninf) atomicAdd(&acc[2 * sc::kLimbs + sc::kNegInf - 1], a.ninf);
}

// Pass 1 over existing outputs (no fused rollout): the same words as the
// rollout epilogue, with per-thread registers for the count, horizon count,
// extrema and exact sum; shared-memory atomics only for exceedance buckets.
__global__ void __launch_bounds__(kPassThreads) pass1_kernel(const double* d, const uint8_t* hz,
                                                             uint64_t n, P1Args a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const P1View v = p1_view(sm, a.m);
    p1_init(v, a);
    __syncthreads();
    RegAcc acc;
    racc_init(acc);
    unsigned long long cnt = 0, hcnt = 0, kmin = ~0ull, kinv = ~0ull;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        const double x = d[i];
        const bool h = hz != nullptr && hz[i] != 0;
        ++cnt;
        hcnt += h ? 1ull : 0ull;
        racc_add(acc, v.s->acc, x);
        if (!sc::is_nan(x)) {
            const unsigned long long k = sc::order_key(x);
            kmin = k < kmin ? k : kmin;
            kinv = ~k < kinv ? ~k : kinv;
        }
        if (a.m) atomicAdd(&v.b[sc::exceed_bucket(v.H, a.m, x, h)], 1u);
    }
    racc_flush(acc, v.s->acc);
    for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        hcnt += __shfl_xor_sync(0xffffffffu, hcnt, o);
        const unsigned long long m1 = __shfl_xor_sync(0xffffffffu, kmin, o);
        const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, kinv, o);
        kmin = m1 < kmin ? m1 : kmin;
        kinv = m2 < kinv ? m2 : kinv;
    }
    if ((threadIdx.x & 31) == 0) {
        if (cnt) atomicAdd(&v.s->count, cnt);
        if (hcnt) atomicAdd(&v.s->horizon, hcnt);
        atomicMin(&v.s->min_key, kmin);
        atomicMin(&v.s->inv_max, kinv);
    }
    __syncthreads();
    p1_flush(v, a);
}

// Carry-normalise `accs` consecutive exact sums starting at word `off`
// (before a cross-GPU SUM merge: digits < 2^32 add without overflow).
__global__ void normalize_kernel(unsigned long long* w, size_t off, int accs) {
    const int k = threadIdx.x;
    if (k < 2 * accs) {
        uint64_t* p = reinterpret_cast<uint64_t*>(w + off + static_cast<size_t>(k / 2) * sc::kAccWords +
                                                  static_cast<size_t>(k % 2) * sc::kLimbs);
        sc::normalize(p);
    }
}

__global__ void finalize1_kernel(StageDev g) {
    uint64_t work[2 * sc::kLimbs];
    sc::finalize_p1(reinterpret_cast<const uint64_t*>(g.w + g.p1_sum),
                    reinterpret_cast<const uint64_t*>(g.w + g.p1_min), g.bin_width, g.hist_cap, work,
                    reinterpret_cast<sc::Scalars*>(g.w + g.scal));
}

struct P2Smem {
    unsigned long long acc[2 * sc::kAccWords];
    unsigned sel_all[sc::kB1];
    unsigned sel_hz[sc::kB1];
    unsigned hist[kSmemHistBins];
};

// Pass 2 (needs the merged P1 scalars): exact m2/m3 (analysis.cpp:39-46,
// dev*dev and (dev*dev)*dev rounded as written), the summarize histogram
// (:64-75) and the level-1 order-statistic histograms (all / stoppers).
// 256 threads x 3 CTAs per SM (80 registers): 875 us at 1e8 against 1.09 ms
// for 512 x 1 (122 registers), ncu, profiles/round2_hbm_stage_ab.txt
#ifndef BMC_P2_THREADS
#define BMC_P2_THREADS 256
#endif
#ifndef BMC_P2_MINB
#define BMC_P2_MINB 3
#endif
#ifndef BMC_P2_VEC
#define BMC_P2_VEC 0
#endif
constexpr int kPass2Threads = BMC_P2_THREADS;
constexpr int kPass2MinBlocks = BMC_P2_MINB;

__global__ void __launch_bounds__(kPass2Threads, kPass2MinBlocks) pass2_kernel(const double* d, const uint8_t* hz,
                                                                 uint64_t n, StageDev g) {
    extern __shared__ __align__(16) unsigned char sm[];
    P2Smem* S = reinterpret_cast<P2Smem*>(sm);
    const sc::Scalars s = *reinterpret_cast<const sc::Scalars*>(g.w + g.scal);
    const bool summary = g.summary != 0;
    const bool hist_on = summary && !s.hist_overflow;
    const bool hist_smem = hist_on && s.bins <= static_cast<uint64_t>(kSmemHistBins);
    unsigned long long* p2 = g.w + g.p2_sum;
    for (int i = threadIdx.x; i < 2 * sc::kAccWords; i += blockDim.x) S->acc[i] = 0ull;
    for (int i = threadIdx.x; i < sc::kB1; i += blockDim.x) {
        S->sel_all[i] = 0u;
        S->sel_hz[i] = 0u;
    }
    if (hist_smem) {
        for (uint64_t i = threadIdx.x; i < s.bins; i += blockDim.x) S->hist[i] = 0u;
    }
    __syncthreads();
    RegAccPos m2;
    RegAccS m3;
    racc_init(m2);
    racc_init(m3);
    const double inv_bw = BMC_DIV(1.0, s.bin_width);
    // a power-of-two bin width (the reference's default 2 m): d / bw == d * (1 / bw)
    // exactly (both are the correctly rounded scaling by 2^-k), no margin test
    const bool bw_pow2 = (sc::bits_of(s.bin_width) & 0x000FFFFFFFFFFFFFull) == 0 &&
                         s.bin_width > 0.0 && inv_bw < 1.0 / 0.0 && inv_bw > 0.0;
    auto one = [&](double v, bool h) {
        if (summary) {
            const double dev = BMC_SUB(v, s.mean);
            const double sq = BMC_MUL(dev, dev);
            racc_add(m2, S->acc, sq);
            racc_add(m3, S->acc + sc::kAccWords, BMC_MUL(sq, dev));
        }
        if (sc::is_nan(v)) return;
        if (hist_on) {
            uint64_t idx;
            if (bw_pow2) {
                const double q = BMC_MUL(BMC_SUB(v, s.lo), inv_bw);
                idx = !(q < 18446744073709551616.0) ? s.bins - 1
                      : (!(q >= 0.0) ? 0 : static_cast<uint64_t>(q));
                idx = idx >= s.bins ? s.bins - 1 : idx;
            } else {
                idx = sc::hist_index_fast(v, s.lo, s.bin_width, inv_bw, s.bins);
            }
            if (hist_smem) {
                atomicAdd(&S->hist[idx], 1u);
            } else {
                atomicAdd(&p2[sc::kP2Hist + idx], 1ull);
            }
        }
        const int b = sc::sel_bucket(v, s.sel_lo, s.sel_scale);
        atomicAdd(&S->sel_all[b], 1u);
        if (h) atomicAdd(&S->sel_hz[b], 1u);  // rare: one atomic per result, not two
    };
    if (BMC_P2_VEC) {
        stream_results<true>(d, hz, n, [&](uint64_t, double v, unsigned h) { one(v, h != 0); });
    } else {
        // four independent strided loads in flight per thread
        constexpr int kUnroll = 4;
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        for (; i + (kUnroll - 1) * stride < n; i += kUnroll * stride) {
            double v[kUnroll];
            uint8_t h[kUnroll];
#pragma unroll
            for (int k = 0; k < kUnroll; ++k) {
                v[k] = __ldcs(d + i + k * stride);
                h[k] = hz != nullptr ? __ldcs(hz + i + k * stride) : 0;
            }
#pragma unroll
            for (int k = 0; k < kUnroll; ++k) one(v[k], h[k] != 0);
        }
        for (; i < n; i += stride) one(d[i], hz != nullptr && hz[i] != 0);
    }
    racc_flush(m2, S->acc);
    racc_flush(m3, S->acc + sc::kAccWords);
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * sc::kAccWords; i += blockDim.x) {
        if (S->acc[i]) atomicAdd(&p2[sc::kP2M2 + i], S->acc[i]);
    }
    const int sa = sc::p2_sel_all(g.summary ? g.hist_cap : 0);
    const int ss = sc::p2_sel_hz(g.summary ? g.hist_cap : 0);
    for (int i = threadIdx.x; i < sc::kB1; i += blockDim.x) {
        if (S->sel_all[i]) atomicAdd(&p2[sa + i], static_cast<unsigned long long>(S->sel_all[i]));
        if (S->sel_hz[i]) atomicAdd(&p2[ss + i], static_cast<unsigned long long>(S->sel_hz[i]));
    }
    if (hist_smem) {
        for (uint64_t i = threadIdx.x; i < s.bins; i += blockDim.x) {
            if (S->hist[i]) atomicAdd(&p2[sc::kP2Hist + i], static_cast<unsigned long long>(S->hist[i]));
        }
    }
}

// Ranks of the order statistics (median ranks over all results,
// analysis.cpp:53-56; min_safe_headway ranks over the stoppers, :182-190)
// and the level-1 bucket + residual rank holding each.
constexpr int kTargetThreads = 1024;
constexpr int kPer = sc::kB1 / kTargetThreads;

__global__ void __launch_bounds__(kTargetThreads) targets_kernel(StageDev g) {
    using Scan = cub::BlockScan<unsigned long long, kTargetThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ sc::Target tg[sc::kMaxTargets];
    const sc::Scalars s = *reinterpret_cast<const sc::Scalars*>(g.w + g.scal);
    const double* risks = reinterpret_cast<const double*>(g.w + g.risks);
    if (threadIdx.x < sc::kMaxTargets) {
        const int t = threadIdx.x;
        sc::Target x{};
        x.bucket = -1;
        if (t < 2) {
            x.population = 0;
            if (g.summary && s.n) x.rank = (t == 0) ? ((s.n % 2 == 0) ? s.n / 2 : 0) : s.n / 2 + 1;
            x.valid = x.rank >= 1 && x.rank <= s.n - s.nan_count;
        } else if (t < 2 + g.n_risk) {
            x.population = 1;
            x.rank = sc::risk_rank(risks[t - 2], s.n);
            x.valid = x.rank >= 1 && x.rank <= s.stopped;
        }
        tg[t] = x;
    }
    __syncthreads();
    const unsigned long long* p2 = g.w + g.p2_sum;
    const int all = sc::p2_sel_all(g.summary ? g.hist_cap : 0);
    const int hzo = sc::p2_sel_hz(g.summary ? g.hist_cap : 0);
    for (int pop = 0; pop < 2; ++pop) {
        unsigned long long items[kPer], sum = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int b = threadIdx.x * kPer + k;
            // population 1 (stoppers) = all results - horizon hits, per bucket
            items[k] = p2[all + b] - (pop ? p2[hzo + b] : 0ull);
            sum += items[k];
        }
        unsigned long long excl = 0;
        Scan(tmp).ExclusiveSum(sum, excl);
        __syncthreads();
        for (int t = 0; t < g.n_targets; ++t) {
            sc::Target& x = tg[t];
            if (x.population != pop || !x.valid || x.rank == 0) continue;
            if (excl < x.rank && x.rank <= excl + sum) {
                unsigned long long cum = excl;
#pragma unroll
                for (int k = 0; k < kPer; ++k) {
                    if (cum + items[k] >= x.rank) {
                        x.bucket = static_cast<int32_t>(threadIdx.x * kPer + k);
                        x.residual = x.rank - cum;
                        break;
                    }
                    cum += items[k];
                }
            }
        }
        __syncthreads();
    }
    if (threadIdx.x < sc::kMaxTargets) {
        sc::Target x = tg[threadIdx.x];
        if (x.valid && x.bucket < 0) x.valid = 0;  // NaN-only remainder (no value to select)
        reinterpret_cast<sc::Target*>(g.w + g.targets)[threadIdx.x] = x;
    }
}

// Values in each target's bucket -> that target's candidate list (order
// keys).  A 4096-bit shared bitmap of the target buckets rejects almost
// every value with one shared load; hit_horizon is read only on a hit.
// Hits (~1e-3 of the values, ~1e5 at 1e8) gather in a per-CTA shared buffer
// and reserve their global slots with one atomic per target per CTA: one
// same-address global atomic per hit serialised in L2.
constexpr int kCandBuf = 128;
__global__ void __launch_bounds__(256) compact_kernel(const double* d, const uint8_t* hz, uint64_t n,
                                                      StageDev g) {
    __shared__ int s_bucket[sc::kMaxTargets];
    __shared__ int s_pop[sc::kMaxTargets];
    __shared__ unsigned s_map[sc::kB1 / 32];
    __shared__ unsigned s_cnt[sc::kMaxTargets];
    __shared__ unsigned long long s_base[sc::kMaxTargets];
    __shared__ unsigned long long s_buf[sc::kMaxTargets][kCandBuf];
    __shared__ int s_T;
    const sc::Scalars s = *reinterpret_cast<const sc::Scalars*>(g.w + g.scal);
    for (int i = threadIdx.x; i < sc::kB1 / 32; i += blockDim.x) s_map[i] = 0u;
    if (threadIdx.x < sc::kMaxTargets) s_cnt[threadIdx.x] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) {
        const sc::Target* tg = reinterpret_cast<const sc::Target*>(g.w + g.targets);
        int T = 0;
        for (int t = 0; t < g.n_targets; ++t) {
            const bool on = tg[t].valid && tg[t].rank && tg[t].bucket >= 0;
            s_bucket[t] = on ? tg[t].bucket : -1;
            s_pop[t] = tg[t].population;
            if (on) {
                T = t + 1;
                s_map[tg[t].bucket >> 5] |= 1u << (tg[t].bucket & 31);
            }
        }
        s_T = T;
    }
    __syncthreads();
    const int T = s_T;
    if (T == 0) return;
    unsigned long long* cnt = g.w + g.cand_count;
    unsigned long long* cand = g.w + g.cand;
    auto one = [&](uint64_t i, double v) {
        const int b = sc::sel_bucket(v, s.sel_lo, s.sel_scale);  // NaN -> bucket 0, filtered below
        if (!((s_map[b >> 5] >> (b & 31)) & 1u) || sc::is_nan(v)) return;
        const bool h = hz != nullptr && hz[i] != 0;
        const unsigned long long key = sc::order_key(v);
        for (int t = 0; t < T; ++t) {
            if (s_bucket[t] != b || (s_pop[t] == 1 && h)) continue;
            const unsigned p = atomicAdd(&s_cnt[t], 1u);
            if (p < kCandBuf) {
                s_buf[t][p] = key;
            } else {  // buffer full: straight to the global list
                const unsigned long long pos = atomicAdd(&cnt[t], 1ull);
                if (pos < g.cand_cap) cand[static_cast<uint64_t>(t) * g.cand_cap + pos] = key;
            }
        }
    };
    stream_results<false>(d, hz, n, [&](uint64_t i, double v, unsigned) { one(i, v); });
    __syncthreads();
    if (threadIdx.x < T) {
        const unsigned c = min(s_cnt[threadIdx.x], static_cast<unsigned>(kCandBuf));
        s_base[threadIdx.x] = c ? atomicAdd(&cnt[threadIdx.x], static_cast<unsigned long long>(c)) : 0ull;
    }
    __syncthreads();
    for (int t = 0; t < T; ++t) {
        const unsigned c = min(s_cnt[t], static_cast<unsigned>(kCandBuf));
        for (unsigned j = threadIdx.x; j < c; j += blockDim.x) {
            const unsigned long long pos = s_base[t] + j;
            if (pos < g.cand_cap) cand[static_cast<uint64_t>(t) * g.cand_cap + pos] = s_buf[t][j];
        }
    }
}

// Local candidates -> one padded block [t0: P0][t1: P1]... (UINT64_MAX pads).
__global__ void pack_kernel(StageDev g, PackArgs p, unsigned long long* dst) {
    const unsigned long long* cnt = g.w + g.cand_count;
    const unsigned long long* cand = g.w + g.cand;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < p.total;
         i += stride) {
        int t = 0;
        while (t + 1 < g.n_targets && i >= p.off[t + 1]) ++t;
        const uint64_t k = i - p.off[t];
        const uint64_t c = cnt[t] < g.cand_cap ? cnt[t] : g.cand_cap;
        dst[i] = k < c ? cand[static_cast<uint64_t>(t) * g.cand_cap + k] : ~0ull;
    }
}

// Exact selection of the residual-th smallest candidate key: repeated
// 14-bit bucketing of [lo, hi] (a level-1 bucket's keys span ~41 bits, so
// three rounds), each round keeping the bucket that holds the residual rank.
constexpr int kSelThreads = 1024;
constexpr int kSelBits = 14;
constexpr int kSelBins = 1 << kSelBits;
constexpr int kSelPer = kSelBins / kSelThreads;

template <class F>
__device__ __forceinline__ void for_keys(const unsigned long long* keys, const SelectSegments& seg,
                                         int t, uint64_t len, F&& f) {
    for (int r = 0; r < seg.world; ++r) {
        const unsigned long long* k = keys + seg.base[t] + static_cast<uint64_t>(r) * seg.rank_stride;
        uint64_t i = threadIdx.x;
        // four independent loads in flight per thread (L2-resident keys)
        for (; i + 3 * kSelThreads < len; i += 4 * kSelThreads) {
            const unsigned long long a = k[i], b = k[i + kSelThreads], c = k[i + 2 * kSelThreads],
                                     e = k[i + 3 * kSelThreads];
            f(a);
            f(b);
            f(c);
            f(e);
        }
        for (; i < len; i += kSelThreads) f(k[i]);
    }
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(StageDev g, SelectSegments seg,
                                                              const unsigned long long* keys) {
    using Scan = cub::BlockScan<unsigned, kSelThreads>;
    __shared__ typename Scan::TempStorage tmp;
    extern __shared__ __align__(16) unsigned hist[];  // kSelBins
    __shared__ unsigned long long s_lo[32], s_hi[32];
    __shared__ unsigned long long s_bin, s_res;
    const int t = blockIdx.x;
    sc::Target* tg = reinterpret_cast<sc::Target*>(g.w + g.targets) + t;
    if (!tg->valid || tg->rank == 0 || tg->overflow) return;
    uint64_t len = seg.len[t];
    if (seg.use_counts) {
        const unsigned long long c = g.w[g.cand_count + t];
        if (c > g.cand_cap) {
            if (threadIdx.x == 0) tg->overflow = 1;
            return;
        }
        len = c;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // min / max key over every rank's segment (pads excluded)
    unsigned long long lo = ~0ull, hi = 0ull;
    for_keys(keys, seg, t, len, [&](unsigned long long x) {
        if (x == ~0ull) return;
        lo = x < lo ? x : lo;
        hi = x > hi ? x : hi;
    });
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if (lane == 0) {
        s_lo[wid] = lo;
        s_hi[wid] = hi;
    }
    __syncthreads();
    lo = ~0ull;
    hi = 0ull;
    for (int w = 0; w < kSelThreads / 32; ++w) {
        lo = s_lo[w] < lo ? s_lo[w] : lo;
        hi = s_hi[w] > hi ? s_hi[w] : hi;
    }
    unsigned long long r = tg->residual;
    __syncthreads();
    while (lo < hi) {
        const unsigned long long span = hi - lo;
        const int nb = 64 - __clzll(static_cast<long long>(span));
        const int sh = nb > kSelBits ? nb - kSelBits : 0;
        for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) hist[i] = 0u;
        __syncthreads();
        const unsigned long long clo = lo, chi = hi;
        for_keys(keys, seg, t, len, [&](unsigned long long x) {
            if (x < clo || x > chi) return;  // also drops pads (~0 > hi)
            atomicAdd(&hist[(x - clo) >> sh], 1u);
        });
        __syncthreads();
        unsigned items[kSelPer], sum = 0;
#pragma unroll
        for (int q = 0; q < kSelPer; ++q) {
            items[q] = hist[threadIdx.x * kSelPer + q];
            sum += items[q];
        }
        unsigned excl = 0;
        if (threadIdx.x == 0) s_bin = ~0ull;
        Scan(tmp).ExclusiveSum(sum, excl);
        if (excl < r && r <= static_cast<unsigned long long>(excl) + sum) {
            unsigned long long cum = excl;
#pragma unroll
            for (int q = 0; q < kSelPer; ++q) {
                if (cum + items[q] >= r) {
                    s_bin = static_cast<unsigned long long>(threadIdx.x * kSelPer + q);
                    s_res = r - cum;
                    break;
                }
                cum += items[q];
            }
        }
        __syncthreads();
        const unsigned long long b = s_bin;
        if (b == ~0ull) {  // rank beyond the keys present: cannot happen for consistent partials
            if (threadIdx.x == 0) tg->valid = 0;
            return;
        }
        r = s_res;
        const unsigned long long nlo = lo + (b << sh);
        if (sh == 0) {
            lo = hi = nlo;
        } else {
            const unsigned long long nhi = nlo + ((1ull << sh) - 1ull);
            lo = nlo;
            hi = nhi < hi ? nhi : hi;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) tg->key = lo;
}

}  // namespace

cudaError_t launch_pass1(const double* d, const uint8_t* hz, uint64_t n, const P1Args& a, int sms,
                         cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const size_t smem = p1_smem_bytes(a.m);
    cudaError_t e = cudaFuncSetAttribute(pass1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    pass1_kernel<<<grid_for(n, sms, 1, kPassThreads), kPassThreads, smem, s>>>(d, hz, n, a);
    return cudaGetLastError();
}

cudaError_t launch_normalize(const StageDev& g, size_t off, int accs, cudaStream_t s) {
    normalize_kernel<<<1, 32, 0, s>>>(g.w, off, accs);
    return cudaGetLastError();
}

cudaError_t launch_finalize1(const StageDev& g, cudaStream_t s) {
    finalize1_kernel<<<1, 1, 0, s>>>(g);
    return cudaGetLastError();
}

cudaError_t launch_pass2(const double* d, const uint8_t* hz, uint64_t n, const StageDev& g, int sms,
                         cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const size_t smem = sizeof(P2Smem);
    cudaError_t e = cudaFuncSetAttribute(pass2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    pass2_kernel<<<grid_for(n, sms, kPass2MinBlocks, kPass2Threads), kPass2Threads, smem, s>>>(d, hz, n, g);
    return cudaGetLastError();
}

cudaError_t launch_targets(const StageDev& g, cudaStream_t s) {
    targets_kernel<<<1, kTargetThreads, 0, s>>>(g);
    return cudaGetLastError();
}

cudaError_t launch_compact(const double* d, const uint8_t* hz, uint64_t n, const StageDev& g,
                           int sms, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    compact_kernel<<<grid_for(n, sms, 8, 256), 256, 0, s>>>(d, hz, n, g);
    return cudaGetLastError();
}

cudaError_t launch_pack(const StageDev& g, const PackArgs& p, unsigned long long* dst, int sms,
                        cudaStream_t s) {
    if (p.total == 0) return cudaSuccess;
    pack_kernel<<<grid_for(p.total, sms, 4, 256), 256, 0, s>>>(g, p, dst);
    return cudaGetLastError();
}

cudaError_t launch_select_targets(const StageDev& g, const SelectSegments& seg,
                                  const unsigned long long* keys, cudaStream_t s) {
    if (g.n_targets < 1) return cudaSuccess;
    const size_t smem = kSelBins * sizeof(unsigned);
    const cudaError_t e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    select_kernel<<<g.n_targets, kSelThreads, smem, s>>>(g, seg, keys);
    return cudaGetLastError();
}

}  // namespace bmc
