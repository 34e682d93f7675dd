// bmc_stats.cu -- on-device outcome statistics over the compact rollout
// outputs (stop_distance f64, hit_horizon u8), replacing the host passes of
// analysis.cpp (/root/reference/proj/src/analysis.cpp:13-228).
//
// All of these are HBM-streaming reductions (9 B read per sample per pass):
//   * extrema + horizon count + compensated sum     (summarize, :13-37)
//   * compensated second / third central moments    (summarize, :39-50)
//   * fixed-origin histogram, integer counts        (summarize, :61-75)
//   * exceedance counts for m headways in one pass  (collision_probability,
//     :145-159, and build_risk_curve's grid, :203-228: O(n log m), not O(n m))
//   * exact order statistics by 8-bit radix select  (median :51-57,
//     min_safe_headway :161-194)
// Integer counts, extrema and order statistics are exact.  Sums use
// double-double (TwoSum) accumulation in a fixed reduction order, so they
// are deterministic and within a few ulp of the exact sum; the reference's
// own sequential sum is only within n*eps of it (tolerance stated in tests).
#include "bmc_stats.h"

#include <cfloat>

namespace bmc {
namespace {

struct DD {
    double hi, lo;
};

__device__ __forceinline__ DD dd_add(DD a, double b) {
    // TwoSum(a.hi, b) then fold the low parts
    const double s = __dadd_rn(a.hi, b);
    const double bb = __dsub_rn(s, a.hi);
    const double err = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return DD{s, __dadd_rn(a.lo, err)};
}

__device__ __forceinline__ DD dd_merge(DD a, DD b) {
    DD r = dd_add(a, b.hi);
    r.lo = __dadd_rn(r.lo, b.lo);
    return r;
}

template <class T, class Op>
__device__ __forceinline__ T warp_reduce(T v, Op op) {
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ DD warp_reduce_dd(DD v) {
    for (int o = 16; o > 0; o >>= 1) {
        DD w{__shfl_down_sync(0xffffffffu, v.hi, o), __shfl_down_sync(0xffffffffu, v.lo, o)};
        v = dd_merge(v, w);
    }
    return v;
}

constexpr int kStatsBlock = 256;

// Pass 1: min / max / horizon count / sum.  One partial per block.
__global__ void __launch_bounds__(kStatsBlock) reduce_kernel(const double* d, const uint8_t* hz,
                                                             uint64_t n, BlockPartial* out) {
    double mn = DBL_MAX, mx = -DBL_MAX;
    unsigned long long hcount = 0, count = 0;
    DD sum{0.0, 0.0};
    bool any_nan = false;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        const double v = d[i];
        any_nan |= (v != v);
        mn = fmin(mn, v);
        mx = fmax(mx, v);
        sum = dd_add(sum, v);
        if (hz && hz[i]) ++hcount;
        ++count;
    }
    __shared__ double s_mn[32], s_mx[32], s_hi[32], s_lo[32];
    __shared__ unsigned long long s_h[32], s_c[32];
    __shared__ int s_nan[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    mn = warp_reduce(mn, [](double a, double b) { return fmin(a, b); });
    mx = warp_reduce(mx, [](double a, double b) { return fmax(a, b); });
    hcount = warp_reduce(hcount, [](unsigned long long a, unsigned long long b) { return a + b; });
    count = warp_reduce(count, [](unsigned long long a, unsigned long long b) { return a + b; });
    const int nanw = __any_sync(0xffffffffu, any_nan);
    sum = warp_reduce_dd(sum);
    if (lane == 0) {
        s_mn[wid] = mn;
        s_mx[wid] = mx;
        s_hi[wid] = sum.hi;
        s_lo[wid] = sum.lo;
        s_h[wid] = hcount;
        s_c[wid] = count;
        s_nan[wid] = nanw;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        BlockPartial p{};
        p.min = DBL_MAX;
        p.max = -DBL_MAX;
        DD s{0.0, 0.0};
        for (int w = 0; w < kStatsBlock / 32; ++w) {
            p.min = fmin(p.min, s_mn[w]);
            p.max = fmax(p.max, s_mx[w]);
            s = dd_merge(s, DD{s_hi[w], s_lo[w]});
            p.horizon += s_h[w];
            p.count += s_c[w];
            p.nan |= s_nan[w];
        }
        p.sum_hi = s.hi;
        p.sum_lo = s.lo;
        out[blockIdx.x] = p;
    }
}

// Pass 2: sum of dev^2 and dev^3 with dev = d - mean (analysis.cpp:39-45).
__global__ void __launch_bounds__(kStatsBlock) moments_kernel(const double* d, uint64_t n,
                                                              double mean, MomentPartial* out) {
    DD m2{0.0, 0.0}, m3{0.0, 0.0};
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        const double dev = __dsub_rn(d[i], mean);
        const double sq = __dmul_rn(dev, dev);
        m2 = dd_add(m2, sq);
        m3 = dd_add(m3, __dmul_rn(sq, dev));
    }
    __shared__ double s[4][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    m2 = warp_reduce_dd(m2);
    m3 = warp_reduce_dd(m3);
    if (lane == 0) {
        s[0][wid] = m2.hi;
        s[1][wid] = m2.lo;
        s[2][wid] = m3.hi;
        s[3][wid] = m3.lo;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        DD a{0.0, 0.0}, b{0.0, 0.0};
        for (int w = 0; w < kStatsBlock / 32; ++w) {
            a = dd_merge(a, DD{s[0][w], s[1][w]});
            b = dd_merge(b, DD{s[2][w], s[3][w]});
        }
        out[blockIdx.x] = MomentPartial{a.hi, a.lo, b.hi, b.lo};
    }
}

// Histogram anchored at `lo` (analysis.cpp:61-75): idx = (size_t)((d-lo)/bw),
// clamped to bins-1.  Privatised in shared memory when it fits.
constexpr int kSmemBins = 8192;

__global__ void __launch_bounds__(kStatsBlock) hist_kernel(const double* d, uint64_t n, double lo,
                                                           double bw, uint64_t bins,
                                                           unsigned long long* hist) {
    __shared__ unsigned int s_hist[kSmemBins];
    const bool priv = bins <= kSmemBins;
    if (priv) {
        for (uint64_t b = threadIdx.x; b < bins; b += blockDim.x) s_hist[b] = 0u;
        __syncthreads();
    }
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        const double q = __ddiv_rn(__dsub_rn(d[i], lo), bw);
        // C++ double -> size_t conversion truncates toward zero
        uint64_t idx = static_cast<uint64_t>(q);
        if (idx >= bins) idx = bins - 1;
        if (priv) {
            atomicAdd(&s_hist[idx], 1u);
        } else {
            atomicAdd(&hist[idx], 1ull);
        }
    }
    if (priv) {
        __syncthreads();
        for (uint64_t b = threadIdx.x; b < bins; b += blockDim.x) {
            if (s_hist[b]) atomicAdd(&hist[b], static_cast<unsigned long long>(s_hist[b]));
        }
    }
}

// Exceedance buckets: p(d) = #{sorted headways H < d}; horizon -> m.
// counts for sorted headway j = sum_{p > j} bucket[p] (suffix sum on host).
constexpr int kSmemHeadways = 4000;

__global__ void __launch_bounds__(kStatsBlock) exceed_kernel(const double* d, const uint8_t* hz,
                                                             uint64_t n, const double* sorted_h,
                                                             int m, unsigned long long* buckets) {
    __shared__ double s_h[kSmemHeadways];
    __shared__ unsigned int s_b[kSmemHeadways + 1];
    const bool priv = m <= kSmemHeadways;
    const double* H = sorted_h;
    if (priv) {
        for (int k = threadIdx.x; k < m; k += blockDim.x) s_h[k] = sorted_h[k];
        for (int k = threadIdx.x; k <= m; k += blockDim.x) s_b[k] = 0u;
        __syncthreads();
        H = s_h;
    }
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        int p;
        if (hz && hz[i]) {
            p = m;
        } else {
            const double v = d[i];
            // lower_bound over H for the first H >= v, i.e. p = #{H < v}
            int lo = 0, hi = m;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (H[mid] < v) {
                    lo = mid + 1;
                } else {
                    hi = mid;
                }
            }
            p = lo;
        }
        if (priv) {
            atomicAdd(&s_b[p], 1u);
        } else {
            atomicAdd(&buckets[p], 1ull);
        }
    }
    if (priv) {
        __syncthreads();
        for (int k = threadIdx.x; k <= m; k += blockDim.x) {
            if (s_b[k]) atomicAdd(&buckets[k], static_cast<unsigned long long>(s_b[k]));
        }
    }
}

// Order-preserving map double -> uint64 (total order for non-NaN values).
__device__ __forceinline__ uint64_t order_key(double v) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// One radix-select pass: for every target t whose key prefix (bits above
// `shift`+8) matches, histogram the next 8-bit digit.
__global__ void __launch_bounds__(kStatsBlock) select_kernel(const double* d, const uint8_t* hz,
                                                             uint64_t n, int exclude_horizon,
                                                             int shift, const uint64_t* prefixes,
                                                             int targets,
                                                             unsigned long long* hist) {
    __shared__ unsigned int s_hist[kMaxSelectTargets * 256];
    __shared__ uint64_t s_pref[kMaxSelectTargets];
    for (int k = threadIdx.x; k < targets * 256; k += blockDim.x) s_hist[k] = 0u;
    for (int k = threadIdx.x; k < targets; k += blockDim.x) s_pref[k] = prefixes[k];
    __syncthreads();
    const uint64_t mask = (shift >= 56) ? 0ull : (~0ull << (shift + 8));
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        if (exclude_horizon && hz && hz[i]) continue;
        const uint64_t key = order_key(d[i]);
        const unsigned digit = static_cast<unsigned>((key >> shift) & 0xffu);
        for (int t = 0; t < targets; ++t) {
            if ((key & mask) == s_pref[t]) atomicAdd(&s_hist[t * 256 + digit], 1u);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < targets * 256; k += blockDim.x) {
        if (s_hist[k]) atomicAdd(&hist[k], static_cast<unsigned long long>(s_hist[k]));
    }
}

int stats_grid(uint64_t n) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t need = (n + kStatsBlock - 1) / kStatsBlock;
    const uint64_t cap = static_cast<uint64_t>(sms) * 8;
    return static_cast<int>(need < cap ? (need ? need : 1) : cap);
}

}  // namespace

int stats_partials(uint64_t n) { return stats_grid(n); }

cudaError_t launch_reduce(const double* d, const uint8_t* hz, uint64_t n, BlockPartial* out,
                          cudaStream_t s) {
    reduce_kernel<<<stats_grid(n), kStatsBlock, 0, s>>>(d, hz, n, out);
    return cudaGetLastError();
}

cudaError_t launch_moments(const double* d, uint64_t n, double mean, MomentPartial* out,
                           cudaStream_t s) {
    moments_kernel<<<stats_grid(n), kStatsBlock, 0, s>>>(d, n, mean, out);
    return cudaGetLastError();
}

cudaError_t launch_hist(const double* d, uint64_t n, double lo, double bw, uint64_t bins,
                        unsigned long long* hist, cudaStream_t s) {
    hist_kernel<<<stats_grid(n), kStatsBlock, 0, s>>>(d, n, lo, bw, bins, hist);
    return cudaGetLastError();
}

cudaError_t launch_exceed(const double* d, const uint8_t* hz, uint64_t n, const double* sorted_h,
                          int m, unsigned long long* buckets, cudaStream_t s) {
    exceed_kernel<<<stats_grid(n), kStatsBlock, 0, s>>>(d, hz, n, sorted_h, m, buckets);
    return cudaGetLastError();
}

cudaError_t launch_select(const double* d, const uint8_t* hz, uint64_t n, int exclude_horizon,
                          int shift, const uint64_t* prefixes, int targets,
                          unsigned long long* hist, cudaStream_t s) {
    if (targets < 1 || targets > kMaxSelectTargets) return cudaErrorInvalidValue;
    select_kernel<<<stats_grid(n), kStatsBlock, 0, s>>>(d, hz, n, exclude_horizon, shift,
                                                        prefixes, targets, hist);
    return cudaGetLastError();
}

}  // namespace bmc
