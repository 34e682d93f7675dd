// bmc_capi_stats.cpp -- C-ABI of the on-device statistics (brakemc_cuda.h).
//
// The kernels (bmc_stats.cu) stream the compact device outputs; this file
// does the O(#blocks) / O(#bins) host composition with the reference's own
// formulas (analysis.cpp:13-76, 145-194).  g++ -ffp-contract=off.
#include "bmc_ctx.h"

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

double dd_value(DDh a) { return a.hi + a.lo; }

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

extern "C" {

int bmc_cuda_order_stats(bmc_ctx* ctx, const double* d, const uint8_t* hz, size_t n,
                         int exclude_horizon, const uint64_t* ranks, size_t m, double* out,
                         uint64_t* count_out) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (!d || (m && (!ranks || !out))) return fail(ctx, BMC_E_CONFIG, "order_stats: null argument");
    if (exclude_horizon && !hz) return fail(ctx, BMC_E_CONFIG, "order_stats: horizon flags required");
    ctx->last_launches = 0;
    if (n == 0) return fail(ctx, BMC_E_CONFIG, "risk: needs at least one result");
    return bmc::select_ranks(ctx, d, hz, n, exclude_horizon, ranks, m, out, count_out);
}

int bmc_cuda_summarize(bmc_ctx* ctx, const double* d, const uint8_t* hz, size_t n, double bin_width,
                       bmc_summary* out, uint64_t* hist, size_t hist_cap) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    // analysis.cpp:14-19
    if (n == 0) return fail(ctx, BMC_E_CONFIG, "summarize: needs at least one result");
    if (!(bin_width > 0.0)) return fail(ctx, BMC_E_CONFIG, "outputs.bin_width: must be > 0");
    if (!d || !out) return fail(ctx, BMC_E_CONFIG, "summarize: null argument");
    ctx->last_launches = 0;
    cudaStream_t s = ctx->stream;
    const int P = bmc::stats_partials(n);
    BMC_CK(ctx, ctx->partials.reserve(static_cast<size_t>(P) * sizeof(bmc::BlockPartial)));
    std::vector<bmc::BlockPartial> parts(P);
    BMC_CK(ctx, bmc::launch_reduce(d, hz, n, ctx->partials.as<bmc::BlockPartial>(), s));
    BMC_CK(ctx, cudaMemcpyAsync(parts.data(), ctx->partials.p, P * sizeof(bmc::BlockPartial),
                                cudaMemcpyDeviceToHost, s));
    BMC_CK(ctx, cudaStreamSynchronize(s));
    ctx->last_launches += 1;

    bmc_summary sm;
    std::memset(&sm, 0, sizeof sm);
    sm.n = n;
    double mn = std::numeric_limits<double>::max(), mx = -std::numeric_limits<double>::max();
    bmc::DDh sum;
    for (const auto& p : parts) {  // fixed block order: deterministic
        mn = std::fmin(mn, p.min);
        mx = std::fmax(mx, p.max);
        sum = bmc::dd_merge_h(sum, p.sum_hi, p.sum_lo);
        sm.horizon_count += p.horizon;
    }
    const double dn = static_cast<double>(n);
    sm.mean = bmc::dd_value(sum) / dn;

    std::vector<bmc::MomentPartial> mom(P);
    BMC_CK(ctx, ctx->partials.reserve(static_cast<size_t>(P) * sizeof(bmc::MomentPartial)));
    BMC_CK(ctx, bmc::launch_moments(d, n, sm.mean, ctx->partials.as<bmc::MomentPartial>(), s));
    BMC_CK(ctx, cudaMemcpyAsync(mom.data(), ctx->partials.p, P * sizeof(bmc::MomentPartial),
                                cudaMemcpyDeviceToHost, s));
    BMC_CK(ctx, cudaStreamSynchronize(s));
    ctx->last_launches += 1;
    bmc::DDh m2, m3;
    for (const auto& p : mom) {
        m2 = bmc::dd_merge_h(m2, p.m2_hi, p.m2_lo);
        m3 = bmc::dd_merge_h(m3, p.m3_hi, p.m3_lo);
    }
    const double M2 = bmc::dd_value(m2), M3 = bmc::dd_value(m3);
    // analysis.cpp:47-50
    sm.sd = n > 1 ? std::sqrt(M2 / (dn - 1.0)) : 0.0;
    const double var_pop = M2 / dn;
    sm.skewness = var_pop > 0.0 ? (M3 / dn) / std::pow(var_pop, 1.5) : 0.0;

    // analysis.cpp:51-57 -- exact order statistics (min/max are exact already)
    sm.min = mn;
    sm.max = mx;
    uint64_t ranks[2];
    double vals[2];
    size_t nr;
    if (n % 2 == 1) {
        ranks[0] = n / 2 + 1;
        nr = 1;
    } else {
        ranks[0] = n / 2;
        ranks[1] = n / 2 + 1;
        nr = 2;
    }
    uint32_t launches = ctx->last_launches;
    if ((rc = bmc::select_ranks(ctx, d, hz, n, 0, ranks, nr, vals, nullptr)) != BMC_OK) return rc;
    launches += ctx->last_launches;
    sm.median = nr == 1 ? vals[0] : 0.5 * (vals[0] + vals[1]);
    sm.right_skewed = sm.mean > sm.median ? 1 : 0;

    // analysis.cpp:59-75
    const double lo = std::floor(sm.min);
    const double hi = std::ceil(sm.max);
    const double nb = std::ceil((hi - lo) / bin_width);
    const uint64_t bins = std::max<uint64_t>(1, static_cast<uint64_t>(nb));
    sm.origin = lo;
    sm.bin_width = bin_width;
    sm.bins = bins;
    if (hist != nullptr) {
        if (hist_cap < bins) {
            *out = sm;
            return fail(ctx, BMC_E_RANGE, "summarize: histogram buffer smaller than bin count");
        }
        BMC_CK(ctx, ctx->hist_buf.reserve(bins * sizeof(unsigned long long)));
        BMC_CK(ctx, cudaMemsetAsync(ctx->hist_buf.p, 0, bins * sizeof(unsigned long long), s));
        BMC_CK(ctx, bmc::launch_hist(d, n, lo, bin_width, bins, ctx->hist_buf.as<unsigned long long>(), s));
        BMC_CK(ctx, cudaMemcpyAsync(hist, ctx->hist_buf.p, bins * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        BMC_CK(ctx, cudaStreamSynchronize(s));
        launches += 1;
    }
    ctx->last_launches = launches;
    *out = sm;
    return BMC_OK;
}

int bmc_cuda_exceedance_ttc_noise(bmc_ctx* ctx, const double* d, const uint8_t* hz, size_t n,
                                  uint64_t first, uint64_t noise_seed, double sigma,
                                  const double* ttc, size_t m, double closing_speed,
                                  uint64_t* counts) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
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
}

int bmc_cuda_exceedance(bmc_ctx* ctx, const double* d, const uint8_t* hz, size_t n,
                        const double* headways, size_t m, uint64_t* counts) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
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
}

// ----------------------------------------------------------------------
// Mergeable building blocks: every output below is exactly additive (counts)
// or exactly mergeable (min/max, double-double sums) across shards, so a
// multi-GPU run combines them with one allreduce per quantity.

int bmc_cuda_partials(bmc_ctx* ctx, const double* d, const uint8_t* hz, size_t n,
                      bmc_partials* out) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
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
}

int bmc_cuda_moments(bmc_ctx* ctx, const double* d, size_t n, double mean, double* m2m3) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
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
}

int bmc_cuda_histogram(bmc_ctx* ctx, const double* d, size_t n, double origin, double bin_width,
                       uint64_t bins, uint64_t* counts) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
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
}

int bmc_cuda_select_pass(bmc_ctx* ctx, const double* d, const uint8_t* hz, size_t n,
                         int exclude_horizon, int shift, const uint64_t* prefixes, size_t m,
                         uint64_t* hist) {
    int rc = bmc::prepare(ctx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
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
}

}  // extern "C"
