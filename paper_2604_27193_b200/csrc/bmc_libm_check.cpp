// bmc_libm_check.cpp -- proves, on the running host, that the glibc port in
// bmc_libm.h reproduces the host's own libm bit for bit (the gate of the
// on-device sampler).
//
// Compiled by g++ with -ffp-contract=off: the port's host instantiation uses
// the same add/sub/mul/fma/sqrt sequence the sm_100a instantiation uses, so
// host-port == glibc here and device-port == host-port (tests/test_gpu_sampler.py)
// together give device == reference.  std::log / std::cos / std::sin below
// resolve to the same glibc entry points the reference calls
// (sampling.cpp:52, dynamics.cpp:64).
#include "bmc_internal.h"
#include "bmc_libm.h"

#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

namespace bmc {

namespace {

const uint64_t kLogTab[glibc::kLogTabWords] = {BMC_GLIBC_LOG_TAB_INIT};
const uint64_t kSinCosTab[glibc::kSinCosTabWords] = {BMC_GLIBC_SINCOSTAB_INIT};

inline bool same(double a, double b) { return glibc::u64(a) == glibc::u64(b); }

// The reference's deviate, verbatim semantics (sampling.cpp:48-53)
inline double ref_normal(uint64_t seed, uint64_t index) {
    const double u1 = glibc::stream_uniform(seed, 2u * index);
    const double u2 = glibc::stream_uniform(seed, 2u * index + 1u);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

// Boundary arguments of every branch of the ported routines, +-4 ulp.
void boundary_values(std::vector<double>* out) {
    const double edges[] = {0x1p-27,    0x1p-26,        0.85546875, 0.126,   2.426265,
                            2.4262652,  1.5707963267948966, 0.9375, 1.0,     1.064697265625,
                            0.6875,     1.375,          0.7853981633974483,  3.141592653589793,
                            4.71238898038469, 6.283185307179586, 1.5,    1e-300,  0.5};
    for (double e : edges) {
        uint64_t b = glibc::u64(e);
        for (int d = -4; d <= 4; ++d) out->push_back(glibc::f64(b + static_cast<uint64_t>(d)));
    }
}

}  // namespace

const uint64_t* host_log_tab() { return kLogTab; }
const uint64_t* host_sincos_tab() { return kSinCosTab; }

// mism[0] log over the sampler's u1, [1] log near 1, [2] cos(2*pi*u),
// [3] sin over |x| <= 1.5 (+ tiny), [4] sin/cos with range reduction,
// [5] standard_normal_at, [6] boundary arguments (all functions)
void libm_port_check(uint64_t n, uint64_t seed, unsigned threads, uint64_t mism[7]) {
    std::atomic<uint64_t> m[7];
    for (auto& a : m) a = 0;
    host_pool().parallel_for(
        n,
        [&](std::size_t b, std::size_t e) {
            uint64_t c[7] = {0, 0, 0, 0, 0, 0, 0};
            bool bad = false;
            for (std::size_t i = b; i < e; ++i) {
                const double u = glibc::stream_uniform(seed, 2 * i);
                const double v = glibc::stream_uniform(seed, 2 * i + 1);
                c[0] += !same(glibc::log_fma(u, kLogTab, &bad), std::log(u));
                const double x1 = 0.9375 + 0.13 * v;  // covers the |x - 1| < 2^-4 branch
                c[1] += !same(glibc::log_fma(x1, kLogTab, &bad), std::log(x1));
                const double xc = 6.283185307179586 * v;
                c[2] += !same(glibc::cos_fma(xc, kSinCosTab, &bad), std::cos(xc));
                const double xs = (i & 1) ? 3.0 * u - 1.5 : (u - 0.5) * 0x1p-18;
                c[3] += !same(glibc::sin_fma(xs, kSinCosTab, &bad), std::sin(xs));
                const double xr = 200.0 * v - 100.0;
                c[4] += !same(glibc::sin_fma(xr, kSinCosTab, &bad), std::sin(xr)) ||
                        !same(glibc::cos_fma(xr, kSinCosTab, &bad), std::cos(xr));
                c[5] += !same(glibc::standard_normal_at(seed, i, kLogTab, kSinCosTab, &bad),
                              ref_normal(seed, i));
            }
            if (bad) c[6] += 1;  // an argument fell outside the ported range
            for (int k = 0; k < 7; ++k) m[k] += c[k];
        },
        threads);
    std::vector<double> edge;
    boundary_values(&edge);
    bool bad = false;
    for (double x : edge) {
        for (double s : {x, -x}) {
            if (s > 0.0 && !same(glibc::log_fma(s, kLogTab, &bad), std::log(s))) ++m[6];
            if (!same(glibc::sin_fma(s, kSinCosTab, &bad), std::sin(s))) ++m[6];
            if (!same(glibc::cos_fma(s, kSinCosTab, &bad), std::cos(s))) ++m[6];
        }
    }
    if (bad) ++m[6];
    for (int k = 0; k < 7; ++k) mism[k] = m[k];
}

// Process-wide verdict of a quick check (2^15 draws + boundaries), cached.
bool device_sampler_supported(std::string* why) {
    static std::once_flag once;
    static bool ok = false;
    static std::string reason;
    std::call_once(once, [] {
        uint64_t mm[7];
        libm_port_check(uint64_t{1} << 15, 0x5eedULL, 0, mm);
        ok = true;
        reason.clear();
        const char* names[7] = {"log", "log~1", "cos", "sin", "sincos-reduce", "normal", "edges"};
        for (int k = 0; k < 7; ++k) {
            if (mm[k]) {
                ok = false;
                reason += std::string(reason.empty() ? "" : ", ") + names[k] + " mismatches " +
                          std::to_string(mm[k]);
            }
        }
        if (!ok) {
            reason = "host libm is not the glibc 2.39 FMA variant the device sampler replays (" +
                     reason + "; port built from libm sha256 " BMC_GLIBC_LIBM_SHA256 ")";
        }
    });
    if (why) *why = reason;
    return ok;
}

}  // namespace bmc

extern "C" int bmc_libm_selftest(uint64_t n, uint64_t seed, int threads, uint64_t* mismatches) {
    try {
        if (mismatches == nullptr) {
            bmc::set_error("bmc_libm_selftest: null argument");
            return BMC_E_CONFIG;
        }
        bmc::libm_port_check(n, seed, bmc::resolve_threads(threads), mismatches);
        for (int k = 0; k < 7; ++k) {
            if (mismatches[k]) {
                bmc::set_error("glibc port differs from the host libm");
                return BMC_E_CONFIG;
            }
        }
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception();
    }
}

extern "C" int bmc_device_sampler_available(int* available) {
    try {
        if (available == nullptr) {
            bmc::set_error("bmc_device_sampler_available: null argument");
            return BMC_E_CONFIG;
        }
        std::string why;
        *available = bmc::device_sampler_supported(&why) ? 1 : 0;
        if (!*available) bmc::set_error(why);
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception();
    }
}
