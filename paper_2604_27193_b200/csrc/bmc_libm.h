// bmc_libm.h -- op-for-op port of the glibc 2.39 libm variants the reference
// sampler runs on x86-64 hosts with FMA+AVX2 (the ifunc targets __log_fma,
// __cos_fma, __sin_fma), for host (g++ -ffp-contract=off) and sm_100a
// (nvcc -fmad=false) alike, plus the reference's sampler and
// RolloutTerms::from built on it.
//
// Why a port: the reference draws every sample with glibc log/cos
// (/root/reference/proj/src/sampling.cpp:48-53) and stages sin(grade)
// (dynamics.cpp:64).  glibc 2.39 is not correctly rounded (~0.1% of results
// differ from the correctly rounded value), so CUDA's
// libdevice cannot reproduce the sampled bits.  The FMA variants are short
// table + polynomial routines whose every FP operation is an IEEE-754
// binary64 add/sub/mul/fma/sqrt; replaying them in the same order with
// single-rounding intrinsics gives the same bits on any IEEE machine.
//
// Source of truth: the disassembly of the installed libm
// (/lib/x86_64-linux-gnu/libm.so.6, sha256 pinned in bmc_glibc_tables.h),
// not glibc's C source: the contraction pattern (which a*b+c became one
// vfmadd) is GCC's choice when glibc was built with -mfma, and only the
// binary says which.  The comments give the libm address of each block.
// The tables and constants are read from the same binary by
// tools/extract_glibc_libm.py.  Algorithms (glibc sysdeps/ieee754/dbl-64):
//   e_log.c  (ARM optimized-routines log, 128-entry table, 2018)
//   s_sin.c  (IBM Accurate Mathematical Library, reworked 2018: do_sin,
//             do_cos, reduce_sincos, TAYLOR_SIN; tables sincostab.c)
//
// Coverage: log for positive normal finite x; sin/cos for |x| < 105414350
// (every argument the sampler can produce: 2*pi*u2 in (0, 2*pi), and the
// clamped grade |x| <= 1.5).  Outside that (huge-argument branred path,
// NaN/Inf, log of x <= 0 or subnormal) *bad is set and the caller must
// fail loudly -- the port never guesses.
//
// bmc_libm_selftest (bmc_libm_check.cpp) compares this header against the live
// glibc on the running host; the on-device sampler is only enabled when that
// check passes (a host whose CPU selects another ifunc variant, or another
// libm build, keeps the host sampler).
#pragma once

#include "bmc_glibc_tables.h"

#include <stdint.h>

#include <cmath>
#include <cstring>

#if defined(__CUDACC__)
#define BMC_HD __host__ __device__ __forceinline__
#define BMC_UNROLL _Pragma("unroll")
#else
#define BMC_UNROLL
#define BMC_HD inline
#endif

namespace bmc {
namespace glibc {

// ---------------------------------------------------------------- IEEE ops
BMC_HD double f64(uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double(static_cast<long long>(b));
#else
    double d;
    std::memcpy(&d, &b, 8);
    return d;
#endif
}
BMC_HD uint64_t u64(double d) {
#if defined(__CUDA_ARCH__)
    return static_cast<uint64_t>(__double_as_longlong(d));
#else
    uint64_t b;
    std::memcpy(&b, &d, 8);
    return b;
#endif
}
BMC_HD double add(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
BMC_HD double sub(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
BMC_HD double mul(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
BMC_HD double div(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __ddiv_rn(a, b);
#else
    return a / b;
#endif
}
BMC_HD double fma_(double a, double b, double c) {  // vfmadd*: a*b+c, one rounding
#if defined(__CUDA_ARCH__)
    return __fma_rn(a, b, c);
#else
    return std::fma(a, b, c);
#endif
}
BMC_HD double fnma(double a, double b, double c) {  // vfnmadd*: -(a*b)+c, one rounding
    return fma_(-a, b, c);
}
BMC_HD double sqrt_(double a) {  // sqrtsd: correctly rounded
#if defined(__CUDA_ARCH__)
    return __dsqrt_rn(a);
#else
    return std::sqrt(a);
#endif
}
BMC_HD double fabs_(double a) { return f64(u64(a) & 0x7fffffffffffffffull); }
BMC_HD double neg(double a) { return f64(u64(a) ^ 0x8000000000000000ull); }  // vxorpd signmask
BMC_HD double copysign_(double mag, double sgn) {  // vandnpd/vandpd/vorpd
    return f64((u64(mag) & 0x7fffffffffffffffull) | (u64(sgn) & 0x8000000000000000ull));
}

// Table views: log_tab = 128 x {invc, logc}; sct = 110 x {sn, ssn, cs, ccs}
// (raw bits; BMC_GLIBC_LOG_TAB_INIT / BMC_GLIBC_SINCOSTAB_INIT).
constexpr int kLogTabWords = 256;
constexpr int kSinCosTabWords = 440;

// --------------------------------------------------------------- __log_fma
// libm 0x79d50.  e_log.c with __FP_FAST_FMA: r = fma(z, invc, -1).
BMC_HD double log_fma(double x, const uint64_t* tab, bool* bad) {
    const uint64_t ix = u64(x);
    if (ix - 0x3fee000000000000ull <= 0x308ffffffffffull) {
        // 0x79e50: |x - 1| small (1 - 0x1p-4 <= x < 1 + 0x1.09p-4)
        if (ix == 0x3ff0000000000000ull) return 0.0;
        const double r = sub(x, 1.0);
        const double r2 = mul(r, r);
        const double r3 = mul(r, r2);
        double q1 = fma_(r, f64(BMC_GL_LOG_B2), f64(BMC_GL_LOG_B1));
        double q2 = fma_(r, f64(BMC_GL_LOG_B5), f64(BMC_GL_LOG_B4));
        double q3 = fma_(r, f64(BMC_GL_LOG_B8), f64(BMC_GL_LOG_B7));
        q1 = fma_(r2, f64(BMC_GL_LOG_B3), q1);
        q2 = fma_(r2, f64(BMC_GL_LOG_B6), q2);
        q3 = fma_(r2, f64(BMC_GL_LOG_B9), q3);
        q3 = fma_(r3, f64(BMC_GL_LOG_B10), q3);
        double p = fma_(q3, r3, q2);
        p = fma_(p, r3, q1);
        // w = r * 0x1p27; rhi = r + w - w  (contracted to two FMAs)
        const double t = fma_(r, f64(BMC_GL_TWO27), r);
        const double rhi = fnma(f64(BMC_GL_TWO27), r, t);
        const double b0 = f64(BMC_GL_LOG_B0);
        const double rhi2 = mul(rhi, rhi);
        const double rlo = sub(r, rhi);
        const double hi = fma_(rhi2, b0, r);                 // hi = r + rhi*rhi*B0
        double lo = fma_(rhi2, b0, sub(r, hi));              // lo = r - hi + w
        lo = fma_(mul(b0, rlo), add(r, rhi), lo);            // lo += B0*rlo*(rhi + r)
        const double y = fma_(p, r3, lo);                    // y = r3*p + lo
        return add(hi, y);
    }
    const uint32_t top = static_cast<uint32_t>(ix >> 48);
    if (top - 0x0010u > 0x7fdfu) {  // x < 0x1p-1022, x <= 0, inf or nan: not ported
        *bad = true;
        return 0.0;
    }
    const uint64_t tmp = ix - 0x3fe6000000000000ull;
    const int i = static_cast<int>((tmp >> 45) & 127u);
    const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
    const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
    const double invc = f64(tab[2 * i]);
    const double logc = f64(tab[2 * i + 1]);
    const double z = f64(iz);
    const double kd = static_cast<double>(k);  // vcvtsi2sd: exact
    const double w = fma_(kd, f64(BMC_GL_LN2HI), logc);
    const double r = fma_(z, invc, -1.0);
    const double a21 = fma_(r, f64(BMC_GL_LOG_A2), f64(BMC_GL_LOG_A1));
    const double hi = add(r, w);
    const double r2 = mul(r, r);
    double lo = add(sub(w, hi), r);
    lo = fma_(kd, f64(BMC_GL_LN2LO), lo);
    const double r3 = mul(r, r2);
    const double a43 = fma_(r, f64(BMC_GL_LOG_A4), f64(BMC_GL_LOG_A3));
    lo = fma_(r2, f64(BMC_GL_LOG_A0), lo);
    const double p = fma_(a43, r2, a21);
    const double y = fma_(r3, p, lo);
    return add(y, hi);
}

// ------------------------------------------------- s_sin.c building blocks
// Index into __sincostab: u = big + |x| puts round(|x| * 128) in the low
// mantissa bits; k = that << 2 (int arithmetic, as the binary does).
BMC_HD int sct_index(double ax, double* xs) {
    const double u = add(ax, f64(BMC_GL_BIG));
    *xs = sub(ax, sub(u, f64(BMC_GL_BIG)));
    return static_cast<int>(static_cast<uint32_t>(u64(u))) << 2;
}

// do_cos(x, dx) as inlined in __cos_fma (0x7bb36) / __sin_fma (0x7b5e0)
BMC_HD double do_cos(double x, double dx, const uint64_t* sct) {
    if (x < 0.0) dx = neg(dx);
    double xs;
    const int k = sct_index(fabs_(x), &xs);
    xs = add(xs, dx);
    const double xx = mul(xs, xs);
    const double ps = fma_(xx, f64(BMC_GL_SN5), f64(BMC_GL_SN3));
    const double s = fma_(mul(xs, xx), ps, xs);
    double pc = fma_(xx, f64(BMC_GL_CS6), f64(BMC_GL_CS4));
    pc = fma_(xx, pc, f64(BMC_GL_CS2));
    const double c = mul(xx, pc);
    const double sn = f64(sct[k]), ssn = f64(sct[k + 1]), cs = f64(sct[k + 2]),
                 ccs = f64(sct[k + 3]);
    double cor = fnma(s, ssn, ccs);  // (ccs - s*ssn
    cor = fnma(c, cs, cor);          //  - cs*c)
    cor = fnma(s, sn, cor);          //  - sn*s
    return add(cs, cor);
}

// TAYLOR_SIN(a*a, a, da) (0x7c0d0)
BMC_HD double taylor_sin(double a, double da) {
    const double xx = mul(a, a);
    double p = fma_(xx, f64(BMC_GL_S5), f64(BMC_GL_S4));
    p = fma_(xx, p, f64(BMC_GL_S3));
    p = fma_(xx, p, f64(BMC_GL_S2));
    p = fma_(xx, p, f64(BMC_GL_S1));
    double t = fma_(p, a, neg(mul(da, 0.5)));  // vfmsub: P*a - 0.5*da
    t = fma_(xx, t, da);
    return add(a, t);
}

// do_sin(x, dx) as inlined in __cos_fma (0x7bc7f) / __sin_fma (0x7b377)
BMC_HD double do_sin(double x, double dx, const uint64_t* sct) {
    if (fabs_(x) < f64(BMC_GL_SMALL_0126)) return taylor_sin(x, dx);
    if (x <= 0.0) dx = neg(dx);
    double xs;
    const int k = sct_index(fabs_(x), &xs);
    const double xx = mul(xs, xs);
    const double ps = fma_(xx, f64(BMC_GL_SN5), f64(BMC_GL_SN3));
    const double s = add(xs, fma_(mul(xs, xx), ps, dx));
    double pc = fma_(xx, f64(BMC_GL_CS6), f64(BMC_GL_CS4));
    pc = fma_(xx, pc, f64(BMC_GL_CS2));
    const double c = fma_(xs, dx, mul(xx, pc));
    const double sn = f64(sct[k]), ssn = f64(sct[k + 1]), cs = f64(sct[k + 2]),
                 ccs = f64(sct[k + 3]);
    double cor = fma_(s, ccs, ssn);  // (ssn + s*ccs
    cor = fnma(c, sn, cor);          //  - sn*c)
    cor = fma_(s, cs, cor);          //  + cs*s
    return copysign_(add(sn, cor), x);
}

// reduce_sincos (0x7bd53 / 0x7b476): x = n*pi/2 + (a + da)
BMC_HD int reduce_sincos(double x, double* a, double* da) {
    const double t = fma_(x, f64(BMC_GL_HPINV), f64(BMC_GL_TOINT));
    const double xn = sub(t, f64(BMC_GL_TOINT));
    const int n = static_cast<int>(static_cast<uint32_t>(u64(t)) & 3u);
    double y = fnma(xn, f64(BMC_GL_MP1), x);
    y = fnma(xn, f64(BMC_GL_MP2), y);
    const double t2 = fnma(xn, f64(BMC_GL_PP3), y);
    double db = fnma(xn, f64(BMC_GL_PP3), sub(y, t2));
    const double b = fnma(xn, f64(BMC_GL_PP4), t2);
    db = add(db, fnma(xn, f64(BMC_GL_PP4), sub(t2, b)));
    *a = b;
    *da = db;
    return n;
}

BMC_HD double do_sincos(double a, double da, int n, const uint64_t* sct) {
    const double r = (n & 1) ? do_cos(a, da, sct) : do_sin(a, da, sct);
    return (n & 2) ? neg(r) : r;
}

BMC_HD uint32_t high_word_abs(double x) {
    return static_cast<uint32_t>(u64(x) >> 32) & 0x7fffffffu;
}

// --------------------------------------------------------------- __cos_fma
// libm 0x7bad0 (round-to-nearest path; the device always runs RN)
BMC_HD double cos_fma(double x, const uint64_t* sct, bool* bad) {
    const uint32_t k = high_word_abs(x);
    if (k < 0x3e400000u) return 1.0;                          // |x| < 2^-27
    if (k < 0x3feb6000u) return do_cos(x, 0.0, sct);          // |x| < 0.855469
    if (k < 0x400368fdu) {                                    // |x| < 2.426265
        const double y = sub(f64(BMC_GL_HP0), fabs_(x));
        const double a = add(y, f64(BMC_GL_HP1));
        const double da = add(sub(y, a), f64(BMC_GL_HP1));
        return do_sin(a, da, sct);
    }
    if (k < 0x419921fbu) {                                    // |x| < 105414350
        double a, da;
        const int n = reduce_sincos(x, &a, &da);
        return do_sincos(a, da, n + 1, sct);
    }
    *bad = true;  // branred range, Inf, NaN: not ported
    return 0.0;
}

// --------------------------------------------------------------- __sin_fma
// libm 0x7b2d0
BMC_HD double sin_fma(double x, const uint64_t* sct, bool* bad) {
    const uint32_t k = high_word_abs(x);
    if (k < 0x3e500000u) return x;                            // |x| < 2^-26
    if (k < 0x3feb6000u) return do_sin(x, 0.0, sct);          // |x| < 0.855469
    if (k < 0x400368fdu) {                                    // |x| < 2.426265
        const double t = sub(f64(BMC_GL_HP0), fabs_(x));
        return copysign_(do_cos(t, f64(BMC_GL_HP1), sct), x);
    }
    if (k < 0x419921fbu) {
        double a, da;
        const int n = reduce_sincos(x, &a, &da);
        return do_sincos(a, da, n, sct);
    }
    *bad = true;
    return 0.0;
}

// ------------------------------------------------- the reference sampler
// stream_word (sampling.cpp:36-42): splitmix64 output at seed + (c+1)*gamma
BMC_HD uint64_t stream_word(uint64_t seed, uint64_t counter) {
    uint64_t z = seed + (counter + 1u) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// stream_uniform (sampling.cpp:44-46): ((w >> 12) + 0.5) * 2^-52, exact
BMC_HD double stream_uniform(uint64_t seed, uint64_t counter) {
    const uint64_t w = stream_word(seed, counter) >> 12;
#if defined(__CUDA_ARCH__)
    const double d = __ull2double_rn(w);
#else
    const double d = static_cast<double>(w);
#endif
    return mul(add(d, 0.5), 0x1.0p-52);
}

// standard_normal_at (sampling.cpp:48-53):
// sqrt(-2 log u1) * cos(two_pi * u2), u at counters 2i, 2i+1
BMC_HD double standard_normal_at(uint64_t seed, uint64_t index, const uint64_t* log_tab,
                                 const uint64_t* sct, bool* bad) {
    const double u1 = stream_uniform(seed, 2u * index);
    const double u2 = stream_uniform(seed, 2u * index + 1u);
    const double l = log_fma(u1, log_tab, bad);
    const double c = cos_fma(mul(6.283185307179586, u2), sct, bad);
    return mul(sqrt_(mul(-2.0, l)), c);
}

// One sample of draw_batch (sampling.cpp:73-97): streams 5i..5i+4 in the
// order (v0, mu, theta, m, c_d); floor clamps and the |grade| <= 1.5 clamp.
// Returns the number of clamps applied (0..5).  SpecT: any {mean, sd} pair.
template <class SpecT>
BMC_HD int draw_sample(uint64_t seed, const SpecT* spec, uint64_t index, const uint64_t* log_tab,
                       const uint64_t* sct, double out[5], bool* bad) {
    const uint64_t base = 5u * index;
    double p[5];
BMC_UNROLL
    for (int j = 0; j < 5; ++j) {
        p[j] = add(spec[j].mean, mul(spec[j].sd, standard_normal_at(seed, base + j, log_tab, sct, bad)));
    }
    int clamps = 0;
    if (p[0] < 0.1) { p[0] = 0.1; ++clamps; }
    if (p[1] < 0.05) { p[1] = 0.05; ++clamps; }
    if (p[3] < 500.0) { p[3] = 500.0; ++clamps; }
    if (p[4] < 0.0) { p[4] = 0.0; ++clamps; }
    if (p[2] > 1.5) {
        p[2] = 1.5;
        ++clamps;
    } else if (p[2] < -1.5) {
        p[2] = -1.5;
        ++clamps;
    }
BMC_UNROLL
    for (int j = 0; j < 5; ++j) out[j] = p[j];
    return clamps;
}

// RolloutTerms::from (dynamics.cpp:57-68) with friction_limit (:48-55).
// Returns false for a non-positive weight-transfer denominator (the
// reference throws std::domain_error).
struct TermsIn {
    double cg_height, wheelbase, gravity, air_density, frontal_area;
};
BMC_HD bool rollout_terms(const double s[5], const TermsIn& w, const uint64_t* sct, double* floor_,
                          double* drag, double* grade, bool* bad) {
    const double mu = s[1];
    const double denom = add(1.0, div(mul(mu, w.cg_height), w.wheelbase));
    if (!(denom > 0.0)) return false;
    *floor_ = div(neg(mul(mu, w.gravity)), denom);
    *drag = div(mul(mul(mul(0.5, w.air_density), s[4]), w.frontal_area), s[3]);
    *grade = mul(w.gravity, sin_fma(s[2], sct, bad));
    return true;
}

}  // namespace glibc
}  // namespace bmc
