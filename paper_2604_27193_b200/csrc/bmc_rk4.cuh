// bmc_rk4.cuh -- the FP64 arithmetic of one RK4 step, shared by every
// rollout kernel (bmc_kernels.cu) and the step probe (tools/rk4_step_probe.cu).
//
// Every operation is spelled with an explicit _rn intrinsic in the
// reference's association order (integrator.hpp:39-68, dynamics.hpp:115-132;
// paths under /root/reference/proj), so the results are bit-identical to the
// reference's -ffp-contract=off build regardless of compiler flags.
#pragma once

#include <cuda_runtime.h>

namespace bmc {

__device__ __forceinline__ double clamp_brake(double a, double floor_) {
    // dynamics.hpp:82-84 (ternary semantics, not fmax)
    return a > floor_ ? a : floor_;
}

// longitudinal_accel (dynamics.hpp:115-118): (braking - D*(v*v)) - G
__device__ __forceinline__ double accel(double braking, double v, double D, double G) {
    return __dsub_rn(__dsub_rn(braking, __dmul_rn(D, __dmul_rn(v, v))), G);
}

// The (position, speed) lanes of rk4_step (integrator.hpp:39-68) for given
// clamped stage brake values b1..b4.  k_i.d_position = stage speed, so the
// position stages (dead code in the reference) are not formed.  32 FP64 ops:
// k1 + 2.0*k2 is fma(2.0, k2, k1) -- 2.0*k2 is exact in binary64, so the
// FMA's single rounding equals the reference's rounding of the add.
__device__ __forceinline__ void rk4_xv(double& x, double& v, double b1, double b2, double b3,
                                       double b4, double D, double G, double dt, double half,
                                       double sixth) {
    const double k1 = accel(b1, v, D, G);
    const double s2 = __dadd_rn(v, __dmul_rn(half, k1));
    const double k2 = accel(b2, s2, D, G);
    const double s3 = __dadd_rn(v, __dmul_rn(half, k2));
    const double k3 = accel(b3, s3, D, G);
    const double s4 = __dadd_rn(v, __dmul_rn(dt, k3));
    const double k4 = accel(b4, s4, D, G);
    // ((k1 + 2k2) + 2k3) + k4 with exact doubling folded into FMAs
    const double cv = __dadd_rn(__fma_rn(2.0, k3, __fma_rn(2.0, k2, k1)), k4);
    const double cx = __dadd_rn(__fma_rn(2.0, s3, __fma_rn(2.0, s2, v)), s4);
    x = __dadd_rn(x, __dmul_rn(sixth, cx));
    v = __dadd_rn(v, __dmul_rn(sixth, cv));
}

// v <= 0.0 (integrator.cpp:22) on the integer pipe: a binary64 pattern read
// as int64 is <= 0 exactly for +0, -0 and every negative value, so the test
// agrees with the FP compare for every non-NaN v and leaves the FP64 pipe to
// the RK4 arithmetic.  (Only a sign-bit-set NaN would differ; finite inputs
// cannot produce one.)
__device__ __forceinline__ bool not_positive(double v) { return __double_as_longlong(v) <= 0ll; }

// Coarse form on the high word only: true for every v not_positive accepts,
// plus positive subnormals below 2^-1042 (high word 0).  Loops that batch
// their termination test on it confirm with not_positive before acting.
__device__ __forceinline__ int hi_word(double v) { return __double2hiint(v); }

}  // namespace bmc
