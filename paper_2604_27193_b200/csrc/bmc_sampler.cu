// bmc_sampler.cu -- on-device sampler: draw_batch (sampling.cpp:67-100)
// fused with RolloutTerms::from (dynamics.cpp:57-68), bit-identical to the
// host producers (bmc_host.cpp) through the glibc port in bmc_libm.h.
//
// One thread per sample index, grid-stride; the 5.5 KB of glibc tables are
// staged in shared memory per CTA (divergent table indices would serialise
// on the constant cache).  Cost per sample: 10 splitmix64 words, 5 log,
// 5 sqrt, 5 cos, 1 sin, 2 divisions -- ~0.3% of one rollout's 32 x 5161
// FP64 ops, so the sampler never shows in the step time, and it removes the
// host feed (242 ns/sample/core) from the model-driven
// path.  Outputs are written SoA (coalesced 8-B stores per field).
#include "bmc_kernels.h"
#include "bmc_libm.h"

namespace bmc {
namespace {

__device__ const uint64_t g_log_tab[glibc::kLogTabWords] = {BMC_GLIBC_LOG_TAB_INIT};
__device__ const uint64_t g_sincos_tab[glibc::kSinCosTabWords] = {BMC_GLIBC_SINCOSTAB_INIT};

constexpr int kDrawThreads = 256;

__global__ void __launch_bounds__(kDrawThreads) draw_terms_kernel(DrawArgs a) {
    __shared__ uint64_t s_log[glibc::kLogTabWords];
    __shared__ uint64_t s_sct[glibc::kSinCosTabWords];
    for (int i = threadIdx.x; i < glibc::kLogTabWords; i += blockDim.x) s_log[i] = g_log_tab[i];
    for (int i = threadIdx.x; i < glibc::kSinCosTabWords; i += blockDim.x) s_sct[i] = g_sincos_tab[i];
    __syncthreads();

    uint64_t seed = a.seed, first = a.first;
    bmc_normal spec[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) spec[j] = a.spec[j];
    if (a.dyn) {
        seed = a.dyn->seed;
        first = a.dyn->first;
#pragma unroll
        for (int j = 0; j < 5; ++j) spec[j] = a.dyn->spec[j];
    }
    const glibc::TermsIn tw{a.cg_height, a.wheelbase, a.gravity, a.air_density, a.frontal_area};
    unsigned long long clamps = 0;
    unsigned int flags = 0;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n;
         i += stride) {
        bool bad = false;
        double s[5];
        clamps += glibc::draw_sample(seed, spec, first + i, s_log, s_sct, s, &bad);
        if (a.samples) {
            double* o = a.samples + 5 * i;  // bmc_sample: v0, mu, theta, m, c_d
            o[0] = s[0];
            o[1] = s[1];
            o[2] = s[2];
            o[3] = s[3];
            o[4] = s[4];
        }
        if (a.v0) {
            double fl = 0.0, dr = 0.0, gr = 0.0;
            if (!glibc::rollout_terms(s, tw, s_sct, &fl, &dr, &gr, &bad)) flags |= kDrawDomain;
            a.v0[i] = s[0];
            a.brake_floor[i] = fl;
            a.drag[i] = dr;
            a.grade[i] = gr;
        }
        if (bad) flags |= kDrawUnported;
    }
    // warp-aggregated counters: one atomic per warp
    for (int o = 16; o > 0; o >>= 1) {
        clamps += __shfl_xor_sync(0xffffffffu, clamps, o);
        flags |= __shfl_xor_sync(0xffffffffu, flags, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (clamps) atomicAdd(a.clamps, clamps);
        if (flags) atomicOr(a.flags, flags);
    }
}

__global__ void __launch_bounds__(kDrawThreads) noise_exceed_kernel(NoiseExceedArgs a) {
    __shared__ uint64_t s_log[glibc::kLogTabWords];
    __shared__ uint64_t s_sct[glibc::kSinCosTabWords];
    __shared__ double s_t[kNoiseMaxThresholds];
    __shared__ unsigned int s_b[kNoiseMaxThresholds + 1];
    for (int i = threadIdx.x; i < glibc::kLogTabWords; i += blockDim.x) s_log[i] = g_log_tab[i];
    for (int i = threadIdx.x; i < glibc::kSinCosTabWords; i += blockDim.x) s_sct[i] = g_sincos_tab[i];
    for (int j = threadIdx.x; j < a.m; j += blockDim.x) s_t[j] = a.ttc[j];
    for (int j = threadIdx.x; j <= a.m; j += blockDim.x) s_b[j] = 0u;
    __syncthreads();
    unsigned int flags = 0;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n;
         i += stride) {
        int p;
        if (a.hz && a.hz[i]) {
            p = a.m;
        } else {
            bool bad = false;
            const double z = glibc::standard_normal_at(a.seed, a.first + i, s_log, s_sct, &bad);
            if (bad) flags |= kDrawUnported;
            const double eps = __dmul_rn(a.sigma, z);
            const double v = a.d[i];
            int lo = 0, hi = a.m;  // first j with !(H_j < v); H_j = (T_j + eps) * closing
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (__dmul_rn(__dadd_rn(s_t[mid], eps), a.closing) < v) {
                    lo = mid + 1;
                } else {
                    hi = mid;
                }
            }
            p = lo;
        }
        atomicAdd(&s_b[p], 1u);
    }
    __syncthreads();
    for (int j = threadIdx.x; j <= a.m; j += blockDim.x) {
        if (s_b[j]) atomicAdd(&a.buckets[j], static_cast<unsigned long long>(s_b[j]));
    }
    for (int o = 16; o > 0; o >>= 1) flags |= __shfl_xor_sync(0xffffffffu, flags, o);
    if ((threadIdx.x & 31) == 0 && flags) atomicOr(a.flags, flags);
}

}  // namespace

cudaError_t launch_noise_exceed(const NoiseExceedArgs& a, int sms, cudaStream_t s) {
    if (a.n == 0) return cudaSuccess;
    if (a.m < 1 || a.m > kNoiseMaxThresholds) return cudaErrorInvalidValue;
    const uint64_t blocks_needed = (a.n + kDrawThreads - 1) / kDrawThreads;
    const uint64_t cap = static_cast<uint64_t>(sms > 0 ? sms : 148) * 4;
    const unsigned grid = static_cast<unsigned>(blocks_needed < cap ? blocks_needed : cap);
    noise_exceed_kernel<<<grid, kDrawThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_draw_terms(const DrawArgs& a, int sms, cudaStream_t s) {
    if (a.n == 0) return cudaSuccess;
    const uint64_t blocks_needed = (a.n + kDrawThreads - 1) / kDrawThreads;
    // 8 CTAs per SM resident (256 threads, 5.5 KB smem); grid-stride beyond
    const uint64_t cap = static_cast<uint64_t>(sms > 0 ? sms : 148) * 8;
    const unsigned grid = static_cast<unsigned>(blocks_needed < cap ? blocks_needed : cap);
    draw_terms_kernel<<<grid, kDrawThreads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace bmc
