// bmc_stats_dev.cuh -- pass 1 of the fused statistics stage as per-CTA
// shared-memory partials: used by the rollout epilogue (bmc_kernels.cu) and
// the standalone pass over existing outputs (bmc_fused_stats.cu).
//
// Per result (d, hit_horizon): count, horizon count, order keys of min and
// max, the exact sum of d (superaccumulator limbs, bmc_stats_core.h) and the
// exceedance bucket p = #{H_j < d} (m for a horizon hit) over the sorted
// headways H.  Shared-memory atomics per result; one flush of the non-zero
// words per CTA into the stage's P1 words (u64 atomics), so the global
// traffic is O(CTAs x words), not O(results).
#pragma once

#include "bmc_stats_core.h"

#include <cuda_runtime.h>

namespace bmc {

struct P1Smem {
    unsigned long long acc[sc::kAccWords];
    unsigned long long count, horizon, min_key, inv_max;
};

// The P1 words a launch accumulates into (nullptr sum: disabled).
struct P1Args {
    unsigned long long* sum;   // SUM section (sc::p1_sum_words(m) words)
    unsigned long long* minw;  // MIN section (2 words)
    const double* H;           // sorted headways, m entries (device)
    int m;                     // 0: exceedance not accumulated here
};

#if defined(__CUDACC__)
__host__ __device__
#endif
constexpr size_t p1_smem_bytes(int m) {
    return ((sizeof(P1Smem) + 8 * static_cast<size_t>(m) + 4 * (static_cast<size_t>(m) + 1)) + 15) &
           ~static_cast<size_t>(15);
}

#if defined(__CUDACC__)
struct P1View {
    P1Smem* s;
    double* H;
    unsigned* b;
};

__device__ __forceinline__ P1View p1_view(unsigned char* base, int m) {
    P1View v;
    v.s = reinterpret_cast<P1Smem*>(base);
    v.H = reinterpret_cast<double*>(v.s + 1);
    v.b = reinterpret_cast<unsigned*>(v.H + m);
    return v;
}

// All threads of the CTA; caller synchronises afterwards.
__device__ __forceinline__ void p1_init(const P1View& v, const P1Args& a) {
    for (int i = threadIdx.x; i < sc::kAccWords; i += blockDim.x) v.s->acc[i] = 0ull;
    if (threadIdx.x == 0) {
        v.s->count = 0ull;
        v.s->horizon = 0ull;
        v.s->min_key = ~0ull;
        v.s->inv_max = ~0ull;
    }
    for (int j = threadIdx.x; j < a.m; j += blockDim.x) v.H[j] = a.H[j];
    for (int j = threadIdx.x; j <= a.m; j += blockDim.x) v.b[j] = 0u;
}

__device__ __forceinline__ void p1_add(const P1View& v, int m, double d, bool horizon) {
    atomicAdd(&v.s->count, 1ull);
    if (horizon) atomicAdd(&v.s->horizon, 1ull);
    const int sp = sc::special_of(d);
    if (sp != sc::kFinite) {
        atomicAdd(&v.s->acc[2 * sc::kLimbs + sp - 1], 1ull);
    } else {
        int L;
        uint32_t w0, w1, w2;
        sc::split(d, &L, &w0, &w1, &w2);
        unsigned long long* a = v.s->acc + ((sc::bits_of(d) >> 63) ? sc::kLimbs : 0) + L;
        if (w0) atomicAdd(a, static_cast<unsigned long long>(w0));
        if (w1) atomicAdd(a + 1, static_cast<unsigned long long>(w1));
        if (w2) atomicAdd(a + 2, static_cast<unsigned long long>(w2));
    }
    if (sp != sc::kNaN) {
        const unsigned long long k = sc::order_key(d);
        atomicMin(&v.s->min_key, k);
        atomicMin(&v.s->inv_max, ~k);
    }
    if (m) atomicAdd(&v.b[sc::exceed_bucket(v.H, m, d, horizon)], 1u);
}

// All threads, after a __syncthreads that follows the last p1_add.
__device__ __forceinline__ void p1_flush(const P1View& v, const P1Args& a) {
    for (int i = threadIdx.x; i < sc::kAccWords; i += blockDim.x) {
        const unsigned long long w = v.s->acc[i];
        if (w) atomicAdd(&a.sum[sc::kP1Acc + i], w);
    }
    if (threadIdx.x == 0) {
        if (v.s->count) atomicAdd(&a.sum[sc::kP1Count], v.s->count);
        if (v.s->horizon) atomicAdd(&a.sum[sc::kP1Horizon], v.s->horizon);
        if (v.s->min_key != ~0ull) atomicMin(&a.minw[0], v.s->min_key);
        if (v.s->inv_max != ~0ull) atomicMin(&a.minw[1], v.s->inv_max);
    }
    for (int j = threadIdx.x; j <= a.m; j += blockDim.x) {
        const unsigned c = v.b[j];
        if (c) atomicAdd(&a.sum[sc::kP1Exceed + j], static_cast<unsigned long long>(c));
    }
}

#endif  // __CUDACC__

}  // namespace bmc
