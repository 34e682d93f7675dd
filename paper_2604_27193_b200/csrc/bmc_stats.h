// bmc_stats.h -- launchers of the on-device statistics kernels (bmc_stats.cu).
#pragma once

#include "bmc_internal.h"

#include <cuda_runtime.h>

namespace bmc {

constexpr int kMaxSelectTargets = 16;

struct BlockPartial {
    double min, max, sum_hi, sum_lo;
    unsigned long long horizon, count;
    int nan;
    int pad_;
};

struct MomentPartial {
    double m2_hi, m2_lo, m3_hi, m3_lo;
};

int stats_partials(uint64_t n);
cudaError_t launch_reduce(const double* d, const uint8_t* hz, uint64_t n, BlockPartial* out,
                          cudaStream_t s);
cudaError_t launch_moments(const double* d, uint64_t n, double mean, MomentPartial* out,
                           cudaStream_t s);
cudaError_t launch_hist(const double* d, uint64_t n, double lo, double bw, uint64_t bins,
                        unsigned long long* hist, cudaStream_t s);
cudaError_t launch_exceed(const double* d, const uint8_t* hz, uint64_t n, const double* sorted_h,
                          int m, unsigned long long* buckets, cudaStream_t s);
cudaError_t launch_select(const double* d, const uint8_t* hz, uint64_t n, int exclude_horizon,
                          int shift, const uint64_t* prefixes, int targets,
                          unsigned long long* hist, cudaStream_t s);

}  // namespace bmc
