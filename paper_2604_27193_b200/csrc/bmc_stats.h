// bmc_stats.h -- launchers of the on-device statistics kernels (bmc_stats.cu).
#pragma once

#include "bmc_internal.h"
#include "bmc_stats_core.h"
#include "bmc_stats_dev.cuh"

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


// fused statistics stage (bmc_fused_stats.cu; orchestration in bmc_stats_pipeline.h)
cudaError_t launch_pass1(const double* d, const uint8_t* hz, uint64_t n, const P1Args& a, int sms,
                         cudaStream_t s);
cudaError_t launch_normalize(const StageDev& g, size_t off, int accs, cudaStream_t s);
cudaError_t launch_finalize1(const StageDev& g, cudaStream_t s);
cudaError_t launch_pass2(const double* d, const uint8_t* hz, uint64_t n, const StageDev& g, int sms,
                         cudaStream_t s);
cudaError_t launch_targets(const StageDev& g, cudaStream_t s);
cudaError_t launch_compact(const double* d, const uint8_t* hz, uint64_t n, const StageDev& g,
                           int sms, cudaStream_t s);
cudaError_t launch_pack(const StageDev& g, const PackArgs& p, unsigned long long* dst, int sms,
                        cudaStream_t s);
cudaError_t launch_select_targets(const StageDev& g, const SelectSegments& seg,
                                  const unsigned long long* keys, cudaStream_t s);

}  // namespace bmc
