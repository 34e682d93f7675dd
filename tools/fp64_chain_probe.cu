// fp64_chain_probe.cu -- characterises the B200 FP64 pipe for the rollout
// kernel's roofline discussion:
//   1. dependent-chain latency of DADD / DMUL / DFMA (one warp, one chain);
//   2. issue-limited throughput with W warps per SM x C independent chains
//      per thread of an unfused DMUL+DADD pair (the probe of
//      bmc_cuda_fp64_peak is W=64, C=8).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false \
//          tools/fp64_chain_probe.cu -o build/fp64_chain_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void latency_kernel(double* out, int iters, double a, double b, long long* cycles) {
    double x = 1.0 + threadIdx.x * 1e-9;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (OP == 0) x = __dadd_rn(x, b);
            if (OP == 1) x = __dmul_rn(x, a);
            if (OP == 2) x = __fma_rn(x, a, b);
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) *cycles = t1 - t0;
    if (x == 12345.678) out[0] = x;
}

template <int C>
__global__ void chains_kernel(double* out, int iters, double a, double b) {
    double x[C];
#pragma unroll
    for (int k = 0; k < C; ++k) x[k] = 1.0 + 1e-9 * (threadIdx.x + 37 * k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < C; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], a), b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < C; ++k) s = __dadd_rn(s, x[k]);
    if (s == 12345.678) out[0] = s;
}

template <int C>
double run_chains(int warps_per_sm, int sms, double* out) {
    const int threads = warps_per_sm * 32 > 1024 ? 1024 : warps_per_sm * 32;
    const int blocks_per_sm = warps_per_sm * 32 / threads;
    const int blocks = sms * blocks_per_sm;
    const int iters = 4096 * 8 / C;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    chains_kernel<C><<<blocks, threads>>>(out, 16, 0.99999999, 1e-8);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        chains_kernel<C><<<blocks, threads>>>(out, iters, 0.99999999, 1e-8);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double ops = static_cast<double>(blocks) * threads * iters * C * 2.0;
    return ops / (best * 1e-3);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64);
    cudaMalloc(&cyc, 8);
    const char* names[3] = {"DADD", "DMUL", "DFMA"};
    for (int op = 0; op < 3; ++op) {
        long long c = 0;
        const int iters = 4096;
        for (int r = 0; r < 2; ++r) {
            if (op == 0) latency_kernel<0><<<1, 32>>>(out, iters, 0.99999999, 1e-8, cyc);
            if (op == 1) latency_kernel<1><<<1, 32>>>(out, iters, 0.99999999, 1e-8, cyc);
            if (op == 2) latency_kernel<2><<<1, 32>>>(out, iters, 0.99999999, 1e-8, cyc);
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        }
        printf("latency %s: %.2f cycles (dependent chain, 1 warp)\n", names[op],
               static_cast<double>(c) / (iters * 16.0));
    }
    printf("throughput of unfused DMUL+DADD chains (T op/s):\n");
    printf("%8s %10s %10s %10s %10s\n", "warps/SM", "C=1", "C=2", "C=4", "C=8");
    const int ws[] = {4, 8, 12, 16, 20, 24, 32, 48, 64};
    for (int w : ws) {
        printf("%8d %10.3f %10.3f %10.3f %10.3f\n", w, run_chains<1>(w, sms, out) / 1e12,
               run_chains<2>(w, sms, out) / 1e12, run_chains<4>(w, sms, out) / 1e12,
               run_chains<8>(w, sms, out) / 1e12);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("CUDA error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
