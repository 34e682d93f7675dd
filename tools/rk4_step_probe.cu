// rk4_step_probe.cu -- where does the rollout kernel lose FP64 pipe time?
// Runs the exact 32-op RK4 (x, v) step of bmc_kernels.cu (rk4_xv) on
// synthetic lanes with no early exit, adding one ingredient of the real
// loop at a time, at several warps/SM and chains/thread:
//   pure   : the 32 FP64 ops only (brake values are loop constants)
//   test   : + the integer v <= 0 test and its (never taken) branch
//   table  : + the per-step 32-B actuator-table row from shared memory
//            (two LDS.128, prefetched one step ahead, warp-uniform index)
//   hi     : per-step branch on the high word only (one ISETP + BRA)
//   minK   : per-step IMNMX of the high word into a running minimum, one
//            branch per K steps (the exact step is recovered by replay)
// Rates are executed FP64 ops/s (32 per step).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false \
//        tools/rk4_step_probe.cu -o build/rk4_step_probe
#include <cstdio>
#include <cuda_runtime.h>

struct StageA {
    double a0, a1, a2, a3;
};

__device__ __forceinline__ double accel(double b, double v, double D, double G) {
    return __dsub_rn(__dsub_rn(b, __dmul_rn(D, __dmul_rn(v, v))), G);
}

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
    const double cv = __dadd_rn(__fma_rn(2.0, k3, __fma_rn(2.0, k2, k1)), k4);
    const double cx = __dadd_rn(__fma_rn(2.0, s3, __fma_rn(2.0, s2, v)), s4);
    x = __dadd_rn(x, __dmul_rn(sixth, cx));
    v = __dadd_rn(v, __dmul_rn(sixth, cv));
}

__device__ __forceinline__ bool not_positive(double v) { return __double_as_longlong(v) <= 0ll; }

constexpr int kRows = 4096;
constexpr StageA kB{-5.0, -5.1, -5.2, -5.3};
constexpr int kConstRows = 2048;  // 64 KB of __constant__
constexpr int kParamRows = 960;   // 30 KB of kernel parameters
struct ParamRows {
    StageA r[kParamRows];
};
__constant__ StageA c_tab[kConstRows];

// MODE 0 pure, 1 + test, 2 + test + table, 3 table + hi-word test,
// 4 table without any test, 10 + K: table + running-minimum test per K
// steps, 20 + K: the same with constant brake values.  C chains per thread.
template <int MODE, int C, bool LANEB = false>
__global__ void probe(double* out, int steps, double dt, double half, double sixth,
                      const StageA* gtab, StageA bb4) {
    const double bb[4] = {bb4.a0, bb4.a1, bb4.a2, bb4.a3};
    extern __shared__ StageA tab[];
    if (MODE >= 2 && MODE < 20 && MODE != 5 && MODE != 7) {
        for (int i = threadIdx.x; i < kRows; i += blockDim.x) tab[i] = gtab[i];
        __syncthreads();
    }
    double x[C], v[C], D[C], G[C];
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        x[c] = 0.0;
        v[c] = 1e30 + t + c;  // never reaches 0 within the probe
        D[c] = 1e-70 * (1 + (t & 7));  // D*v*v ~ 1e-10: no subnormals
        G[c] = -1.0 - 1e-3 * (c + (t & 3));  // runtime per-lane, like the kernel's G
    }
    // brake values: kernel arguments (warp-uniform) or, with LANEB, per-lane
    // registers (the kernel's clamped constants)
    const double lb = LANEB ? 1e-9 * (t & 1) : 0.0;
    const double b1 = bb[0] + lb, b2 = bb[1] + lb, b3 = bb[2] + lb, b4 = bb[3] + lb;
    StageA nx = tab[0];
    int n = 0;
    if (MODE >= 10 && MODE < 30) {
        // running minimum of hi(v) over a block of K steps, one branch per block
        // (MODE >= 20: constant brake values instead of table rows)
        constexpr int K = MODE % 10;
        constexpr bool kTab = MODE < 20;
        for (; n + K <= steps; n += K) {
            int m = 0x7fffffff;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                StageA s{b1, b2, b3, b4};
                if (kTab) {
                    s = nx;
                    nx = tab[(n + k + 1) & (kRows - 1)];
                }
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    rk4_xv(x[c], v[c], s.a0, s.a1, s.a2, s.a3, D[c], G[c], dt, half, sixth);
                    m = min(m, __double2hiint(v[c]));
                }
            }
            if (m <= 0) break;
        }
    }
    if (MODE == 5 || MODE == 7) {
        // table rows from __constant__ memory with a warp-uniform index
        for (; n < steps; ++n) {
            const StageA s = c_tab[n & (kConstRows - 1)];
#pragma unroll
            for (int c = 0; c < C; ++c) rk4_xv(x[c], v[c], s.a0, s.a1, s.a2, s.a3, D[c], G[c], dt, half, sixth);
            if (MODE == 7) {
                bool stop = false;
#pragma unroll
                for (int c = 0; c < C; ++c) stop |= not_positive(v[c]);
                if (stop) break;
            }
        }
    }
    if (MODE >= 30 && MODE < 40) {
        // __constant__ rows, warp-uniform block loop: running min of hi(v)
        // over K steps, one vote + uniform branch per block
        constexpr int K = MODE - 30;
        for (; n + K <= steps; n += K) {
            int m = 0x7fffffff;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const StageA s = c_tab[(n + k) & (kConstRows - 1)];
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    rk4_xv(x[c], v[c], s.a0, s.a1, s.a2, s.a3, D[c], G[c], dt, half, sixth);
                    m = min(m, __double2hiint(v[c]));
                }
            }
            if (__any_sync(0xffffffffu, m <= 0)) break;
        }
    }
    if (MODE == 6) {
        // half the row from shared memory (one LDS.128), half constant
        double2 h = reinterpret_cast<const double2*>(tab)[0];
        for (; n < steps; ++n) {
            const double2 s = h;
            h = reinterpret_cast<const double2*>(tab)[2 * ((n + 1) & (kRows - 1))];
#pragma unroll
            for (int c = 0; c < C; ++c) rk4_xv(x[c], v[c], s.x, s.y, b3, b4, D[c], G[c], dt, half, sixth);
        }
    }
    for (; MODE < 5 && n < steps; ++n) {  // NOLINT
        double a0 = b1, a1 = b2, a2 = b3, a3 = b4;
        if (MODE == 2 || MODE == 3 || MODE == 4) {
            const StageA s = nx;
            nx = tab[(n + 1) & (kRows - 1)];
            a0 = s.a0;
            a1 = s.a1;
            a2 = s.a2;
            a3 = s.a3;
        }
#pragma unroll
        for (int c = 0; c < C; ++c) rk4_xv(x[c], v[c], a0, a1, a2, a3, D[c], G[c], dt, half, sixth);
        if (MODE == 3) {
            bool stop = false;
#pragma unroll
            for (int c = 0; c < C; ++c) stop |= __double2hiint(v[c]) <= 0;
            if (stop) break;
        }
        if (MODE == 1 || MODE == 2) {
            bool stop = false;
#pragma unroll
            for (int c = 0; c < C; ++c) stop |= not_positive(v[c]);
            if (stop) break;
        }
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < C; ++c) s = __dadd_rn(s, __dadd_rn(x[c], v[c]));
    if (s == 12345.678 || n == -7) out[0] = s;
}

// Table rows passed by value as a __grid_constant__ kernel parameter (one
// launch per 960-row phase), warp-uniform block loop with vote (K steps).
template <int K>
__global__ void probe_param(double* out, int steps, double dt, double half, double sixth,
                            const __grid_constant__ ParamRows rows) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    double x = 0.0, v = 1e30 + t, D = 1e-70 * (1 + (t & 7)), G = -1.0 - 1e-3 * (t & 3);
    int n = 0;
    for (; n + K <= steps; n += K) {
        int m = 0x7fffffff;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const StageA s = rows.r[(n + k) % kParamRows];
            rk4_xv(x, v, s.a0, s.a1, s.a2, s.a3, D, G, dt, half, sixth);
            m = min(m, __double2hiint(v));
        }
        if (__any_sync(0xffffffffu, m <= 0)) break;
    }
    if (__dadd_rn(x, v) == 12345.678 || n == -7) out[0] = x;
}

template <int K>
double run_param(int warps_per_sm, int sms, double* out) {
    static ParamRows h;
    for (int i = 0; i < kParamRows; ++i) h.r[i] = StageA{-5.0 - 1e-4 * i, -5.1, -5.2, -5.3};
    const int threads = warps_per_sm * 32 > 1024 ? 1024 : warps_per_sm * 32;
    const int blocks = sms * (warps_per_sm * 32 / threads);
    const int steps = 960 * 20;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe_param<K><<<blocks, threads>>>(out, 16, 1e-3, 5e-4, 1e-3 / 6.0, h);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        probe_param<K><<<blocks, threads>>>(out, steps, 1e-3, 5e-4, 1e-3 / 6.0, h);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return static_cast<double>(blocks) * threads * steps * 32.0 / (best * 1e-3);
}

template <int MODE, int C, bool LANEB = false>
double run(int warps_per_sm, int sms, double* out, const StageA* gtab) {
    int threads = warps_per_sm * 32;
    int per_sm = 1;
    while (threads > 1024) {
        threads /= 2;
        per_sm *= 2;
    }
    const size_t smem = MODE >= 2 && MODE < 20 && MODE != 5 && MODE != 7 ? kRows * sizeof(StageA) : 0;
    cudaFuncSetAttribute(probe<MODE, C, LANEB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int fit = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, probe<MODE, C, LANEB>, threads, smem);
    if (fit < per_sm) return -1.0;
    const int blocks = sms * per_sm;
    const int steps = 20000 / C;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe<MODE, C, LANEB><<<blocks, threads, smem>>>(out, 16, 1e-3, 5e-4, 1e-3 / 6.0, gtab, kB);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        probe<MODE, C, LANEB><<<blocks, threads, smem>>>(out, steps, 1e-3, 5e-4, 1e-3 / 6.0, gtab, kB);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return static_cast<double>(blocks) * threads * steps * C * 32.0 / (best * 1e-3);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    StageA* gtab;
    cudaMalloc(&out, 64);
    cudaMalloc(&gtab, kRows * sizeof(StageA));
    StageA h[kRows];
    for (int i = 0; i < kRows; ++i) h[i] = StageA{-5.0 - 1e-4 * i, -5.1, -5.2, -5.3};
    cudaMemcpy(gtab, h, sizeof h, cudaMemcpyHostToDevice);
    cudaMemcpyToSymbol(c_tab, h, kConstRows * sizeof(StageA));
    printf("executed FP64 op rate of the 32-op RK4 step (T op/s); -1 = does not fit\n");
    printf("%-18s %8s %8s %8s %8s %8s %8s %8s\n", "variant", "w1", "w4", "w16", "w24", "w32", "w48", "w64");
    const int ws[] = {1, 4, 16, 24, 32, 48, 64};
#define ROW(M, C, name)                                                         \
    {                                                                           \
        printf("%-18s", name);                                                  \
        for (int w : ws) printf(" %8.3f", run<M, C>(w, sms, out, gtab) / 1e12); \
        printf("\n");                                                           \
    }
#define ROW3(M, C, name)                                                              \
    {                                                                                 \
        printf("%-18s", name);                                                        \
        for (int w : ws) printf(" %8.3f", run<M, C, true>(w, sms, out, gtab) / 1e12); \
        printf("\n");                                                                 \
    }
    ROW(0, 1, "pure C=1");
    ROW3(0, 1, "pure laneb C=1");
    ROW(1, 1, "test C=1");
    ROW(4, 1, "table notest C=1");
    ROW(2, 1, "table C=1");
    ROW(5, 1, "ctable notest C=1");
    ROW(7, 1, "ctable test C=1");
    ROW(6, 1, "half table C=1");
    ROW(34, 1, "ctable+vote4 C=1");
    ROW(38, 1, "ctable+vote8 C=1");
    ROW(34, 2, "ctable+vote4 C=2");
    printf("cycles per step for one warp per SM (latency-bound regime): rate -> 148*32*32 ops per step\n");
    printf("%-18s", "ptable+vote8 C=1");
    for (int w : ws) printf(" %8.3f", run_param<8>(w, sms, out) / 1e12);
    printf("\n");
    printf("%-18s", "ptable+vote4 C=1");
    for (int w : ws) printf(" %8.3f", run_param<4>(w, sms, out) / 1e12);
    printf("\n");
    ROW(3, 1, "table+hi C=1");
    ROW(14, 1, "table+min4 C=1");
    ROW(18, 1, "table+min8 C=1");
    ROW(28, 1, "const+min8 C=1");
    ROW3(28, 1, "laneb+min8 C=1");
    ROW(0, 2, "pure C=2");
    ROW(2, 2, "table C=2");
    ROW(18, 2, "table+min8 C=2");
    ROW(14, 2, "table+min4 C=2");
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("CUDA error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
