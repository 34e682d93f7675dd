// bmc_ctx.h -- the device context behind the opaque bmc_ctx handle, shared
// by the C-ABI translation units (bmc_capi.cpp, bmc_capi_stats.cpp).
#pragma once

#include "bmc_kernels.h"
#include "bmc_stats.h"

#include <string>

namespace bmc {

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t reserve(size_t b) {
        if (b <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        const cudaError_t e = cudaMalloc(&p, b);
        if (e == cudaSuccess) bytes = b;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct PinBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t reserve(size_t b) {
        if (b <= bytes) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        const cudaError_t e = cudaHostAlloc(&p, b, cudaHostAllocDefault);
        if (e == cudaSuccess) bytes = b;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct KernelEvents {
    cudaEvent_t p0 = nullptr, p1 = nullptr, r0 = nullptr, r1 = nullptr;
    bool predicted = false;
    cudaError_t create() {
        cudaError_t e;
        if ((e = cudaEventCreate(&p0)) != cudaSuccess) return e;
        if ((e = cudaEventCreate(&p1)) != cudaSuccess) return e;
        if ((e = cudaEventCreate(&r0)) != cudaSuccess) return e;
        return cudaEventCreate(&r1);
    }
    void destroy() {
        for (cudaEvent_t* ev : {&p0, &p1, &r0, &r1}) {
            if (*ev) cudaEventDestroy(*ev);
            *ev = nullptr;
        }
    }
};

struct Slot {
    PinBuf h_terms, h_out;
    DevBuf d_terms, d_out;
    cudaEvent_t h2d_done = nullptr, compute_done = nullptr, d2h_done = nullptr;
    KernelEvents kev;
    size_t offset = 0, len = 0;
    bool busy = false;
};

}  // namespace bmc

struct bmc_ctx {
    int device = 0;
    int sms = 0;
    cudaStream_t stream = nullptr, h2d = nullptr, d2h = nullptr;
    bmc::KernelEvents kev;
    std::string err;
    std::mutex mu;

    bool have_table = false;
    bmc::WorldDerived tkey{};
    bool t_converged = false;
    double t_min = 0.0;
    int t_len = 0;
    bmc::DevBuf d_table, d_coarse;
    int coarse_len = 0;
    float coarse_h = 0.0f;

    bmc::DevBuf keys, perm, hist, counter, total_steps;
    uint32_t last_launches = 0;
    float last_roll_ms = 0.0f, last_pred_ms = 0.0f;

    bmc::Slot slots[2];
    bmc::DevBuf partials, sel_hist, sel_pref, sorted_h, buckets, hist_buf;
    bmc::PinBuf h_small;
};


namespace bmc {

inline int fail(bmc_ctx* ctx, int code, const std::string& msg) {
    set_error(msg);
    if (ctx) ctx->err = msg;
    return code;
}

#define BMC_CK(ctx, expr)                                                                   \
    do {                                                                                    \
        const cudaError_t e_ = (expr);                                                      \
        if (e_ != cudaSuccess)                                                              \
            return ::bmc::fail((ctx), BMC_E_CUDA,                                           \
                               std::string(#expr) + ": " + cudaGetErrorString(e_));         \
    } while (0)

inline int prepare(bmc_ctx* ctx) {
    if (ctx == nullptr) {
        set_error("bmc: null context");
        return BMC_E_CONFIG;
    }
    BMC_CK(ctx, cudaSetDevice(ctx->device));
    return BMC_OK;
}


}  // namespace bmc
