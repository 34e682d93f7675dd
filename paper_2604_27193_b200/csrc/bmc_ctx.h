// bmc_ctx.h -- the device context behind the opaque bmc_ctx handle, shared
// by the C-ABI translation units (bmc_capi.cpp, bmc_capi_stats.cpp,
// bmc_graph.cpp).
#pragma once

#include "bmc_kernels.h"
#include "bmc_stats.h"

#include <memory>
#include <string>
#include <vector>

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

// Events around the stages of one rollout launch: binning (p0..p1),
// rollout (r0..r1), unpermute (r1..u1).
struct KernelEvents {
    cudaEvent_t p0 = nullptr, p1 = nullptr, r0 = nullptr, r1 = nullptr, u1 = nullptr;
    bool predicted = false, unpermuted = false;
    cudaError_t create() {
        cudaError_t e;
        if ((e = cudaEventCreate(&p0)) != cudaSuccess) return e;
        if ((e = cudaEventCreate(&p1)) != cudaSuccess) return e;
        if ((e = cudaEventCreate(&r0)) != cudaSuccess) return e;
        if ((e = cudaEventCreate(&u1)) != cudaSuccess) return e;
        return cudaEventCreate(&r1);
    }
    void destroy() {
        for (cudaEvent_t* ev : {&p0, &p1, &r0, &r1, &u1}) {
            if (*ev) cudaEventDestroy(*ev);
            *ev = nullptr;
        }
    }
};

// Device buffers one rollout launch needs besides its inputs/outputs.
// A CUDA graph owns its own Scratch so captured pointers stay valid.
struct Scratch {
    DevBuf keys, perm, hist, counter, packed_in, packed_out;
    void release() {
        keys.release();
        perm.release();
        hist.release();
        counter.release();
        packed_in.release();
        packed_out.release();
    }
};

// Everything a rollout launch needs that depends on the world, not on the
// samples: the actuator table, the predictor's coarse table and the chosen
// kernel variant.  Pointers refer to ctx-owned (or graph-owned) buffers.
struct Plan {
    WorldDerived d{};
    int mode = kTableNone;
    int sched = kScheduleIndex;
    int bt = 1024;
    int ilp = 1;
    int test_block = 1;
    const StageA* table = nullptr;
    int table_len = 0;
    double table_min = 0.0;
    const float* coarse = nullptr;
    int coarse_len = 0;
    float coarse_h = 0.0f;
    int coarse_steps = 0;
    float coarse_inf = 0.0f;
};

// One pipeline slot: its own compute stream and rollout scratch, so chunk
// k+1's binning and rollout fill the SMs chunk k's persistent rollout
// releases during its tail instead of waiting for the whole kernel.
struct Slot {
    cudaStream_t compute = nullptr;
    Scratch sc;
    PinBuf h_terms, h_out;
    DevBuf d_terms, d_out;
    cudaEvent_t h2d_done = nullptr, compute_done = nullptr, d2h_done = nullptr;
    KernelEvents kev;
    size_t offset = 0, len = 0;
    bool busy = false;
};

}  // namespace bmc

namespace bmc {

// The device tables one world needs (actuator stage table, predictor's coarse
// table).  Entries are immutable once built: a launch in flight always reads
// the table of its own world, whatever world a later call asks for (a new
// world gets a new entry; eviction frees, and cudaFree waits for the device).
struct TableEntry {
    WorldDerived key{};
    bool converged = false;
    double t_min = 0.0;
    int t_len = 0;
    DevBuf table, coarse;
    int coarse_len = 0;
    float coarse_h = 0.0f;
    int coarse_steps = 0;     // predictor: numeric coarse steps (transient)
    float coarse_inf = 0.0f;  // predictor: brake_accel after the transient
    ~TableEntry() {
        table.release();
        coarse.release();
    }
};
constexpr size_t kTableCacheEntries = 4;

}  // namespace bmc

struct bmc_ctx {
    int device = 0;
    int sms = 0;
    cudaStream_t stream = nullptr, h2d = nullptr, d2h = nullptr;
    bmc::KernelEvents kev;
    std::string err;
    std::mutex mu;

    // most recently used first
    std::vector<std::unique_ptr<bmc::TableEntry>> tables;

    // host staging / unpack workers of THIS context (one pool per device,
    // so several devices driven from one process never queue on each other)
    std::unique_ptr<bmc::ThreadPool> pool;
    unsigned pool_threads = 0;

    // the per-context scratch below is reused by every device-resident call;
    // each launch waits for the previous one's completion event, whatever
    // stream either was enqueued on
    cudaEvent_t scratch_done = nullptr;
    bool scratch_used = false;

    bmc::Scratch scratch;
    bmc::DevBuf total_steps;
    bmc::DevBuf draw_ctr;  // device sampler: u64 clamp count + u32 flags
    uint32_t last_launches = 0;

    // the stage bmc_cuda_stats reuses while the request and size class match
    bmc_stats_stage* stats_cache = nullptr;

    // pipeline slots (bmc_capi.cpp run_pipeline): three, so a chunk's host
    // staging never waits on the chunk the device finished last
    bmc::Slot slots[3];
    bmc::DevBuf partials, sel_hist, sel_pref, sorted_h, buckets, hist_buf;
};

namespace bmc {

inline int fail(bmc_ctx* ctx, int code, const std::string& msg) {
    set_error(msg);
    if (ctx) ctx->err = msg;
    return code;
}

// abi_exception() that also records the message on the context
inline int abi_exception(bmc_ctx* ctx) {
    const int rc = abi_exception();
    if (ctx) ctx->err = get_error();
    return rc;
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

// bmc_capi.cpp
// The (cached, immutable) table entry of a world.
int ensure_table(bmc_ctx* ctx, const WorldDerived& d, TableEntry** out);
// This context's host pool, grown to at least `threads` workers.
ThreadPool& ctx_pool(bmc_ctx* ctx, unsigned threads);
int make_plan(bmc_ctx* ctx, const WorldDerived& d, const bmc_run_opts& opts, uint64_t n,
              Plan* plan);
// Output path of a binned launch: -1 = the default (packed sorted records +
// unpermute; BMC_DIRECT_OUTPUTS=1 flips it), 0 = packed + unpermute,
// 1 = direct writes at each sample's index through the forward map.
int reserve_scratch(bmc_ctx* ctx, Scratch& sc, const Plan& plan, uint64_t n, int direct = -1);
// 1 when a launch of n results writes them directly (13 B/result <= 64 MiB:
// they merge in L2): the streamed pipeline's chunks and the decision graph.
int direct_outputs_for(uint64_t n);
// Device sampler (bmc_capi.cpp): resolve bmc_run_opts.sampler to a yes/no.
int use_device_sampler(bmc_ctx* ctx, const bmc_run_opts& o, bool* device);
// Fill DrawArgs from a model + world (no output pointers set).
DrawArgs draw_args(const bmc_model& m, uint64_t first, uint64_t n, const bmc_world& w);
// Read back + reset the draw counters; maps flags to BMC_E_DOMAIN/RANGE.
int finish_draw(bmc_ctx* ctx, const DevBuf& ctr, uint64_t* clamps);
bool device_sampler_supported(std::string* why);  // bmc_libm_check.cpp

// Statistics stage pieces a CUDA graph captures (bmc_capi_stats.cpp).
int stats_stage_create(bmc_ctx* ctx, const bmc_stats_req* req, size_t max_n, bmc_stats_stage** out);
int stats_begin_enqueue(bmc_stats_stage* st, cudaStream_t s);
// pass-1 words for a rollout; false when the headways are too many to fuse
bool stats_p1_args(bmc_stats_stage* st, P1Args* p1);
void fit_stats_plan(Plan* plan, const P1Args& p1);
// every device stage with no merge (no host read back: capturable)
int stats_enqueue_device(bmc_stats_stage* st, const double* d, const uint8_t* hz, uint64_t n,
                         cudaStream_t s);
// the words the host composition reads, copied into a pinned mirror laid
// out like the stage memory (stats_mirror_words words)
size_t stats_mirror_words(const bmc_stats_stage* st);
int stats_enqueue_readback(bmc_stats_stage* st, uint64_t* mirror, cudaStream_t s);
int stats_compose_mirror(bmc_stats_stage* st, const uint64_t* mirror, const double* d,
                         const uint8_t* hz, uint64_t n, bmc_stats* out);
uint32_t stats_launches(const bmc_stats_stage* st);
size_t stats_max_n(const bmc_stats_stage* st);
// Enqueue predictor/binning (when planned) + rollout on `s`.  ev may be
// null (no timing events, e.g. under stream capture).
// p1 (nullable): fuse statistics pass 1 into the rollout epilogue.
int enqueue_rollout(bmc_ctx* ctx, const Plan& plan, Scratch& sc, const bmc_terms& terms,
                    uint64_t n, const bmc_outputs& out, unsigned long long* total_steps_dev,
                    cudaStream_t s, KernelEvents* ev, uint32_t* launches,
                    const P1Args* p1 = nullptr, int direct = -1);
// Legacy statistics calls run on ctx->stream: order them after the last
// device-resident rollout, whatever stream it was enqueued on.
inline int order_after_rollouts(bmc_ctx* ctx) {
    if (ctx->scratch_used) BMC_CK(ctx, cudaStreamWaitEvent(ctx->stream, ctx->scratch_done, 0));
    return BMC_OK;
}

}  // namespace bmc
