// bmc_nccl.cpp -- NCCL merge hooks for the statistics stage (brakemc_cuda.h
// bmc_nccl_*): one communicator per device from one process
// (ncclCommInitAll), and a bmc_merge per rank whose allreduce / allgather run
// ncclAllReduce / ncclAllGather on the stage's own stream -- the collective is
// ordered with the stage kernels on the device, no host staging.  Partials
// are u64 words: SUM for counts, limbs and histograms, MIN for the extrema
// keys ("one ncclAllReduce phase per run ... integer results
// bit-identical for any GPU count").
//
// libnccl is opened at run time (dlopen "libnccl.so.2", or BMC_NCCL_LIB), so
// the product library keeps no link-time dependency on it; callers that never
// merge across devices never load it.  g++ -ffp-contract=off.
#include "bmc_ctx.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>
#include <vector>

struct bmc_comm {
    ncclComm_t comm = nullptr;
    int device = 0;
    int rank = 0;
    int world = 1;
    bmc_merge merge{};
};

namespace bmc {
namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    int version = 0;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
};

const NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* path = std::getenv("BMC_NCCL_LIB");
        void* h = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("dlopen libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) {
            void* p = dlsym(h, name);
            if (!p) a.why = std::string("libnccl: missing ") + name;
            return p;
        };
        a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(sym("ncclCommInitAll"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
        a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
        a.GetVersion = reinterpret_cast<decltype(a.GetVersion)>(sym("ncclGetVersion"));
        if (a.CommInitAll && a.CommDestroy && a.AllReduce && a.AllGather && a.GetErrorString &&
            a.GetVersion) {
            a.GetVersion(&a.version);
            a.ok = true;
        }
    });
    return a;
}

// ---- bmc_merge hooks (user = bmc_comm*)
int nccl_allreduce(void* user, uint64_t* buf, size_t count, int op, void* stream) {
    auto* c = static_cast<bmc_comm*>(user);
    const NcclApi& a = api();
    ncclRedOp_t r = op == BMC_MERGE_MIN ? ncclMin : op == BMC_MERGE_MAX ? ncclMax : ncclSum;
    const ncclResult_t e = a.AllReduce(buf, buf, count, ncclUint64, r, c->comm,
                                       static_cast<cudaStream_t>(stream));
    if (e != ncclSuccess) set_error(std::string("ncclAllReduce: ") + a.GetErrorString(e));
    return e == ncclSuccess ? 0 : 1;
}

int nccl_allgather(void* user, const uint64_t* send, uint64_t* recv, size_t count, void* stream) {
    auto* c = static_cast<bmc_comm*>(user);
    const NcclApi& a = api();
    const ncclResult_t e = a.AllGather(send, recv, count, ncclUint64, c->comm,
                                       static_cast<cudaStream_t>(stream));
    if (e != ncclSuccess) set_error(std::string("ncclAllGather: ") + a.GetErrorString(e));
    return e == ncclSuccess ? 0 : 1;
}

}  // namespace
}  // namespace bmc

using bmc::fail;

extern "C" {

int bmc_nccl_available(int* version) {
    try {
        const bmc::NcclApi& a = bmc::api();
        if (version) *version = a.version;
        if (!a.ok) return fail(nullptr, BMC_E_CUDA, a.why);
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception();
    }
}

int bmc_nccl_init_all(int ndev, const int* devices, bmc_comm** comms) {
    try {
        if (ndev < 1 || !devices || !comms) return fail(nullptr, BMC_E_CONFIG, "bmc_nccl_init_all: bad arguments");
        const bmc::NcclApi& a = bmc::api();
        if (!a.ok) return fail(nullptr, BMC_E_CUDA, a.why);
        std::vector<ncclComm_t> c(static_cast<size_t>(ndev), nullptr);
        const ncclResult_t e = a.CommInitAll(c.data(), ndev, devices);
        if (e != ncclSuccess) return fail(nullptr, BMC_E_CUDA, std::string("ncclCommInitAll: ") + a.GetErrorString(e));
        for (int r = 0; r < ndev; ++r) {
            auto* x = new bmc_comm;
            x->comm = c[static_cast<size_t>(r)];
            x->device = devices[r];
            x->rank = r;
            x->world = ndev;
            x->merge.user = x;
            x->merge.world = ndev;
            x->merge.rank = r;
            x->merge.allreduce_u64 = bmc::nccl_allreduce;
            x->merge.allgather_u64 = bmc::nccl_allgather;
            comms[r] = x;
        }
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception();
    }
}

const bmc_merge* bmc_nccl_merge(const bmc_comm* comm) { return comm ? &comm->merge : nullptr; }

void bmc_nccl_destroy(bmc_comm* comm) {
    if (!comm) return;
    const bmc::NcclApi& a = bmc::api();
    if (a.ok && comm->comm) {
        cudaSetDevice(comm->device);
        a.CommDestroy(comm->comm);
    }
    delete comm;
}

}  // extern "C"
