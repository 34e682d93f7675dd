// bmc_internal.h -- shared declarations between the host staging code
// (bmc_host.cpp, g++ -ffp-contract=off), the kernels (bmc_kernels.cu,
// nvcc -fmad=false) and the C-ABI layer (bmc_capi.cpp).
#pragma once

#include "brakemc_cuda.h"

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace bmc {

// One RK4 step's actuator stage values (a, s2.a, s3.a, s4.a), integrator.hpp:39-68.
struct StageA {
    double a0, a1, a2, a3;
};

// Sample-independent actuator trajectory.  The brake_accel component of the
// RK4 state never reads position or speed (dynamics.hpp:126-132), so for a
// fixed (dt, brake_cmd, inv_tau) every rollout walks the same FP64 sequence.
// It is tabulated once per batch with the reference's exact operation order;
// once a_{n+1} == a_n bit-for-bit the sequence is constant forever (the step
// is a pure function of a_n).  len = entries stored; entries >= len-1 repeat
// the last one.  converged == false means the table was truncated at the cap
// and the kernel must not use it.
struct ActuatorTable {
    std::vector<StageA> stages;
    int64_t max_steps = 0;
    bool converged = false;
};

struct WorldDerived {
    double dt, half, sixth, brake_cmd, inv_tau;
    int64_t max_steps;
};

// Host-side exact derivations (bmc_host.cpp).
int derive_world(const bmc_world& w, WorldDerived* out, std::string* err);
ActuatorTable build_actuator_table(const WorldDerived& d, std::size_t cap);

// Persistent worker pool for host staging / unpack (fork-join parallel_for).
class ThreadPool {
public:
    explicit ThreadPool(unsigned threads);
    ~ThreadPool();
    unsigned size() const { return static_cast<unsigned>(workers_.size()) + 1; }
    // Calls fn(begin, end) over [0, n) split into contiguous slices; the
    // calling thread takes part.  Blocks until every slice is done.
    void parallel_for(std::size_t n, const std::function<void(std::size_t, std::size_t)>& fn,
                      unsigned max_threads = 0);

private:
    void worker_main(unsigned id);
    std::vector<std::thread> workers_;
    std::mutex call_mu_;  // serialises concurrent parallel_for callers
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(std::size_t, std::size_t)>* job_ = nullptr;
    std::size_t job_n_ = 0;
    unsigned job_parts_ = 0;
    unsigned pending_ = 0;
    uint64_t generation_ = 0;
    bool stop_ = false;
};

ThreadPool& host_pool();
unsigned resolve_threads(int requested);

// Host producers (bmc_host.cpp).
uint64_t draw_range_serial(const bmc_model& m, uint64_t first, std::size_t n, bmc_sample* out);
int stage_terms_serial(const bmc_sample* s, std::size_t n, const bmc_world& w, double* v0,
                       double* floor, double* drag, double* grade);
int draw_terms_serial(const bmc_model& m, uint64_t first, std::size_t n, const bmc_world& w,
                      double* v0, double* floor, double* drag, double* grade, uint64_t* clamps);

void set_error(const std::string& msg);
// Called from the catch (...) around every C-ABI entry point: the in-flight
// C++ exception becomes an error code + message (no exception crosses the
// ABI).  std::bad_alloc -> BMC_E_NOMEM, anything else -> BMC_E_CONFIG.
int abi_exception();
const std::string& get_error();

} // namespace bmc
