// bmc_host.cpp -- host-side producers for the CUDA executor.
//
// Compiled by g++ with -ffp-contract=off (never by nvcc, never with
// -ffast-math): every FP64 expression here must round exactly like the
// reference build (/root/reference/proj/CMakeLists.txt:12-14), and the libm
// calls (log, cos, sqrt, sin) must be the same glibc entry points the
// reference calls.  That is why sampling and RolloutTerms staging stay on the
// host: glibc's log/cos/sin are not correctly rounded
// and cannot be regenerated bit-identically with CUDA's libdevice.
#include "bmc_internal.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>

namespace bmc {

namespace {
thread_local std::string t_error;
}

void set_error(const std::string& msg) { t_error = msg; }

int abi_exception() {
    try {
        throw;
    } catch (const std::bad_alloc&) {
        set_error("out of host memory");
        return BMC_E_NOMEM;
    } catch (const std::exception& e) {
        set_error(std::string("internal error: ") + e.what());
        return BMC_E_CONFIG;
    } catch (...) {
        set_error("internal error: unknown exception");
        return BMC_E_CONFIG;
    }
}
const std::string& get_error() { return t_error; }

// ----------------------------------------------------------------- world

int derive_world(const bmc_world& w, WorldDerived* out, std::string* err) {
    // integrator.hpp:39-68 (half, sixth), dynamics.hpp:96-106 (inv_tau),
    // integrator.cpp:19 (max_steps = llround(t_max / dt)).
    const double steps_real = w.t_max / w.dt;
    if (!std::isfinite(steps_real)) {
        *err = "sim.dt: t_max / dt must be finite";
        return BMC_E_CONFIG;
    }
    const long long max_steps = std::llround(steps_real);
    if (max_steps > 2147483647LL || max_steps < -2147483647LL) {
        *err = "sim.t_max: round(t_max / dt) must fit in 31 bits on the CUDA executor";
        return BMC_E_CONFIG;
    }
    out->dt = w.dt;
    out->half = 0.5 * w.dt;
    out->sixth = w.dt / 6.0;
    out->brake_cmd = w.brake_cmd;
    out->inv_tau = 1.0 / w.actuator_tau;
    out->max_steps = max_steps;
    return BMC_OK;
}

// The brake_accel lane of rk4_step (integrator.hpp:39-68) with
// state_derivative's third component (dynamics.hpp:130), same association.
ActuatorTable build_actuator_table(const WorldDerived& d, std::size_t cap) {
    ActuatorTable t;
    t.max_steps = d.max_steps;
    const std::size_t need = d.max_steps > 0 ? static_cast<std::size_t>(d.max_steps) : 1;
    t.stages.reserve(std::min(need, cap));
    double a = 0.0;
    for (;;) {
        const double k1 = (d.brake_cmd - a) * d.inv_tau;
        const double s2 = a + d.half * k1;
        const double k2 = (d.brake_cmd - s2) * d.inv_tau;
        const double s3 = a + d.half * k2;
        const double k3 = (d.brake_cmd - s3) * d.inv_tau;
        const double s4 = a + d.dt * k3;
        const double k4 = (d.brake_cmd - s4) * d.inv_tau;
        const double next = a + d.sixth * (((k1 + 2.0 * k2) + 2.0 * k3) + k4);
        t.stages.push_back(StageA{a, s2, s3, s4});
        uint64_t ba, bn;
        std::memcpy(&ba, &a, 8);
        std::memcpy(&bn, &next, 8);
        if (ba == bn || t.stages.size() >= need) {
            t.converged = true;  // fixed point reached, or every step covered
            break;
        }
        if (t.stages.size() >= cap) {
            t.converged = false;
            break;
        }
        a = next;
    }
    return t;
}

// -------------------------------------------------------------- sampler

namespace {

inline uint64_t splitmix_word(uint64_t seed, uint64_t counter) {
    // sampling.cpp:36-42
    uint64_t z = seed + (counter + 1u) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

inline double open_uniform(uint64_t seed, uint64_t counter) {
    // sampling.cpp:44-46
    return (static_cast<double>(splitmix_word(seed, counter) >> 12) + 0.5) * 0x1.0p-52;
}

inline double normal_deviate(uint64_t seed, uint64_t index) {
    // sampling.cpp:48-53 (glibc log / sqrt / cos, same entry points)
    const double u1 = open_uniform(seed, 2u * index);
    const double u2 = open_uniform(seed, 2u * index + 1u);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

inline double floor_clamp(double v, double lo, uint64_t& clamps) {
    if (v < lo) {
        ++clamps;
        return lo;
    }
    return v;
}

} // namespace

uint64_t draw_range_serial(const bmc_model& m, uint64_t first, std::size_t n, bmc_sample* out) {
    // sampling.cpp:67-100 for sample indices [first, first + n)
    const bmc_normal* spec[5] = {&m.initial_speed, &m.friction, &m.grade, &m.mass,
                                 &m.drag_coeff};
    uint64_t clamps = 0;
    for (std::size_t k = 0; k < n; ++k) {
        const uint64_t base = 5u * (first + k);
        double p[5];
        for (int j = 0; j < 5; ++j) {
            p[j] = spec[j]->mean + spec[j]->sd * normal_deviate(m.seed, base + j);
        }
        bmc_sample& s = out[k];
        s.initial_speed = floor_clamp(p[0], 0.1, clamps);
        s.friction = floor_clamp(p[1], 0.05, clamps);
        s.mass = floor_clamp(p[3], 500.0, clamps);
        s.drag_coeff = floor_clamp(p[4], 0.0, clamps);
        s.grade = p[2];
        if (s.grade > 1.5) {
            s.grade = 1.5;
            ++clamps;
        } else if (s.grade < -1.5) {
            s.grade = -1.5;
            ++clamps;
        }
    }
    return clamps;
}

int stage_terms_serial(const bmc_sample* s, std::size_t n, const bmc_world& w, double* v0,
                       double* floor, double* drag, double* grade) {
    // RolloutTerms::from (dynamics.cpp:57-68) + friction_limit (:48-55)
    for (std::size_t i = 0; i < n; ++i) {
        const double mu = s[i].friction;
        const double denom = 1.0 + mu * w.cg_height / w.wheelbase;
        if (!(denom > 0.0)) {
            return BMC_E_DOMAIN;
        }
        v0[i] = s[i].initial_speed;
        floor[i] = -(mu * w.gravity) / denom;
        drag[i] = 0.5 * w.air_density * s[i].drag_coeff * w.frontal_area / s[i].mass;
        grade[i] = w.gravity * std::sin(s[i].grade);
    }
    return BMC_OK;
}

int draw_terms_serial(const bmc_model& m, uint64_t first, std::size_t n, const bmc_world& w,
                      double* v0, double* floor, double* drag, double* grade, uint64_t* clamps) {
    // draw_batch (sampling.cpp:67-100) fused with RolloutTerms::from
    // (dynamics.cpp:57-68): no AoS sample is materialised, each sample goes
    // straight into the pinned SoA staging buffers.
    constexpr std::size_t kBlock = 256;
    bmc_sample tmp[kBlock];
    uint64_t c = 0;
    for (std::size_t b = 0; b < n; b += kBlock) {
        const std::size_t k = std::min(kBlock, n - b);
        c += draw_range_serial(m, first + b, k, tmp);
        const int rc = stage_terms_serial(tmp, k, w, v0 + b, floor + b, drag + b, grade + b);
        if (rc != BMC_OK) return rc;
    }
    if (clamps) *clamps += c;
    return BMC_OK;
}

// ------------------------------------------------------------ thread pool

ThreadPool::ThreadPool(unsigned threads) {
    const unsigned extra = threads > 1 ? threads - 1 : 0;
    for (unsigned i = 0; i < extra; ++i) {
        workers_.emplace_back([this, i] { worker_main(i + 1); });
    }
}

ThreadPool::~ThreadPool() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
}

void ThreadPool::worker_main(unsigned id) {
    uint64_t seen = 0;
    for (;;) {
        const std::function<void(std::size_t, std::size_t)>* job;
        std::size_t n;
        unsigned parts;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || generation_ != seen; });
            if (stop_) return;
            seen = generation_;
            job = job_;
            n = job_n_;
            parts = job_parts_;
        }
        if (id < parts) {
            const std::size_t b = n * id / parts, e = n * (id + 1) / parts;
            if (b < e) (*job)(b, e);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
}

void ThreadPool::parallel_for(std::size_t n,
                              const std::function<void(std::size_t, std::size_t)>& fn,
                              unsigned max_threads) {
    if (n == 0) return;
    std::lock_guard<std::mutex> call(call_mu_);
    unsigned parts = size();
    if (max_threads > 0) parts = std::min(parts, max_threads);
    parts = static_cast<unsigned>(std::min<std::size_t>(parts, n));
    if (parts <= 1) {
        fn(0, n);
        return;
    }
    {
        std::lock_guard<std::mutex> lk(mu_);
        job_ = &fn;
        job_n_ = n;
        job_parts_ = parts;
        pending_ = parts - 1;
        ++generation_;
    }
    cv_.notify_all();
    fn(0, n / parts);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
}

unsigned resolve_threads(int requested) {
    if (requested > 0) return static_cast<unsigned>(requested);
    const unsigned hc = std::thread::hardware_concurrency();
    // one process per GPU (torchrun sets LOCAL_WORLD_SIZE): share the host's
    // cores between the local ranks instead of oversubscribing them
    unsigned local = 1;
    if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) {
        const long v = std::strtol(e, nullptr, 10);
        if (v > 1) local = static_cast<unsigned>(v);
    }
    const unsigned t = (hc ? hc : 1u) / local;
    return t ? t : 1u;
}

ThreadPool& host_pool() {
    // One pool per process, sized to the hardware; callers cap per call.
    static ThreadPool pool(resolve_threads(0));
    return pool;
}

} // namespace bmc

// ---------------------------------------------------------------- C-ABI

extern "C" int bmc_draw_range(const bmc_model* model, uint64_t first, size_t n, bmc_sample* out,
                              uint64_t* clamp_count, int threads) {
    try {
        if (model == nullptr || out == nullptr) {
            bmc::set_error("bmc_draw_range: null argument");
            return BMC_E_CONFIG;
        }
        if (n == 0) {
            bmc::set_error("samples: must be >= 1");  // sampling.cpp:68-70
            return BMC_E_CONFIG;
        }
        std::atomic<uint64_t> clamps{0};
        bmc::host_pool().parallel_for(
            n,
            [&](std::size_t b, std::size_t e) {
                clamps += bmc::draw_range_serial(*model, first + b, e - b, out + b);
            },
            bmc::resolve_threads(threads));
        if (clamp_count) *clamp_count = clamps.load();
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception();
    }
}

extern "C" int bmc_stage_terms(const bmc_sample* samples, size_t n, const bmc_world* world,
                               double* v0, double* floor, double* drag, double* grade,
                               int threads) {
    try {
        if (samples == nullptr || world == nullptr || !v0 || !floor || !drag || !grade) {
            bmc::set_error("bmc_stage_terms: null argument");
            return BMC_E_CONFIG;
        }
        std::atomic<int> status{BMC_OK};
        bmc::host_pool().parallel_for(
            n,
            [&](std::size_t b, std::size_t e) {
                const int rc = bmc::stage_terms_serial(samples + b, e - b, *world, v0 + b,
                                                       floor + b, drag + b, grade + b);
                if (rc != BMC_OK) status = rc;
            },
            bmc::resolve_threads(threads));
        if (status != BMC_OK) {
            bmc::set_error("friction_limit: weight-transfer denominator <= 0");
            return status;
        }
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception();
    }
}

// ------------------------------------------------------------ results.csv

// results_csv (io.cpp:17-31): "index,d_stop_m,t_stop_s,horizon_flag", doubles
// as glibc "%.17g" (io.cpp:11-15; same libc call => same bytes), formatted
// by the host pool in slices and written in index order.
extern "C" int bmc_write_results_csv(const char* path, const bmc_result* r, size_t n,
                                     int threads) {
    try {
        if (!path || (n && !r)) {
            bmc::set_error("bmc_write_results_csv: null argument");
            return BMC_E_CONFIG;
        }
        std::FILE* f = std::fopen(path, "wb");
        if (!f) {
            bmc::set_error(std::string("cannot open for writing: ") + path);  // IoError analogue
            return BMC_E_IO;
        }
        const char* header = "index,d_stop_m,t_stop_s,horizon_flag\n";
        bool ok = std::fputs(header, f) >= 0;
        const std::size_t kSlice = std::size_t{1} << 18;
        std::vector<std::string> bufs;
        for (std::size_t s0 = 0; ok && s0 < n; s0 += kSlice * 64) {
            const std::size_t s1 = std::min(n, s0 + kSlice * 64);
            const std::size_t parts = (s1 - s0 + kSlice - 1) / kSlice;
            bufs.assign(parts, std::string());
            bmc::host_pool().parallel_for(
                parts,
                [&](std::size_t b, std::size_t e) {
                    char line[128];
                    for (std::size_t p = b; p < e; ++p) {
                        std::string& out = bufs[p];
                        const std::size_t i0 = s0 + p * kSlice, i1 = std::min(s1, i0 + kSlice);
                        out.reserve((i1 - i0) * 48);
                        for (std::size_t i = i0; i < i1; ++i) {
                            const int len = std::snprintf(line, sizeof line, "%zu,%.17g,%.17g,%c\n", i,
                                                          r[i].stop_distance, r[i].stop_time,
                                                          r[i].hit_horizon ? '1' : '0');
                            out.append(line, static_cast<std::size_t>(len));
                        }
                    }
                },
                bmc::resolve_threads(threads));
            for (const auto& b : bufs) {
                if (std::fwrite(b.data(), 1, b.size(), f) != b.size()) ok = false;
            }
        }
        if (std::fclose(f) != 0) ok = false;
        if (!ok) {
            bmc::set_error(std::string("write failed: ") + path);
            return BMC_E_IO;
        }
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception();
    }
}

// parse_results_csv (io.cpp:94-123) + the step reconstruction of cmd_verify
// (cli.cpp:96-100: steps = llround(t_stop / dt)).  *n_out is the row count;
// BMC_E_RANGE if it exceeds cap (then *n_out is the count needed).
extern "C" int bmc_read_results_csv(const char* path, double dt, bmc_result* out, size_t cap,
                                    size_t* n_out) {
    try {
        if (!path || !n_out) {
            bmc::set_error("bmc_read_results_csv: null argument");
            return BMC_E_CONFIG;
        }
        std::FILE* f = std::fopen(path, "rb");
        if (!f) {
            bmc::set_error(std::string("cannot open for reading: ") + path);
            return BMC_E_IO;
        }
        char line[512];
        if (!std::fgets(line, sizeof line, f) ||
            std::strcmp(line, "index,d_stop_m,t_stop_s,horizon_flag\n") != 0) {
            std::fclose(f);
            bmc::set_error("results csv: missing or unexpected header");
            return BMC_E_IO;
        }
        std::size_t count = 0, line_no = 1;
        int rc = BMC_OK;
        while (std::fgets(line, sizeof line, f)) {
            ++line_no;
            if (line[0] == '\n' || line[0] == '\0') continue;
            unsigned long long index = 0;
            unsigned flag = 0;
            double d = 0.0, t = 0.0;
            if (std::sscanf(line, "%llu,%lf,%lf,%u", &index, &d, &t, &flag) != 4) {
                bmc::set_error("results csv: malformed line " + std::to_string(line_no));
                rc = BMC_E_IO;
                break;
            }
            if (index != count) {
                bmc::set_error("results csv: non-contiguous index at line " + std::to_string(line_no));
                rc = BMC_E_IO;
                break;
            }
            if (out && count < cap) {
                bmc_result r;
                std::memset(&r, 0, sizeof r);
                r.stop_distance = d;
                r.stop_time = t;
                r.steps = std::llround(t / dt);
                r.hit_horizon = flag != 0 ? 1 : 0;
                out[count] = r;
            }
            ++count;
        }
        std::fclose(f);
        *n_out = count;
        if (rc != BMC_OK) return rc;
        if (count > cap) {
            bmc::set_error("results csv: output buffer too small");
            return BMC_E_RANGE;
        }
        return BMC_OK;
    } catch (...) {
        return bmc::abi_exception();
    }
}

extern "C" const char* bmc_last_error(void) { return bmc::get_error().c_str(); }
extern "C" int bmc_abi_version(void) { return BMC_ABI_VERSION; }
