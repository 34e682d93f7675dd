/*
 * bmc_oracle.c -- CPU restatement of the brakemc rollout path (parity checker).
 *
 * TEST INFRASTRUCTURE ONLY -- see bmc_oracle.h.  Build: oracle/Makefile
 * (gcc -O2 -ffp-contract=off, matching the reference's no-contraction build,
 * /root/reference/proj/CMakeLists.txt:12-14).  All arithmetic below keeps the
 * reference's association order literally; each block cites the reference
 * line it restates (paths relative to /root/reference/proj).
 */
#include "bmc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ sampler */

/* sampling.cpp:36-42 -- splitmix64 output at state seed + (counter+1)*gamma */
uint64_t orc_stream_word(uint64_t seed, uint64_t counter) {
    uint64_t z = seed + (counter + 1u) * UINT64_C(0x9E3779B97F4A7C15);
    z = (z ^ (z >> 30)) * UINT64_C(0xBF58476D1CE4E5B9);
    z = (z ^ (z >> 27)) * UINT64_C(0x94D049BB133111EB);
    return z ^ (z >> 31);
}

/* sampling.cpp:44-46 -- top 52 bits, half-ulp offset, scaled by 2^-52 */
double orc_stream_uniform(uint64_t seed, uint64_t counter) {
    const uint64_t top = orc_stream_word(seed, counter) >> 12;
    return ((double)top + 0.5) * 0x1.0p-52;
}

/* sampling.cpp:48-53 -- Box-Muller on counters (2i, 2i+1), glibc libm */
double orc_standard_normal_at(uint64_t seed, uint64_t stream_index) {
    const double u1 = orc_stream_uniform(seed, 2u * stream_index);
    const double u2 = orc_stream_uniform(seed, 2u * stream_index + 1u);
    const double r = sqrt(-2.0 * log(u1));
    return r * cos(6.283185307179586 * u2);
}

/* sampling.cpp:55-64 -- lower clamp that counts */
static double clamp_low(double value, double lo, uint64_t* count) {
    if (value < lo) {
        *count += 1u;
        return lo;
    }
    return value;
}

/* sampling.cpp:67-100 -- sample i owns stream indices 5i..5i+4 in the order
 * (initial_speed, friction, grade, mass, drag_coeff); unphysical tails are
 * clamped and counted.  Restated for an arbitrary index window so that a
 * shard [first, first+n) equals the same slice of draw_batch(model, N). */
uint64_t orc_draw_range(const orc_model* m, uint64_t first, size_t n, orc_sample* out) {
    uint64_t clamps = 0;
    for (size_t k = 0; k < n; ++k) {
        const uint64_t base = 5u * (first + (uint64_t)k);
        double p[5];
        for (int j = 0; j < 5; ++j) {
            p[j] = m->mean[j] + m->sd[j] * orc_standard_normal_at(m->seed, base + (uint64_t)j);
        }
        orc_sample* s = &out[k];
        s->initial_speed = clamp_low(p[0], 0.1, &clamps);
        s->friction = clamp_low(p[1], 0.05, &clamps);
        s->grade = p[2];
        s->mass = clamp_low(p[3], 500.0, &clamps);
        s->drag_coeff = clamp_low(p[4], 0.0, &clamps);
        if (s->grade > 1.5) {
            s->grade = 1.5;
            clamps += 1u;
        } else if (s->grade < -1.5) {
            s->grade = -1.5;
            clamps += 1u;
        }
    }
    return clamps;
}

/* ----------------------------------------------------------------- dynamics */

/* dynamics.cpp:48-55 -- -(mu*g) / (1 + mu*h/L), denominator checked */
int orc_friction_limit(double mu, const orc_world* w, double* out) {
    const double denom = 1.0 + mu * w->cg_height / w->wheelbase;
    if (!(denom > 0.0)) {
        return -1;
    }
    *out = -(mu * w->gravity) / denom;
    return 0;
}

/* dynamics.cpp:57-68 -- per-rollout constants; left-to-right drag product */
int orc_rollout_terms(const orc_sample* s, const orc_world* w, double out[5]) {
    if (orc_friction_limit(s->friction, w, &out[0]) != 0) {
        return -1;
    }
    out[1] = 0.5 * w->air_density * s->drag_coeff * w->frontal_area / s->mass;
    out[2] = w->gravity * sin(s->grade);
    out[3] = w->brake_cmd;
    out[4] = 1.0 / w->actuator_tau;
    return 0;
}

/* dynamics.hpp:82-84, 115-118, 126-132 -- the RHS with the ternary clamp */
static void rhs(const double st[3], const double t[5], double d[3]) {
    const double braking = st[2] > t[0] ? st[2] : t[0];
    d[0] = st[1];
    d[1] = braking - t[1] * (st[1] * st[1]) - t[2];
    d[2] = (t[3] - st[2]) * t[4];
}

/* integrator.hpp:39-68 -- classical RK4, component-wise fixed order */
void orc_rk4_step(double st[3], const double t[5], double dt) {
    const double half = 0.5 * dt;
    double k1[3], k2[3], k3[3], k4[3], s[3];
    rhs(st, t, k1);
    for (int c = 0; c < 3; ++c) s[c] = st[c] + half * k1[c];
    rhs(s, t, k2);
    for (int c = 0; c < 3; ++c) s[c] = st[c] + half * k2[c];
    rhs(s, t, k3);
    for (int c = 0; c < 3; ++c) s[c] = st[c] + dt * k3[c];
    rhs(s, t, k4);
    const double sixth = dt / 6.0;
    for (int c = 0; c < 3; ++c) {
        st[c] = st[c] + sixth * (((k1[c] + 2.0 * k2[c]) + 2.0 * k3[c]) + k4[c]);
    }
}

/* integrator.cpp:13-29 -- run to the first post-step v <= 0, else horizon */
int orc_rollout(const orc_sample* s, const orc_world* w, orc_result* out) {
    double t[5];
    if (orc_rollout_terms(s, w, t) != 0) {
        return -1;
    }
    double st[3] = {0.0, s->initial_speed, 0.0};
    const int64_t max_steps = llround(w->t_max / w->dt);
    memset(out, 0, sizeof *out);
    for (int64_t step = 1; step <= max_steps; ++step) {
        orc_rk4_step(st, t, w->dt);
        if (st[1] <= 0.0) {
            out->stop_distance = st[0];
            out->stop_time = (double)step * w->dt;
            out->steps = step;
            out->hit_horizon = 0;
            return 0;
        }
    }
    out->stop_distance = st[0];
    out->stop_time = (double)max_steps * w->dt;
    out->steps = max_steps;
    out->hit_horizon = 1;
    return 0;
}

typedef struct {
    const orc_sample* s;
    const orc_world* w;
    orc_result* out;
    size_t begin, end;
    int status;
} run_slice;

static void* run_slice_main(void* arg) {
    run_slice* job = (run_slice*)arg;
    for (size_t i = job->begin; i < job->end; ++i) {
        if (orc_rollout(&job->s[i], job->w, &job->out[i]) != 0) {
            job->status = -1;
        }
    }
    return NULL;
}

/* backends.cpp:38-106 -- index-aligned results; partitioning is irrelevant
 * to the bits (each slot is a pure function of its sample). */
int orc_run(const orc_sample* s, size_t n, const orc_world* w, orc_result* out, int threads) {
    if (n == 0) {
        return -1;
    }
    if (threads < 1) threads = 1;
    if ((size_t)threads > n) threads = (int)n;
    run_slice jobs[256];
    pthread_t tid[256];
    if (threads > 256) threads = 256;
    for (int k = 0; k < threads; ++k) {
        jobs[k].s = s;
        jobs[k].w = w;
        jobs[k].out = out;
        jobs[k].begin = n * (size_t)k / (size_t)threads;
        jobs[k].end = n * (size_t)(k + 1) / (size_t)threads;
        jobs[k].status = 0;
    }
    for (int k = 1; k < threads; ++k) pthread_create(&tid[k], NULL, run_slice_main, &jobs[k]);
    run_slice_main(&jobs[0]);
    int status = jobs[0].status;
    for (int k = 1; k < threads; ++k) {
        pthread_join(tid[k], NULL);
        if (jobs[k].status != 0) status = -1;
    }
    return status;
}

/* --------------------------------------------------------------- statistics */

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* analysis.cpp:13-76 -- sequential sum, two-pass m2/m3, full sort, histogram
 * anchored at floor(min) */
int orc_summarize(const orc_result* r, size_t n, double bin_width, orc_summary* out,
                  uint64_t* hist, size_t hist_cap) {
    if (n == 0 || !(bin_width > 0.0)) {
        return -1;
    }
    memset(out, 0, sizeof *out);
    out->n = n;
    double* d = (double*)malloc(n * sizeof(double));
    if (!d) return -1;
    for (size_t i = 0; i < n; ++i) {
        d[i] = r[i].stop_distance;
        if (r[i].hit_horizon) out->horizon_count += 1u;
    }
    const double dn = (double)n;
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) sum += d[i];
    out->mean = sum / dn;
    double m2 = 0.0, m3 = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double dev = d[i] - out->mean;
        m2 += dev * dev;
        m3 += dev * dev * dev;
    }
    out->sd = n > 1 ? sqrt(m2 / (dn - 1.0)) : 0.0;
    const double var_pop = m2 / dn;
    out->skewness = var_pop > 0.0 ? (m3 / dn) / pow(var_pop, 1.5) : 0.0;

    double* sorted = (double*)malloc(n * sizeof(double));
    if (!sorted) {
        free(d);
        return -1;
    }
    memcpy(sorted, d, n * sizeof(double));
    qsort(sorted, n, sizeof(double), cmp_double);
    out->min = sorted[0];
    out->max = sorted[n - 1];
    out->median = (n % 2 == 1) ? sorted[n / 2] : 0.5 * (sorted[n / 2 - 1] + sorted[n / 2]);
    out->right_skewed = out->mean > out->median;
    free(sorted);

    const double lo = floor(out->min);
    const double hi = ceil(out->max);
    size_t bins = (size_t)ceil((hi - lo) / bin_width);
    if (bins < 1) bins = 1;
    out->origin = lo;
    out->bin_width = bin_width;
    out->bins = bins;
    if (hist != NULL) {
        if (hist_cap < bins) {
            free(d);
            return -2;
        }
        memset(hist, 0, bins * sizeof(uint64_t));
        for (size_t i = 0; i < n; ++i) {
            size_t idx = (size_t)((d[i] - lo) / bin_width);
            if (idx >= bins) idx = bins - 1;
            hist[idx] += 1u;
        }
    }
    free(d);
    return 0;
}

/* analysis.cpp:145-159 (numerator only; the caller divides by n) */
uint64_t orc_exceed_count(const orc_result* r, size_t n, double headway) {
    uint64_t c = 0;
    for (size_t i = 0; i < n; ++i) {
        if (r[i].hit_horizon || r[i].stop_distance > headway) c += 1u;
    }
    return c;
}

/* Sensor-noise TTC sweep (the engine's C4 extension; not in the reference):
 * eps_i = sigma * standard_normal_at(seed, first + i) (sampling.cpp:48-53),
 * collision iff hit_horizon || d > (ttc[j] + eps_i) * v.  Plain loops. */
void orc_exceed_ttc_noise(const orc_result* r, size_t n, uint64_t first, uint64_t seed,
                          double sigma, const double* ttc, size_t m, double v, uint64_t* counts) {
    for (size_t j = 0; j < m; ++j) counts[j] = 0;
    for (size_t i = 0; i < n; ++i) {
        if (r[i].hit_horizon) {
            for (size_t j = 0; j < m; ++j) counts[j] += 1u;
            continue;
        }
        const double eps = sigma * orc_standard_normal_at(seed, first + i);
        for (size_t j = 0; j < m; ++j) {
            if (r[i].stop_distance > (ttc[j] + eps) * v) counts[j] += 1u;
        }
    }
}

/* analysis.cpp:161-194 -- nudged rank over the finite stoppers */
int orc_min_safe_headway(const orc_result* r, size_t n, double risk, double* out) {
    if (!(risk > 0.0 && risk < 1.0) || n == 0) {
        return -1;
    }
    double* stopped = (double*)malloc(n * sizeof(double));
    if (!stopped) return -1;
    size_t m = 0;
    for (size_t i = 0; i < n; ++i) {
        if (!r[i].hit_horizon) stopped[m++] = r[i].stop_distance;
    }
    const double raw = (1.0 - risk) * (double)n;
    const size_t rank = (size_t)ceil(raw - raw * 1e-12);
    if (rank > m) {
        *out = INFINITY;
    } else {
        qsort(stopped, m, sizeof(double), cmp_double);
        *out = stopped[rank - 1];
    }
    free(stopped);
    return 0;
}

/* analysis.cpp:230-241 */
long orc_headway_grid(double start, double stop, double step, double* out, size_t cap) {
    if (!(step > 0.0) || !(stop >= start)) {
        return -1;
    }
    const size_t count = (size_t)floor((stop - start) / step + 1e-9);
    if (count + 1 > cap) return -2;
    for (size_t i = 0; i <= count; ++i) out[i] = start + (double)i * step;
    return (long)(count + 1);
}

/* ------------------------------------------------- fine-step independent oracle */

/* tests/oracles.cpp:9-54 -- naive force balance ('/tau', drag recomputed),
 * used only for the known-answer value kNominalFineStopDistance. */
static void naive_rhs(const double st[3], const orc_sample* s, const orc_world* w, double d[3]) {
    const double limit =
        -s->friction * w->gravity / (1.0 + s->friction * w->cg_height / w->wheelbase);
    const double braking = st[2] < limit ? limit : st[2];
    const double drag =
        0.5 * w->air_density * s->drag_coeff * w->frontal_area * st[1] * st[1] / s->mass;
    d[0] = st[1];
    d[1] = braking - drag - w->gravity * sin(s->grade);
    d[2] = (w->brake_cmd - st[2]) / w->actuator_tau;
}

double orc_fine_stopping_distance(const orc_sample* s, const orc_world* w, double dt,
                                  double t_limit) {
    double st[3] = {0.0, s->initial_speed, 0.0};
    const size_t max_steps = (size_t)(t_limit / dt);
    for (size_t i = 0; i < max_steps; ++i) {
        double k1[3], k2[3], k3[3], k4[3], m[3];
        naive_rhs(st, s, w, k1);
        for (int c = 0; c < 3; ++c) m[c] = st[c] + 0.5 * dt * k1[c];
        naive_rhs(m, s, w, k2);
        for (int c = 0; c < 3; ++c) m[c] = st[c] + 0.5 * dt * k2[c];
        naive_rhs(m, s, w, k3);
        for (int c = 0; c < 3; ++c) m[c] = st[c] + dt * k3[c];
        naive_rhs(m, s, w, k4);
        for (int c = 0; c < 3; ++c) {
            st[c] = st[c] + dt / 6.0 * (k1[c] + 2.0 * k2[c] + 2.0 * k3[c] + k4[c]);
        }
        if (st[1] <= 0.0) break;
    }
    return st[0];
}
