"""Python face of the B200 rollout engine (tests, bench and smoke use it).

The product's host side is C/C++ (the reference is a C++ library): the
executor is ``brakemc::run_cuda`` (include/brakemc/cuda_executor.hpp) over
the C-ABI in include/brakemc_cuda.h.  This module binds the same C-ABI with
ctypes and mirrors the reference API names (/root/reference/proj/include/
brakemc/{sampling,backends,analysis}.hpp) so parity tests read like the
reference's own tests.  Device buffers are torch tensors (plumbing only).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N

SAMPLE_DTYPE = np.dtype(
    [("initial_speed", "<f8"), ("friction", "<f8"), ("grade", "<f8"), ("mass", "<f8"),
     ("drag_coeff", "<f8")])
RESULT_DTYPE = np.dtype(
    [("stop_distance", "<f8"), ("stop_time", "<f8"), ("steps", "<i8"), ("hit_horizon", "u1"),
     ("pad_", "V7")])

# schedule / table modes (bmc_run_opts)
SCHEDULE = {"default": 0, "index": 1, "binned": 2}
TABLE = {"auto": 0, "shared": 1, "global": 2, "none": 3}
# model-driven sampler (bmc_run_opts.sampler)
SAMPLER = {"auto": 0, "host": 1, "device": 2}


@dataclass
class SimWorld:
    """SimConfig + VehicleGeometry + PhysicalConstants (dynamics.hpp:17-60)."""
    dt: float = 0.001
    t_max: float = 10.0
    brake_cmd: float = -6.0
    cg_height: float = 0.5
    wheelbase: float = 2.7
    actuator_tau: float = 0.15
    gravity: float = 9.81
    air_density: float = 1.225
    frontal_area: float = 2.2

    def c(self) -> N.World:
        return N.World(self.dt, self.t_max, self.brake_cmd, self.cg_height, self.wheelbase,
                       self.actuator_tau, self.gravity, self.air_density, self.frontal_area)

    @property
    def max_steps(self) -> int:
        # integrator.cpp:19 -- llround (half away from zero)
        q = self.t_max / self.dt
        return int(math.floor(abs(q) + 0.5)) * (1 if q >= 0 else -1)


@dataclass
class UncertaintyModel:
    """sampling.hpp:24-33; stream order (initial_speed, friction, grade, mass, drag_coeff)."""
    seed: int = 3
    initial_speed: tuple = (30.0, 2.0)
    friction: tuple = (0.8, 0.1)
    grade: tuple = (0.0, 0.05)
    mass: tuple = (1500.0, 100.0)
    drag_coeff: tuple = (0.3, 0.05)

    def c(self) -> N.Model:
        return N.Model(self.seed, N.Normal(*self.initial_speed), N.Normal(*self.friction),
                       N.Normal(*self.grade), N.Normal(*self.mass), N.Normal(*self.drag_coeff))

    @staticmethod
    def mixed(seed: int = 3) -> "UncertaintyModel":
        """C4: wet/icy friction spread, +-6% grade."""
        return UncertaintyModel(seed=seed, friction=(0.45, 0.20), grade=(0.0, math.atan(0.06)))


def _p(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def draw_batch(model: UncertaintyModel, n: int, first: int = 0, threads: int = 0):
    """draw_batch (sampling.cpp:67-100) on the host thread pool; returns
    (samples[n] with SAMPLE_DTYPE, clamp_count).  ``first`` selects the
    shard [first, first+n) of the counter-based stream."""
    lib = N.load()
    out = np.empty(n, dtype=SAMPLE_DTYPE)
    clamps = C.c_uint64(0)
    m = model.c()
    N.check(lib.bmc_draw_range(C.byref(m), first, n, _p(out), C.byref(clamps), threads))
    return out, int(clamps.value)


def stage_terms(samples: np.ndarray, world: SimWorld = SimWorld(), threads: int = 0):
    """RolloutTerms::from (dynamics.cpp:57-68), SoA: (v0, floor, drag, grade)."""
    lib = N.load()
    samples = np.ascontiguousarray(samples, dtype=SAMPLE_DTYPE)
    n = samples.shape[0]
    out = np.empty((4, n), dtype=np.float64)
    w = world.c()
    N.check(lib.bmc_stage_terms(_p(samples), n, C.byref(w), _p(out[0]), _p(out[1]), _p(out[2]),
                                _p(out[3]), threads))
    return out


def write_results_csv(path: str, results: np.ndarray, threads: int = 0) -> None:
    """results.csv (io.cpp:17-31), byte-identical to the reference writer."""
    lib = N.load()
    results = np.ascontiguousarray(results, dtype=RESULT_DTYPE)
    N.check(lib.bmc_write_results_csv(path.encode(), _p(results), results.shape[0], threads))


def read_results_csv(path: str, dt: float) -> np.ndarray:
    """parse_results_csv (io.cpp:94-123) + steps = llround(t/dt) (cli.cpp:96-100)."""
    lib = N.load()
    n = C.c_size_t(0)
    rc = lib.bmc_read_results_csv(path.encode(), dt, None, 0, C.byref(n))
    if rc not in (N.BMC_OK, N.BMC_E_RANGE):
        N.check(rc)
    out = np.zeros(n.value, dtype=RESULT_DTYPE)
    N.check(lib.bmc_read_results_csv(path.encode(), dt, _p(out), out.shape[0], C.byref(n)))
    return out


def libm_selftest(n: int = 1 << 20, seed: int = 12345, threads: int = 0) -> np.ndarray:
    """Compare the glibc port (csrc/bmc_libm.h) with the live host libm; returns
    the 7 mismatch counters (all zero on a matching host, see brakemc_cuda.h)."""
    lib = N.load()
    out = np.zeros(7, dtype=np.uint64)
    lib.bmc_libm_selftest(n, seed, threads, _p(out))
    return out


def device_sampler_available() -> bool:
    lib = N.load()
    v = C.c_int(0)
    N.check(lib.bmc_device_sampler_available(C.byref(v)))
    return bool(v.value)


def device_count() -> int:
    lib = N.load()
    c = C.c_int(0)
    rc = lib.bmc_device_count(C.byref(c))
    return int(c.value) if rc == 0 else 0


@dataclass
class RunReport:
    """ExecutionReport (backends.hpp:25-30) + timing breakdown."""
    results: np.ndarray
    wall_time_s: float
    executor: str = "cuda"
    worker_count: int = 1
    kernel_ms: float = 0.0
    predict_ms: float = 0.0
    total_steps: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    launches: int = 0
    chunks: int = 0


class CudaExecutor:
    """One device context (streams, actuator-table cache, scratch)."""

    def __init__(self, device: int = 0):
        self.lib = N.load()
        self.device = device
        h = C.c_void_p()
        N.check(self.lib.bmc_cuda_init(device, C.byref(h)))
        self.ctx = h

    def close(self):
        if self.ctx:
            self.lib.bmc_cuda_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        N.check(rc, self.ctx)

    @staticmethod
    def _opts(schedule="default", block_threads=0, table="auto", host_threads=0, chunk=0, ilp=0,
              sampler="auto", test_block=0):
        return N.RunOpts(SCHEDULE[schedule], block_threads, TABLE[table], host_threads, chunk,
                         ilp, SAMPLER[sampler], test_block)

    # -------------------------------------------------------------- executor
    def run(self, samples: np.ndarray, world: SimWorld = SimWorld(), out: np.ndarray = None,
            **opts) -> RunReport:
        """run_cuda: host AoS samples -> host AoS results (bit-identical to
        run_sequential, backends.cpp:38-55).  Synchronous."""
        samples = np.ascontiguousarray(samples, dtype=SAMPLE_DTYPE)
        n = samples.shape[0]
        if out is None:
            out = np.empty(n, dtype=RESULT_DTYPE)
        w = world.c()
        o = self._opts(**opts)
        info = N.RunInfo()
        self._check(self.lib.bmc_cuda_run(self.ctx, _p(samples), n, C.byref(w), C.byref(o),
                                          _p(out), C.byref(info)))
        return RunReport(out, info.wall_s, "cuda", 1, info.kernel_ms, info.predict_ms,
                         int(info.total_steps), int(info.h2d_bytes), int(info.d2h_bytes),
                         int(info.launches), int(info.chunks))

    def run_model(self, model: UncertaintyModel, n: int, first: int = 0,
                  world: SimWorld = SimWorld(), out: np.ndarray = None, device_out=None,
                  stats=None, **opts):
        """Streaming executor: draw samples [first, first+n) of ``model`` on the
        host pool straight into pinned SoA terms, overlapped with the GPU.
        Results go to a host AoS array (``out``/default) or, when
        ``device_out=(d f64, steps i32, hz u8)`` CUDA tensors are given, stay on
        the device (stats-only mode; ``stats``: a begun StatsStage whose pass 1
        is fused into every chunk's rollout).  Returns (RunReport, clamp_count)."""
        w = world.c()
        o = self._opts(**opts)
        info = N.RunInfo()
        clamps = C.c_uint64(0)
        m = model.c()
        if device_out is not None:
            outs = N.Outputs(*[int(x.data_ptr()) if x is not None else None for x in device_out])
            self._check(self.lib.bmc_cuda_run_model_stats(
                self.ctx, C.byref(m), first, n, C.byref(w), C.byref(o), None, C.byref(outs),
                C.byref(clamps), C.byref(info), stats.h if stats is not None else None))
            res = None
        else:
            if out is None:
                out = np.empty(n, dtype=RESULT_DTYPE)
            self._check(self.lib.bmc_cuda_run_model(self.ctx, C.byref(m), first, n, C.byref(w),
                                                    C.byref(o), _p(out), None, C.byref(clamps),
                                                    C.byref(info)))
            res = out
        rep = RunReport(res, info.wall_s, "cuda", 1, info.kernel_ms, info.predict_ms,
                        int(info.total_steps), int(info.h2d_bytes), int(info.d2h_bytes),
                        int(info.launches), int(info.chunks))
        return rep, int(clamps.value)

    def draw_device(self, model: UncertaintyModel, n: int, first: int = 0,
                    world: SimWorld = SimWorld(), terms: bool = True, samples: bool = True):
        """On-device draw_batch (sampling.cpp:67-100) + RolloutTerms::from
        (dynamics.cpp:57-68) through the glibc port: returns (terms, samples,
        clamp_count) with terms a (4, n) float64 CUDA tensor [v0, floor, drag,
        grade] and samples an (n, 5) float64 CUDA tensor (ScenarioSample
        field order), each None when not requested."""
        import torch
        dev = torch.device("cuda", self.device)
        t = torch.empty((4, n), dtype=torch.float64, device=dev) if terms else None
        smp = torch.empty((n, 5), dtype=torch.float64, device=dev) if samples else None
        w = world.c()
        m = model.c()
        clamps = C.c_uint64(0)
        self._check(self.lib.bmc_cuda_draw_device(
            self.ctx, C.byref(m), first, n, C.byref(w),
            C.c_void_p(t.data_ptr()) if t is not None else None,
            C.c_void_p(smp.data_ptr()) if smp is not None else None, C.byref(clamps)))
        return t, smp, int(clamps.value)

    def graph(self, n: int, world: SimWorld = SimWorld(), stats=None, **opts) -> "DecisionGraph":
        """Capture the real-time decision batch of size n as a CUDA graph;
        ``stats`` (a StatsRequest) adds the fused statistics stage."""
        return DecisionGraph(self, n, world, stats=stats, **opts)

    def rollout_device(self, terms, outputs, world: SimWorld = SimWorld(), total_steps=None,
                       stream=None, stats=None, **opts) -> None:
        """Device-resident rollout. terms: 4 float64 CUDA tensors (v0, floor,
        drag, grade); outputs: (stop_distance f64, steps i32, hit_horizon u8)
        CUDA tensors or None.  Enqueued on ``stream`` (torch stream or None).
        ``stats``: a begun StatsStage whose pass 1 is fused into the rollout
        epilogue (bmc_cuda_rollout_stats)."""
        n = int(terms[0].numel())
        t = N.Terms(*[int(x.data_ptr()) for x in terms])
        o = N.Outputs(*[int(x.data_ptr()) if x is not None else None for x in outputs])
        w = world.c()
        op = self._opts(**opts)
        ts = C.c_void_p(int(total_steps.data_ptr())) if total_steps is not None else None
        st = C.c_void_p(int(stream.cuda_stream)) if stream is not None else None
        self._check(self.lib.bmc_cuda_rollout_stats(self.ctx, C.byref(t), n, C.byref(w),
                                                    C.byref(op), C.byref(o), ts,
                                                    stats.h if stats is not None else None, st))

    # ------------------------------------------------- fused statistics stage
    def stats_stage(self, max_n: int, headways=(), risk_levels=(), summarize=False,
                    bin_width=2.0, hist_cap=0, cand_cap=0):
        """A device statistics stage (bmc_stats_create) for up to max_n results."""
        from .stats import StatsRequest, StatsStage
        return StatsStage(self, StatsRequest(headways, risk_levels, summarize, bin_width, hist_cap,
                                             cand_cap), max_n)

    def stats(self, d, hz, headways=(), risk_levels=(), summarize=False, bin_width=2.0,
              hist_cap=0, cand_cap=0) -> dict:
        """analysis.cpp over device outputs in one call (bmc_cuda_stats)."""
        from .stats import StatsRequest, stats
        return stats(self, d, hz, StatsRequest(headways, risk_levels, summarize, bin_width,
                                               hist_cap, cand_cap))

    def last_kernel_ms(self):
        r, p = C.c_float(0), C.c_float(0)
        self._check(self.lib.bmc_cuda_last_kernel_ms(self.ctx, C.byref(r), C.byref(p)))
        return float(r.value), float(p.value)

    def last_stage_ms(self):
        """(binning, rollout, unpermute) device ms of the last device-resident rollout."""
        b, r, u = C.c_float(0), C.c_float(0), C.c_float(0)
        self._check(self.lib.bmc_cuda_last_stage_ms(self.ctx, C.byref(b), C.byref(r), C.byref(u)))
        return float(b.value), float(r.value), float(u.value)

    def lane_efficiency(self):
        """(executed steps, lane slots, efficiency) of the last rollout launch."""
        a, b = C.c_uint64(0), C.c_uint64(0)
        self._check(self.lib.bmc_cuda_last_lane_stats(self.ctx, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value), (a.value / b.value if b.value else 0.0)

    def last_launches(self) -> int:
        v = C.c_uint32(0)
        self._check(self.lib.bmc_cuda_last_launches(self.ctx, C.byref(v)))
        return int(v.value)

    def sync(self):
        self._check(self.lib.bmc_cuda_sync(self.ctx))

    def fp64_peak(self, reps: int = 5):
        """Measured FP64 DADD/DMUL op rate (ops/s) and the best probe time (ms)."""
        ops, ms = C.c_double(0), C.c_double(0)
        self._check(self.lib.bmc_cuda_fp64_peak(self.ctx, reps, C.byref(ops), C.byref(ms)))
        return float(ops.value), float(ms.value)

    @property
    def stream_handle(self) -> int:
        return int(self.lib.bmc_cuda_stream(self.ctx) or 0)

    # ------------------------------------------------------------ statistics
    def summarize(self, d, hz, bin_width: float = 2.0, hist_cap: int = 1 << 16):
        """summarize (analysis.cpp:13-76) over device outputs."""
        n = int(d.numel())
        s = N.Summary()
        hist = np.zeros(hist_cap, dtype=np.uint64)
        self._check(self.lib.bmc_cuda_summarize(self.ctx, C.c_void_p(d.data_ptr()),
                                                C.c_void_p(hz.data_ptr()) if hz is not None else None,
                                                n, bin_width, C.byref(s), _p(hist), hist_cap))
        out = {k: getattr(s, k) for k, _ in N.Summary._fields_ if k != "pad_"}
        out["right_skewed"] = bool(out["right_skewed"])
        out["histogram"] = hist[: s.bins].copy()
        return out

    def exceedance_counts(self, d, hz, headways: Sequence[float]) -> np.ndarray:
        """#{hit_horizon or d > h} per headway (analysis.cpp:145-159 numerators)."""
        n = int(d.numel())
        h = np.ascontiguousarray(headways, dtype=np.float64)
        counts = np.zeros(h.shape[0], dtype=np.uint64)
        self._check(self.lib.bmc_cuda_exceedance(self.ctx, C.c_void_p(d.data_ptr()),
                                                 C.c_void_p(hz.data_ptr()) if hz is not None else None,
                                                 n, _p(h), h.shape[0], _p(counts)))
        return counts

    def exceedance_ttc_noise(self, d, hz, ttc: Sequence[float], closing_speed: float,
                             sigma: float, noise_seed: int, first: int = 0) -> np.ndarray:
        """Sensor-noise TTC sweep: #{hit_horizon or d > (T + eps_i) * v} per
        threshold T, eps_i = sigma * standard_normal_at(noise_seed, first + i)."""
        n = int(d.numel())
        t = np.ascontiguousarray(ttc, dtype=np.float64)
        counts = np.zeros(t.shape[0], dtype=np.uint64)
        self._check(self.lib.bmc_cuda_exceedance_ttc_noise(
            self.ctx, C.c_void_p(d.data_ptr()),
            C.c_void_p(hz.data_ptr()) if hz is not None else None, n, int(first),
            int(noise_seed) & ((1 << 64) - 1), float(sigma), _p(t), t.shape[0],
            float(closing_speed), _p(counts)))
        return counts

    def order_stats(self, d, hz, ranks: Sequence[int], exclude_horizon: bool):
        n = int(d.numel())
        r = np.ascontiguousarray(ranks, dtype=np.uint64)
        out = np.zeros(r.shape[0], dtype=np.float64)
        cnt = C.c_uint64(0)
        self._check(self.lib.bmc_cuda_order_stats(self.ctx, C.c_void_p(d.data_ptr()),
                                                  C.c_void_p(hz.data_ptr()) if hz is not None else None,
                                                  n, 1 if exclude_horizon else 0, _p(r), r.shape[0],
                                                  _p(out), C.byref(cnt)))
        return out, int(cnt.value)

    # mergeable building blocks (distributed.py) -------------------------
    def partials(self, d, hz):
        p = N.Partials()
        self._check(self.lib.bmc_cuda_partials(self.ctx, C.c_void_p(d.data_ptr()),
                                               C.c_void_p(hz.data_ptr()) if hz is not None else None,
                                               int(d.numel()), C.byref(p)))
        return {k: getattr(p, k) for k, _ in N.Partials._fields_ if k != "pad_"}

    def moments(self, d, mean: float):
        out = np.zeros(4)
        self._check(self.lib.bmc_cuda_moments(self.ctx, C.c_void_p(d.data_ptr()), int(d.numel()),
                                              mean, _p(out)))
        return tuple(float(x) for x in out)

    def histogram(self, d, origin: float, bin_width: float, bins: int) -> np.ndarray:
        out = np.zeros(bins, dtype=np.uint64)
        self._check(self.lib.bmc_cuda_histogram(self.ctx, C.c_void_p(d.data_ptr()), int(d.numel()),
                                                origin, bin_width, bins, _p(out)))
        return out

    def select_pass(self, d, hz, exclude_horizon: bool, shift: int, prefixes) -> np.ndarray:
        pre = np.ascontiguousarray(prefixes, dtype=np.uint64)
        out = np.zeros((pre.shape[0], 256), dtype=np.uint64)
        self._check(self.lib.bmc_cuda_select_pass(
            self.ctx, C.c_void_p(d.data_ptr()),
            C.c_void_p(hz.data_ptr()) if hz is not None else None, int(d.numel()),
            1 if exclude_horizon else 0, shift, _p(pre), pre.shape[0], _p(out)))
        return out

    def collision_probability(self, d, hz, headway: float) -> float:
        if not headway >= 0.0:
            raise N.ConfigError("risk.headway: must be >= 0")
        c = self.exceedance_counts(d, hz, [headway])
        return float(c[0]) / float(d.numel())

    def min_safe_headway(self, d, hz, risk: float) -> float:
        """analysis.cpp:161-194: nudged rank, order statistic among stoppers."""
        return self.min_safe_headways(d, hz, [risk])[0]

    def min_safe_headways(self, d, hz, risks: Sequence[float]):
        """min_safe_headway per level through the fused statistics stage
        (level-1 buckets, compaction, exact selection; 16 levels a call)."""
        n = int(d.numel())
        if n == 0:
            raise N.ConfigError("risk: needs at least one result")
        for risk in risks:
            if not (0.0 < risk < 1.0):
                raise N.ConfigError("risk.level: must be strictly between 0 and 1")
        out = []
        risks = list(risks)
        for k0 in range(0, len(risks), 16):
            out += [float(v) for v in self.stats(d, hz, risk_levels=risks[k0:k0 + 16])
                    ["min_safe_headway"]]
        return out

    def build_risk_curve(self, d, hz, grid: Sequence[float], risk_levels: Sequence[float],
                         closing_speed: float):
        """build_risk_curve (analysis.cpp:203-228): the whole grid's
        exceedance counts and every threshold from one statistics stage
        (the reference rescans the results once per grid point)."""
        n = float(d.numel())
        levels = sorted(risk_levels, reverse=True)
        if len(levels) <= 16:
            out = self.stats(d, hz, headways=grid, risk_levels=levels)
            counts, heads = out["exceed"], [float(v) for v in out["min_safe_headway"]]
        else:
            counts = self.exceedance_counts(d, hz, grid)
            heads = self.min_safe_headways(d, hz, levels)
        probs = counts.astype(np.float64) / n
        g = list(grid)
        for i in range(1, len(g)):
            if g[i] >= g[i - 1] and probs[i] > probs[i - 1]:
                raise AssertionError("risk curve must be non-increasing in headway")
        thr = [(r, h, ttc_for_headway(h, closing_speed)) for r, h in zip(levels, heads)]
        return probs, thr


class DecisionGraph:
    """Real-time mode (C2): fixed-size decision batch replayed as a CUDA graph."""

    def __init__(self, ex: CudaExecutor, n: int, world: SimWorld = SimWorld(), stats=None,
                 **opts):
        self.ex = ex
        self.n = n
        self.req = stats
        w = world.c()
        o = ex._opts(**opts)
        h = C.c_void_p()
        if stats is not None:
            ex._check(ex.lib.bmc_cuda_graph_create_stats(ex.ctx, n, C.byref(w), C.byref(o),
                                                         C.byref(stats.c()), C.byref(h)))
        else:
            ex._check(ex.lib.bmc_cuda_graph_create(ex.ctx, n, C.byref(w), C.byref(o),
                                                   C.byref(h)))
        self.g = h
        self.out = np.empty(n, dtype=RESULT_DTYPE)
        if stats is not None:
            from .stats import StatsOut
            self._sout = StatsOut(stats)

    def stats(self) -> dict:
        """Statistics of the last decision (P(collision) per headway, ...)."""
        self.ex._check(self.ex.lib.bmc_cuda_graph_stats(self.g, C.byref(self._sout.s)))
        return self._sout.result()

    def run(self, samples: np.ndarray) -> RunReport:
        samples = np.ascontiguousarray(samples, dtype=SAMPLE_DTYPE)
        if samples.shape[0] != self.n:
            raise N.ConfigError(f"batch: graph captured for {self.n} samples")
        info = N.RunInfo()
        self.ex._check(self.ex.lib.bmc_cuda_graph_run(self.g, _p(samples), _p(self.out),
                                                      C.byref(info)))
        return RunReport(self.out, info.wall_s, "cuda-graph", 1, total_steps=int(info.total_steps),
                         h2d_bytes=int(info.h2d_bytes), d2h_bytes=int(info.d2h_bytes),
                         launches=int(info.launches), chunks=1)

    def run_model(self, model: UncertaintyModel, first: int = 0) -> RunReport:
        info = N.RunInfo()
        clamps = C.c_uint64(0)
        m = model.c()
        self.ex._check(self.ex.lib.bmc_cuda_graph_run_model(self.g, C.byref(m), first,
                                                            _p(self.out), C.byref(clamps),
                                                            C.byref(info)))
        return RunReport(self.out, info.wall_s, "cuda-graph", 1, total_steps=int(info.total_steps),
                         h2d_bytes=int(info.h2d_bytes), d2h_bytes=int(info.d2h_bytes),
                         launches=int(info.launches), chunks=1)

    def close(self):
        if self.g:
            self.ex.lib.bmc_cuda_graph_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def max_feasible_n(timed_run_s, budget_s: float, search_start: int, search_cap: int):
    """Doubling + bisection search (analysis.cpp:258-318, same control flow):
    largest n with timed_run_s(n) <= budget_s.  Returns (n, capped)."""
    if not budget_s > 0.0:
        raise N.ConfigError("budget: must be > 0")
    if search_start == 0 or search_cap == 0:
        raise N.ConfigError("feasibility.search: start and cap must be >= 1")
    probe = min(search_start, search_cap)
    lo = hi = 0
    if timed_run_s(probe) <= budget_s:
        lo = probe
        while lo < search_cap:
            nxt = min(search_cap, lo * 2)
            if timed_run_s(nxt) <= budget_s:
                lo = nxt
            else:
                hi = nxt
                break
        if hi == 0:
            return lo, True
    else:
        hi = probe
        down = probe // 2
        while down >= 1:
            if timed_run_s(down) <= budget_s:
                lo = down
                break
            hi = down
            down //= 2
        if lo == 0:
            return 0, False
    while hi - lo > max(1, lo // 64):
        mid = lo + (hi - lo) // 2
        if timed_run_s(mid) <= budget_s:
            lo = mid
        else:
            hi = mid
    return lo, False


def median_wall_time_s(fn, reps: int = 5, warmup: int = 1) -> float:
    """backends.cpp:161-181 -- median of reps after warm-up, monotonic clock."""
    import time
    if reps < 1:
        raise N.ConfigError("timing.reps: must be >= 1")
    for _ in range(warmup):
        fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    ts.sort()
    mid = len(ts) // 2
    return ts[mid] if len(ts) % 2 else 0.5 * (ts[mid - 1] + ts[mid])


def ttc_for_headway(headway_m: float, closing_speed_mps: float) -> float:
    """analysis.cpp:196-201"""
    if not closing_speed_mps > 0.0:
        raise N.ConfigError("risk.closing_speed: must be > 0")
    return headway_m / closing_speed_mps


def headway_grid(start: float, stop: float, step: float):
    """analysis.cpp:230-241"""
    if not (step > 0.0) or not (stop >= start):
        raise N.ConfigError("risk.grid: needs stop >= start and step > 0")
    count = int(math.floor((stop - start) / step + 1e-9))
    return [start + float(i) * step for i in range(count + 1)]
