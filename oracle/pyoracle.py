"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  It loads:

* ``oracle/_ref/libbrakemc_ref.so`` -- the UNMODIFIED reference hot path
  (/root/reference/proj/src, compiled from where it lies by oracle/Makefile)
  behind the forwarding shim ref_shim.cpp;
* ``oracle/_build/libbmc_oracle.so`` -- the C restatement bmc_oracle.c.

Both are built here (``make -C oracle``) and travel to the GPU box as
prebuilt files; nothing here reads /root/reference at run time.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libbrakemc_ref.so")
PORT_LIB = os.path.join(HERE, "_build", "libbmc_oracle.so")

SAMPLE_DTYPE = np.dtype(
    [("initial_speed", "<f8"), ("friction", "<f8"), ("grade", "<f8"), ("mass", "<f8"),
     ("drag_coeff", "<f8")])
RESULT_DTYPE = np.dtype(
    [("stop_distance", "<f8"), ("stop_time", "<f8"), ("steps", "<i8"), ("hit_horizon", "u1"),
     ("pad_", "V7")])
assert SAMPLE_DTYPE.itemsize == 40 and RESULT_DTYPE.itemsize == 32

_D = C.POINTER(C.c_double)
_U64 = C.POINTER(C.c_uint64)


@dataclass
class World:
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

    def as_array(self) -> np.ndarray:
        return np.array([self.dt, self.t_max, self.brake_cmd, self.cg_height, self.wheelbase,
                         self.actuator_tau, self.gravity, self.air_density, self.frontal_area],
                        dtype=np.float64)


@dataclass
class Model:
    """UncertaintyModel (sampling.hpp:24-33); stream order v0, mu, theta, m, c_d."""
    seed: int = 3
    mean: tuple = (30.0, 0.8, 0.0, 1500.0, 0.3)
    sd: tuple = (2.0, 0.1, 0.05, 100.0, 0.05)

    @staticmethod
    def mixed(seed: int = 3) -> "Model":
        """wet/icy friction spread and +-6% grade."""
        import math
        return Model(seed=seed, mean=(30.0, 0.45, 0.0, 1500.0, 0.3),
                     sd=(2.0, 0.20, math.atan(0.06), 100.0, 0.05))


def _ptr(a: np.ndarray, t=C.c_void_p):
    return C.cast(a.ctypes.data, t)


class OracleError(RuntimeError):
    pass


class Reference:
    """The reference library itself (oracle/_ref)."""

    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(path)
        self.lib = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_hardware_concurrency.restype = C.c_uint
        L.ref_stream_word.restype = C.c_uint64
        L.ref_stream_word.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_stream_uniform.restype = C.c_double
        L.ref_stream_uniform.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_standard_normal_at.restype = C.c_double
        L.ref_standard_normal_at.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_draw_batch.argtypes = [C.c_uint64, _D, _D, C.c_size_t, _D, _U64]
        L.ref_rollout_terms.argtypes = [_D, _D, _D]
        L.ref_run.argtypes = [_D, C.c_size_t, _D, C.c_int, C.c_uint, C.c_size_t, C.c_void_p,
                              _D, C.POINTER(C.c_uint)]
        L.ref_simulate_rollout.argtypes = [_D, _D, C.c_void_p]
        L.ref_summarize.argtypes = [C.c_void_p, C.c_size_t, C.c_double, _D, _U64,
                                    C.POINTER(C.c_int), _U64, C.c_size_t, _U64]
        L.ref_collision_probability.argtypes = [C.c_void_p, C.c_size_t, C.c_double, _D]
        L.ref_min_safe_headway.argtypes = [C.c_void_p, C.c_size_t, C.c_double, _D]
        L.ref_build_risk_curve.argtypes = [C.c_void_p, C.c_size_t, _D, C.c_size_t, _D, C.c_size_t,
                                           C.c_double, _D, _D]
        L.ref_headway_grid.restype = C.c_long
        L.ref_headway_grid.argtypes = [C.c_double, C.c_double, C.c_double, _D, C.c_size_t]
        L.ref_convergence_from_results.argtypes = [C.c_void_p, C.c_size_t, _U64, C.c_size_t,
                                                   C.c_size_t, _D]
        L.ref_verify_consistency.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, _D, _U64,
                                             C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_write_results_csv.argtypes = [C.c_void_p, C.c_size_t, C.c_char_p]
        L.ref_read_results_csv.argtypes = [C.c_char_p, C.c_double, C.c_void_p, C.c_size_t,
                                           C.POINTER(C.c_size_t)]
        L.ref_oracle_stopping_distance.restype = C.c_double
        L.ref_oracle_stopping_distance.argtypes = [_D, _D, C.c_double, C.c_double]

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(self.lib.ref_last_error().decode())

    def hardware_concurrency(self) -> int:
        return int(self.lib.ref_hardware_concurrency())

    def stream_word(self, seed, counter):
        return int(self.lib.ref_stream_word(seed, counter))

    def stream_uniform(self, seed, counter):
        return float(self.lib.ref_stream_uniform(seed, counter))

    def standard_normal_at(self, seed, idx):
        return float(self.lib.ref_standard_normal_at(seed, idx))

    def draw_batch(self, model: Model, n: int):
        out = np.zeros(n, dtype=SAMPLE_DTYPE)
        mean = np.array(model.mean, dtype=np.float64)
        sd = np.array(model.sd, dtype=np.float64)
        clamps = C.c_uint64(0)
        self._check(self.lib.ref_draw_batch(model.seed, _ptr(mean, _D), _ptr(sd, _D), n,
                                            _ptr(out, _D), C.byref(clamps)))
        return out, int(clamps.value)

    def rollout_terms(self, sample, world: World):
        s = np.array(list(sample), dtype=np.float64)
        w = world.as_array()
        out = np.zeros(5)
        self._check(self.lib.ref_rollout_terms(_ptr(s, _D), _ptr(w, _D), _ptr(out, _D)))
        return out

    def run(self, samples: np.ndarray, world: World = World(), executor: str = "parallel",
            workers: int = 0, chunk: int = 256):
        samples = np.ascontiguousarray(samples, dtype=SAMPLE_DTYPE)
        n = samples.shape[0]
        out = np.zeros(n, dtype=RESULT_DTYPE)
        w = world.as_array()
        wall = C.c_double(0.0)
        wc = C.c_uint(0)
        self._check(self.lib.ref_run(_ptr(samples, _D), n, _ptr(w, _D),
                                     0 if executor == "sequential" else 1, workers, chunk,
                                     _ptr(out), C.byref(wall), C.byref(wc)))
        return out, float(wall.value), int(wc.value)

    def simulate_rollout(self, sample, world: World = World()):
        s = np.array(list(sample), dtype=np.float64)
        w = world.as_array()
        out = np.zeros(1, dtype=RESULT_DTYPE)
        self._check(self.lib.ref_simulate_rollout(_ptr(s, _D), _ptr(w, _D), _ptr(out)))
        return out[0]

    def summarize(self, results: np.ndarray, bin_width: float = 2.0):
        results = np.ascontiguousarray(results, dtype=RESULT_DTYPE)
        o8 = np.zeros(8)
        hz = C.c_uint64(0)
        rs = C.c_int(0)
        bins = C.c_uint64(0)
        cap = 1 << 20
        hist = np.zeros(cap, dtype=np.uint64)
        self._check(self.lib.ref_summarize(_ptr(results), results.shape[0], bin_width, _ptr(o8, _D),
                                           C.byref(hz), C.byref(rs), _ptr(hist, _U64), cap,
                                           C.byref(bins)))
        keys = ["n", "mean", "sd", "min", "max", "median", "skewness", "origin"]
        out = dict(zip(keys, o8.tolist()))
        out["n"] = int(out["n"])
        out.update(horizon_count=int(hz.value), right_skewed=bool(rs.value),
                   bins=int(bins.value), bin_width=bin_width,
                   histogram=hist[: int(bins.value)].copy())
        return out

    def collision_probability(self, results, headway):
        v = C.c_double(0)
        results = np.ascontiguousarray(results, dtype=RESULT_DTYPE)
        self._check(self.lib.ref_collision_probability(_ptr(results), results.shape[0], headway,
                                                       C.byref(v)))
        return float(v.value)

    def min_safe_headway(self, results, risk):
        v = C.c_double(0)
        results = np.ascontiguousarray(results, dtype=RESULT_DTYPE)
        self._check(self.lib.ref_min_safe_headway(_ptr(results), results.shape[0], risk,
                                                  C.byref(v)))
        return float(v.value)

    def build_risk_curve(self, results, grid, levels, closing_speed):
        results = np.ascontiguousarray(results, dtype=RESULT_DTYPE)
        g = np.ascontiguousarray(grid, dtype=np.float64)
        lv = np.ascontiguousarray(levels, dtype=np.float64)
        probs = np.zeros(len(g))
        thr = np.zeros(3 * len(lv))
        self._check(self.lib.ref_build_risk_curve(_ptr(results), results.shape[0], _ptr(g, _D),
                                                  len(g), _ptr(lv, _D), len(lv), closing_speed,
                                                  _ptr(probs, _D), _ptr(thr, _D)))
        return probs, thr.reshape(-1, 3)

    def headway_grid(self, start, stop, step):
        cap = 1 << 20
        out = np.zeros(cap)
        k = self.lib.ref_headway_grid(start, stop, step, _ptr(out, _D), cap)
        if k < 0:
            raise OracleError(self.lib.ref_last_error().decode())
        return out[:k].copy()

    def convergence_from_results(self, results, n_values, baseline_n):
        results = np.ascontiguousarray(results, dtype=RESULT_DTYPE)
        nv = np.ascontiguousarray(n_values, dtype=np.uint64)
        rows = np.zeros(5 * len(nv))
        self._check(self.lib.ref_convergence_from_results(_ptr(results), results.shape[0],
                                                          _ptr(nv, _U64), len(nv), baseline_n,
                                                          _ptr(rows, _D)))
        return rows.reshape(-1, 5)

    def verify_consistency(self, a, b):
        a = np.ascontiguousarray(a, dtype=RESULT_DTYPE)
        b = np.ascontiguousarray(b, dtype=RESULT_DTYPE)
        dev = C.c_double(0)
        first = C.c_uint64(0)
        bw = C.c_int(0)
        ok = C.c_int(0)
        self._check(self.lib.ref_verify_consistency(_ptr(a), _ptr(b), a.shape[0], C.byref(dev),
                                                    C.byref(first), C.byref(bw), C.byref(ok)))
        return dict(max_abs_deviation=float(dev.value), first_mismatch=int(first.value),
                    bitwise_equal=bool(bw.value), passed=bool(ok.value))

    def write_results_csv(self, results, path: str):
        results = np.ascontiguousarray(results, dtype=RESULT_DTYPE)
        self._check(self.lib.ref_write_results_csv(_ptr(results), results.shape[0], path.encode()))

    def read_results_csv(self, path: str, dt: float):
        n = C.c_size_t(0)
        self._check(self.lib.ref_read_results_csv(path.encode(), dt, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=RESULT_DTYPE)
        self._check(self.lib.ref_read_results_csv(path.encode(), dt, _ptr(out), out.shape[0],
                                                  C.byref(n)))
        return out

    def oracle_stopping_distance(self, sample, world: World = World(), dt=1e-5, t_limit=30.0):
        s = np.array(list(sample), dtype=np.float64)
        w = world.as_array()
        return float(self.lib.ref_oracle_stopping_distance(_ptr(s, _D), _ptr(w, _D), dt, t_limit))


class _OrcWorld(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("dt", "t_max", "brake_cmd", "cg_height", "wheelbase",
                                          "actuator_tau", "gravity", "air_density",
                                          "frontal_area")]


class _OrcModel(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("mean", C.c_double * 5), ("sd", C.c_double * 5)]


class _OrcSummary(C.Structure):
    _fields_ = [("n", C.c_uint64), ("horizon_count", C.c_uint64), ("bins", C.c_uint64),
                ("mean", C.c_double), ("sd", C.c_double), ("min", C.c_double),
                ("max", C.c_double), ("median", C.c_double), ("skewness", C.c_double),
                ("origin", C.c_double), ("bin_width", C.c_double), ("right_skewed", C.c_int)]


def _orc_world(w: World) -> _OrcWorld:
    return _OrcWorld(*w.as_array().tolist())


class Port:
    """The C restatement (oracle/bmc_oracle.c)."""

    def __init__(self, path: str = PORT_LIB):
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: run `make -C oracle oracle`")
        L = C.CDLL(path)
        self.lib = L
        L.orc_stream_word.restype = C.c_uint64
        L.orc_stream_word.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_stream_uniform.restype = C.c_double
        L.orc_stream_uniform.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_standard_normal_at.restype = C.c_double
        L.orc_standard_normal_at.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_draw_range.restype = C.c_uint64
        L.orc_draw_range.argtypes = [C.POINTER(_OrcModel), C.c_uint64, C.c_size_t, C.c_void_p]
        L.orc_rollout_terms.argtypes = [C.c_void_p, C.POINTER(_OrcWorld), _D]
        L.orc_rollout.argtypes = [C.c_void_p, C.POINTER(_OrcWorld), C.c_void_p]
        L.orc_run.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(_OrcWorld), C.c_void_p, C.c_int]
        L.orc_summarize.argtypes = [C.c_void_p, C.c_size_t, C.c_double, C.POINTER(_OrcSummary),
                                    _U64, C.c_size_t]
        L.orc_exceed_count.restype = C.c_uint64
        L.orc_exceed_count.argtypes = [C.c_void_p, C.c_size_t, C.c_double]
        L.orc_min_safe_headway.argtypes = [C.c_void_p, C.c_size_t, C.c_double, _D]
        L.orc_exceed_ttc_noise.restype = None
        L.orc_exceed_ttc_noise.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64, C.c_uint64,
                                           C.c_double, _D, C.c_size_t, C.c_double, _U64]
        L.orc_headway_grid.restype = C.c_long
        L.orc_headway_grid.argtypes = [C.c_double, C.c_double, C.c_double, _D, C.c_size_t]
        L.orc_fine_stopping_distance.restype = C.c_double
        L.orc_fine_stopping_distance.argtypes = [C.c_void_p, C.POINTER(_OrcWorld), C.c_double,
                                                 C.c_double]

    def stream_word(self, seed, counter):
        return int(self.lib.orc_stream_word(seed, counter))

    def stream_uniform(self, seed, counter):
        return float(self.lib.orc_stream_uniform(seed, counter))

    def standard_normal_at(self, seed, idx):
        return float(self.lib.orc_standard_normal_at(seed, idx))

    def draw_range(self, model: Model, first: int, n: int):
        m = _OrcModel(model.seed, (C.c_double * 5)(*model.mean), (C.c_double * 5)(*model.sd))
        out = np.zeros(n, dtype=SAMPLE_DTYPE)
        clamps = self.lib.orc_draw_range(C.byref(m), first, n, _ptr(out))
        return out, int(clamps)

    def rollout_terms(self, sample, world: World = World()):
        s = np.array(list(sample), dtype=np.float64)
        out = np.zeros(5)
        w = _orc_world(world)
        if self.lib.orc_rollout_terms(_ptr(s), C.byref(w), _ptr(out, _D)) != 0:
            raise OracleError("friction_limit: weight-transfer denominator <= 0")
        return out

    def run(self, samples: np.ndarray, world: World = World(), threads: int = 1):
        samples = np.ascontiguousarray(samples, dtype=SAMPLE_DTYPE)
        out = np.zeros(samples.shape[0], dtype=RESULT_DTYPE)
        w = _orc_world(world)
        if self.lib.orc_run(_ptr(samples), samples.shape[0], C.byref(w), _ptr(out), threads) != 0:
            raise OracleError("orc_run failed")
        return out

    def exceed_ttc_noise(self, results, ttc, closing_speed, sigma, noise_seed, first=0):
        """Sensor-noise TTC sweep counts (orc_exceed_ttc_noise)."""
        results = np.ascontiguousarray(results, dtype=RESULT_DTYPE)
        t = np.ascontiguousarray(ttc, dtype=np.float64)
        out = np.zeros(t.shape[0], dtype=np.uint64)
        self.lib.orc_exceed_ttc_noise(_ptr(results), results.shape[0], int(first),
                                      int(noise_seed) & ((1 << 64) - 1), float(sigma),
                                      _ptr(t, _D), t.shape[0], float(closing_speed),
                                      _ptr(out, _U64))
        return out

    def summarize(self, results, bin_width=2.0):
        results = np.ascontiguousarray(results, dtype=RESULT_DTYPE)
        s = _OrcSummary()
        cap = 1 << 20
        hist = np.zeros(cap, dtype=np.uint64)
        rc = self.lib.orc_summarize(_ptr(results), results.shape[0], bin_width, C.byref(s),
                                    _ptr(hist, _U64), cap)
        if rc != 0:
            raise OracleError(f"orc_summarize rc={rc}")
        out = {k: getattr(s, k) for k, _ in _OrcSummary._fields_}
        out["right_skewed"] = bool(out["right_skewed"])
        out["histogram"] = hist[: s.bins].copy()
        return out

    def exceed_count(self, results, headway):
        results = np.ascontiguousarray(results, dtype=RESULT_DTYPE)
        return int(self.lib.orc_exceed_count(_ptr(results), results.shape[0], headway))

    def min_safe_headway(self, results, risk):
        results = np.ascontiguousarray(results, dtype=RESULT_DTYPE)
        v = C.c_double(0)
        if self.lib.orc_min_safe_headway(_ptr(results), results.shape[0], risk, C.byref(v)) != 0:
            raise OracleError("risk.level: must be strictly between 0 and 1")
        return float(v.value)

    def headway_grid(self, start, stop, step):
        cap = 1 << 20
        out = np.zeros(cap)
        k = self.lib.orc_headway_grid(start, stop, step, _ptr(out, _D), cap)
        if k < 0:
            raise OracleError("risk.grid: needs stop >= start and step > 0")
        return out[:k].copy()

    def fine_stopping_distance(self, sample, world: World = World(), dt=1e-5, t_limit=30.0):
        s = np.array(list(sample), dtype=np.float64)
        w = _orc_world(world)
        return float(self.lib.orc_fine_stopping_distance(_ptr(s), C.byref(w), dt, t_limit))


def results_bitwise_equal(a: np.ndarray, b: np.ndarray) -> bool:
    """bitwise_equal_result over every slot (backends.cpp:24-30): all 4 fields."""
    if a.shape != b.shape:
        return False
    return bool(
        np.array_equal(a["stop_distance"].view(np.uint64), b["stop_distance"].view(np.uint64))
        and np.array_equal(a["stop_time"].view(np.uint64), b["stop_time"].view(np.uint64))
        and np.array_equal(a["steps"], b["steps"])
        and np.array_equal(a["hit_horizon"] != 0, b["hit_horizon"] != 0))
