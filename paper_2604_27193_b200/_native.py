"""ctypes binding of the C-ABI in include/brakemc_cuda.h (libbrakemc_b200.so).

The library is built in-tree (paper_2604_27193_b200/csrc/Makefile) and is
the only compute path: there is no Python or CPU fallback.  Loading fails
loudly when the .so is missing, and every compute entry point raises
``CudaError`` when no sm_100 device is usable.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# BMC_LIB_PATH: an A/B build of the same library (tools/ab_build.sh)
LIB_PATH = os.environ.get("BMC_LIB_PATH") or os.path.join(PKG, "lib", "libbrakemc_b200.so")

BMC_OK, BMC_E_CONFIG, BMC_E_DOMAIN, BMC_E_CUDA, BMC_E_NOMEM, BMC_E_RANGE, BMC_E_IO = (
    0, -1, -2, -3, -4, -5, -6)


class BmcError(RuntimeError):
    code = 0


class ConfigError(BmcError, ValueError):
    """brakemc::ConfigError analogue: message starts with the field path."""
    code = BMC_E_CONFIG


class DomainError(BmcError, ArithmeticError):
    """std::domain_error from friction_limit (dynamics.cpp:48-55)."""
    code = BMC_E_DOMAIN


class CudaError(BmcError):
    code = BMC_E_CUDA


class IoError(BmcError, OSError):
    """brakemc::IoError analogue (errors.hpp:22-25)."""
    code = BMC_E_IO


_ERRORS = {BMC_E_CONFIG: ConfigError, BMC_E_DOMAIN: DomainError, BMC_E_CUDA: CudaError,
           BMC_E_IO: IoError}


class Sample(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("initial_speed", "friction", "grade", "mass",
                                          "drag_coeff")]


class Result(C.Structure):
    _fields_ = [("stop_distance", C.c_double), ("stop_time", C.c_double), ("steps", C.c_int64),
                ("hit_horizon", C.c_uint8), ("pad_", C.c_uint8 * 7)]


class World(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("dt", "t_max", "brake_cmd", "cg_height", "wheelbase",
                                          "actuator_tau", "gravity", "air_density",
                                          "frontal_area")]


class Normal(C.Structure):
    _fields_ = [("mean", C.c_double), ("sd", C.c_double)]


class Model(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("initial_speed", Normal), ("friction", Normal),
                ("grade", Normal), ("mass", Normal), ("drag_coeff", Normal)]


class Terms(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("initial_speed", "brake_floor", "drag_factor",
                                          "grade_accel")]


class Outputs(C.Structure):
    _fields_ = [("stop_distance", C.c_void_p), ("steps", C.c_void_p), ("hit_horizon", C.c_void_p)]


class RunOpts(C.Structure):
    _fields_ = [("schedule", C.c_int32), ("block_threads", C.c_int32), ("table_mode", C.c_int32),
                ("host_threads", C.c_int32), ("chunk_samples", C.c_uint64), ("ilp", C.c_int32),
                ("sampler", C.c_int32), ("test_block", C.c_int32)]


class RunInfo(C.Structure):
    _fields_ = [("wall_s", C.c_double), ("kernel_ms", C.c_double), ("predict_ms", C.c_double),
                ("total_steps", C.c_uint64), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("launches", C.c_uint32), ("chunks", C.c_uint32)]


class Summary(C.Structure):
    _fields_ = [("n", C.c_uint64), ("horizon_count", C.c_uint64), ("bins", C.c_uint64),
                ("mean", C.c_double), ("sd", C.c_double), ("min", C.c_double),
                ("max", C.c_double), ("median", C.c_double), ("skewness", C.c_double),
                ("origin", C.c_double), ("bin_width", C.c_double), ("right_skewed", C.c_int32),
                ("pad_", C.c_int32)]


class Partials(C.Structure):
    _fields_ = [("count", C.c_uint64), ("horizon_count", C.c_uint64), ("min", C.c_double),
                ("max", C.c_double), ("sum_hi", C.c_double), ("sum_lo", C.c_double),
                ("any_nan", C.c_int32), ("pad_", C.c_int32)]


class StatsReq(C.Structure):
    _fields_ = [("headways", C.c_void_p), ("n_headways", C.c_size_t), ("risk_levels", C.c_void_p),
                ("n_risk", C.c_size_t), ("summarize", C.c_int32), ("pad_", C.c_int32),
                ("bin_width", C.c_double), ("hist_cap", C.c_uint64), ("cand_cap", C.c_uint64)]


class Stats(C.Structure):
    _fields_ = [("n", C.c_uint64), ("horizon_count", C.c_uint64), ("summary", Summary),
                ("exceed", C.c_void_p), ("min_safe_headway", C.c_void_p),
                ("histogram", C.c_void_p), ("histogram_cap", C.c_size_t),
                ("launches", C.c_uint32), ("fallbacks", C.c_uint32)]


# bmc_merge: collective hooks of the statistics stage (device buffers, stream-ordered)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
MERGE_SUM, MERGE_MIN, MERGE_MAX = 0, 1, 2


class Merge(C.Structure):
    _fields_ = [("user", C.c_void_p), ("world", C.c_int32), ("rank", C.c_int32),
                ("allreduce_u64", ALLREDUCE_FN), ("allgather_u64", ALLGATHER_FN)]


assert C.sizeof(Sample) == 40 and C.sizeof(Result) == 32 and C.sizeof(Model) == 88

# (name, restype, argtypes) for every entry point declared in brakemc_cuda.h
_P = C.c_void_p
SIGNATURES = [
    ("bmc_abi_version", C.c_int, []),
    ("bmc_last_error", C.c_char_p, []),
    ("bmc_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("bmc_cuda_init", C.c_int, [C.c_int, C.POINTER(_P)]),
    ("bmc_cuda_destroy", None, [_P]),
    ("bmc_cuda_last_error", C.c_char_p, [_P]),
    ("bmc_cuda_sync", C.c_int, [_P]),
    ("bmc_cuda_stream", _P, [_P]),
    ("bmc_draw_range", C.c_int, [C.POINTER(Model), C.c_uint64, C.c_size_t, _P,
                                 C.POINTER(C.c_uint64), C.c_int]),
    ("bmc_stage_terms", C.c_int, [_P, C.c_size_t, C.POINTER(World), _P, _P, _P, _P, C.c_int]),
    ("bmc_libm_selftest", C.c_int, [C.c_uint64, C.c_uint64, C.c_int, _P]),
    ("bmc_device_sampler_available", C.c_int, [C.POINTER(C.c_int)]),
    ("bmc_cuda_draw_device", C.c_int, [_P, C.POINTER(Model), C.c_uint64, C.c_size_t,
                                       C.POINTER(World), _P, _P, C.POINTER(C.c_uint64)]),
    ("bmc_write_results_csv", C.c_int, [C.c_char_p, _P, C.c_size_t, C.c_int]),
    ("bmc_read_results_csv", C.c_int, [C.c_char_p, C.c_double, _P, C.c_size_t,
                                       C.POINTER(C.c_size_t)]),
    ("bmc_cuda_run", C.c_int, [_P, _P, C.c_size_t, C.POINTER(World), C.POINTER(RunOpts), _P,
                               C.POINTER(RunInfo)]),
    ("bmc_cuda_run_model", C.c_int, [_P, C.POINTER(Model), C.c_uint64, C.c_size_t,
                                     C.POINTER(World), C.POINTER(RunOpts), _P,
                                     C.POINTER(Outputs), C.POINTER(C.c_uint64),
                                     C.POINTER(RunInfo)]),
    ("bmc_cuda_graph_create", C.c_int, [_P, C.c_size_t, C.POINTER(World), C.POINTER(RunOpts),
                                        C.POINTER(_P)]),
    ("bmc_cuda_graph_run", C.c_int, [_P, _P, _P, C.POINTER(RunInfo)]),
    ("bmc_cuda_graph_run_model", C.c_int, [_P, C.POINTER(Model), C.c_uint64, _P,
                                           C.POINTER(C.c_uint64), C.POINTER(RunInfo)]),
    ("bmc_cuda_graph_destroy", None, [_P]),
    ("bmc_cuda_rollout_device", C.c_int, [_P, C.POINTER(Terms), C.c_size_t, C.POINTER(World),
                                          C.POINTER(RunOpts), C.POINTER(Outputs), _P, _P]),
    ("bmc_cuda_last_kernel_ms", C.c_int, [_P, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    ("bmc_cuda_last_stage_ms", C.c_int, [_P, C.POINTER(C.c_float), C.POINTER(C.c_float),
                                         C.POINTER(C.c_float)]),
    ("bmc_cuda_last_launches", C.c_int, [_P, C.POINTER(C.c_uint32)]),
    ("bmc_cuda_last_lane_stats", C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("bmc_cuda_summarize", C.c_int, [_P, _P, _P, C.c_size_t, C.c_double, C.POINTER(Summary), _P,
                                     C.c_size_t]),
    ("bmc_cuda_exceedance", C.c_int, [_P, _P, _P, C.c_size_t, _P, C.c_size_t, _P]),
    ("bmc_cuda_exceedance_ttc_noise", C.c_int, [_P, _P, _P, C.c_size_t, C.c_uint64, C.c_uint64,
                                                C.c_double, _P, C.c_size_t, C.c_double, _P]),
    ("bmc_cuda_order_stats", C.c_int, [_P, _P, _P, C.c_size_t, C.c_int, _P, C.c_size_t, _P,
                                       C.POINTER(C.c_uint64)]),
    ("bmc_cuda_fp64_peak", C.c_int, [_P, C.c_int, C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]),
    ("bmc_cuda_alloc", C.c_int, [_P, C.c_size_t, C.POINTER(_P)]),
    ("bmc_cuda_free", C.c_int, [_P, _P]),
    ("bmc_cuda_copy_to_host", C.c_int, [_P, _P, _P, C.c_size_t]),
    ("bmc_cuda_copy_to_device", C.c_int, [_P, _P, _P, C.c_size_t]),
    ("bmc_cuda_partials", C.c_int, [_P, _P, _P, C.c_size_t, C.POINTER(Partials)]),
    ("bmc_cuda_moments", C.c_int, [_P, _P, C.c_size_t, C.c_double, _P]),
    ("bmc_cuda_histogram", C.c_int, [_P, _P, C.c_size_t, C.c_double, C.c_double, C.c_uint64,
                                     _P]),
    ("bmc_cuda_select_pass", C.c_int, [_P, _P, _P, C.c_size_t, C.c_int, C.c_int, _P,
                                       C.c_size_t, _P]),
    ("bmc_stats_create", C.c_int, [_P, C.POINTER(StatsReq), C.c_size_t, C.POINTER(_P)]),
    ("bmc_stats_destroy", None, [_P]),
    ("bmc_stats_begin", C.c_int, [_P, _P]),
    ("bmc_stats_accumulate", C.c_int, [_P, _P, _P, C.c_size_t, _P]),
    ("bmc_stats_finish", C.c_int, [_P, _P, _P, C.c_size_t, C.POINTER(Merge), C.POINTER(Stats),
                                   _P]),
    ("bmc_cuda_rollout_stats", C.c_int, [_P, C.POINTER(Terms), C.c_size_t, C.POINTER(World),
                                         C.POINTER(RunOpts), C.POINTER(Outputs), _P, _P, _P]),
    ("bmc_cuda_stats", C.c_int, [_P, _P, _P, C.c_size_t, C.POINTER(StatsReq), C.POINTER(Stats)]),
    ("bmc_cuda_run_model_stats", C.c_int, [_P, C.POINTER(Model), C.c_uint64, C.c_size_t,
                                           C.POINTER(World), C.POINTER(RunOpts), _P,
                                           C.POINTER(Outputs), C.POINTER(C.c_uint64),
                                           C.POINTER(RunInfo), _P]),
    ("bmc_cuda_graph_create_stats", C.c_int, [_P, C.c_size_t, C.POINTER(World),
                                              C.POINTER(RunOpts), C.POINTER(StatsReq),
                                              C.POINTER(_P)]),
    ("bmc_cuda_graph_stats", C.c_int, [_P, C.POINTER(Stats)]),
    ("bmc_nccl_available", C.c_int, [C.POINTER(C.c_int)]),
    ("bmc_nccl_init_all", C.c_int, [C.c_int, _P, _P]),
    ("bmc_nccl_merge", C.POINTER(Merge), [_P]),
    ("bmc_nccl_destroy", None, [_P]),
]

_lib = None


def load() -> C.CDLL:
    """Load libbrakemc_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (or make -C paper_2604_27193_b200/csrc). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, ctx=None) -> None:
    if rc == BMC_OK:
        return
    lib = load()
    msg = (lib.bmc_cuda_last_error(ctx) if ctx else lib.bmc_last_error()) or b""
    if not msg and ctx:
        msg = lib.bmc_last_error() or b""
    err = _ERRORS.get(rc, BmcError)(msg.decode() or f"bmc error {rc}")
    err.code = rc
    raise err
