"""B200-native Monte Carlo AEB rollout engine (drop-in CUDA executor for the
brakemc reference's run_sequential / run_parallel path).

Compute lives in lib/libbrakemc_b200.so (sm_100a kernels + C-ABI, see
include/brakemc_cuda.h); this package only binds it.
"""
from .engine import (RESULT_DTYPE, SAMPLE_DTYPE, CudaExecutor, RunReport, SimWorld,
                     UncertaintyModel, device_count, device_sampler_available, draw_batch,
                     headway_grid, libm_selftest, stage_terms, ttc_for_headway)
from ._native import BmcError, ConfigError, CudaError, DomainError, LIB_PATH, load

__all__ = [
    "RESULT_DTYPE", "SAMPLE_DTYPE", "CudaExecutor", "RunReport", "SimWorld", "UncertaintyModel",
    "device_count", "device_sampler_available", "draw_batch", "libm_selftest", "headway_grid", "stage_terms", "ttc_for_headway", "BmcError",
    "ConfigError", "CudaError", "DomainError", "LIB_PATH", "load",
]
