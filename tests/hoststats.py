"""Binding of build/libbmc_stats_host.so -- TEST INFRASTRUCTURE.

The host backend of the fused statistics stage (tests/cpp/stats_host.cpp):
the product's own orchestration (csrc/bmc_stats_pipeline.h) and arithmetic
(csrc/bmc_stats_core.h) over host arrays, so merge logic runs on CPU under
gloo, and GPU tests can compare the device stage with it bit for bit.
"""
import ctypes as C
import os

import numpy as np

from paper_2604_27193_b200 import _native as N
from paper_2604_27193_b200.stats import StatsOut, StatsRequest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "build", "libbmc_stats_host.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} missing: make -C tests/cpp stats_host")
        L = C.CDLL(LIB)
        L.bmch_stats_run.restype = C.c_int
        L.bmch_stats_run.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(N.StatsReq),
                                     C.c_uint64, C.POINTER(N.Merge), C.POINTER(N.Stats),
                                     C.c_char_p, C.c_size_t]
        L.bmch_exact_sum.restype = C.c_double
        L.bmch_exact_sum.argtypes = [C.c_void_p, C.c_size_t]
        L.bmch_hist_index_mismatches.restype = C.c_uint64
        L.bmch_hist_index_mismatches.argtypes = [C.c_void_p, C.c_size_t, C.c_double, C.c_double,
                                                 C.c_uint64]
        _lib = L
    return _lib


def exact_sum(v) -> float:
    v = np.ascontiguousarray(v, dtype=np.float64)
    return lib().bmch_exact_sum(C.c_void_p(v.ctypes.data), v.size)


def host_stats(d, hz, req: StatsRequest, merge=None, cand_cap: int = 0, hist_cap: int = 1 << 16):
    d = np.ascontiguousarray(d, dtype=np.float64)
    hz = None if hz is None else np.ascontiguousarray(hz, dtype=np.uint8)
    out = StatsOut(req, hist_cap)
    err = C.create_string_buffer(512)
    rc = lib().bmch_stats_run(C.c_void_p(d.ctypes.data) if d.size else None,
                              C.c_void_p(hz.ctypes.data) if hz is not None and hz.size else None,
                              d.size, C.byref(req.c()), cand_cap,
                              C.byref(merge.struct()) if merge is not None else None,
                              C.byref(out.s), err, 512)
    if merge is not None:
        merge.raise_pending()
    if rc != 0:
        exc = N._ERRORS.get(rc, N.BmcError)(err.value.decode())
        exc.code = rc
        raise exc
    return out.result()


def hist_index_mismatches(v, lo, bw, bins) -> int:
    v = np.ascontiguousarray(v, dtype=np.float64)
    return int(lib().bmch_hist_index_mismatches(C.c_void_p(v.ctypes.data), v.size, lo, bw, bins))
