"""The fused statistics stage (brakemc_cuda.h ``bmc_stats_*``) from Python.

One request describes what analysis.cpp should be computed over a batch of
rollout outputs (/root/reference/proj/src/analysis.cpp):

* ``headways``: collision_probability numerators, one per headway (the
  build_risk_curve grid, :145-159 / :203-228);
* ``risk_levels``: min_safe_headway per level (:161-194);
* ``summarize`` + ``bin_width``: the DistributionSummary (:13-76).

The device pipeline fuses pass 1 into the rollout epilogue
(``CudaExecutor.rollout_device(..., stats=stage)``); ``finish`` runs the rest
and returns plain Python values.  ``merge`` (distributed.TorchMerge) turns a
rank's stage into the merged statistics of every rank's shard.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N


@dataclass
class StatsRequest:
    headways: Sequence[float] = ()
    risk_levels: Sequence[float] = ()
    summarize: bool = False
    bin_width: float = 2.0
    hist_cap: int = 0
    cand_cap: int = 0
    _keep: list = field(default_factory=list, repr=False)

    def c(self) -> N.StatsReq:
        h = np.ascontiguousarray(self.headways, dtype=np.float64)
        r = np.ascontiguousarray(self.risk_levels, dtype=np.float64)
        self._keep = [h, r]
        return N.StatsReq(C.c_void_p(h.ctypes.data) if h.size else None, h.size,
                          C.c_void_p(r.ctypes.data) if r.size else None, r.size,
                          1 if self.summarize else 0, 0, float(self.bin_width),
                          int(self.hist_cap), int(self.cand_cap))


class StatsOut:
    """Caller-owned result arrays of one finish (bmc_stats)."""

    def __init__(self, req: StatsRequest, hist_cap: int = 1 << 16):
        self.req = req
        self.exceed = np.zeros(len(req.headways), dtype=np.uint64)
        self.msh = np.zeros(len(req.risk_levels), dtype=np.float64)
        self.hist = np.zeros(max(1, hist_cap), dtype=np.uint64)
        self.s = N.Stats()
        self.s.exceed = C.c_void_p(self.exceed.ctypes.data) if self.exceed.size else None
        self.s.min_safe_headway = C.c_void_p(self.msh.ctypes.data) if self.msh.size else None
        self.s.histogram = C.c_void_p(self.hist.ctypes.data)
        self.s.histogram_cap = self.hist.size

    def result(self) -> dict:
        s = self.s
        out = {"n": int(s.n), "horizon_count": int(s.horizon_count),
               "exceed": self.exceed.copy(), "min_safe_headway": self.msh.copy(),
               "launches": int(s.launches), "fallbacks": int(s.fallbacks)}
        if self.req.summarize:
            sm = {k: getattr(s.summary, k) for k, _ in N.Summary._fields_ if k != "pad_"}
            sm["right_skewed"] = bool(sm["right_skewed"])
            sm["histogram"] = self.hist[: s.summary.bins].copy()
            out["summary"] = sm
        if s.n:
            out["collision_probability"] = self.exceed.astype(np.float64) / float(s.n)
        return out


class StatsStage:
    """A device stage sized for up to ``max_n`` results per call."""

    def __init__(self, executor, req: StatsRequest, max_n: int):
        self.ex = executor
        self.req = req
        self.max_n = int(max_n)
        h = C.c_void_p()
        executor._check(executor.lib.bmc_stats_create(executor.ctx, C.byref(req.c()), self.max_n,
                                                      C.byref(h)))
        self.h = h

    def begin(self, stream=None):
        st = C.c_void_p(int(stream.cuda_stream)) if stream is not None else None
        self.ex._check(self.ex.lib.bmc_stats_begin(self.h, st))

    def accumulate(self, d, hz, stream=None):
        st = C.c_void_p(int(stream.cuda_stream)) if stream is not None else None
        self.ex._check(self.ex.lib.bmc_stats_accumulate(
            self.h, C.c_void_p(d.data_ptr()), C.c_void_p(hz.data_ptr()) if hz is not None else None,
            int(d.numel()), st))

    def finish(self, d, hz, merge=None, stream=None, hist_cap: int = 1 << 16) -> dict:
        # result arrays allocated once per stage (a bench step calls this every step)
        out = self._out if getattr(self, "_out", None) is not None and \
            self._out.hist.size == max(1, hist_cap) else StatsOut(self.req, hist_cap)
        self._out = out
        st = C.c_void_p(int(stream.cuda_stream)) if stream is not None else None
        mg = C.byref(merge.struct()) if merge is not None else None
        n = int(d.numel()) if d is not None else 0
        self.ex._check(self.ex.lib.bmc_stats_finish(
            self.h, C.c_void_p(d.data_ptr()) if n else None,
            C.c_void_p(hz.data_ptr()) if (hz is not None and n) else None, n, mg,
            C.byref(out.s), st))
        if merge is not None:
            merge.raise_pending()
        return out.result()

    def close(self):
        if self.h:
            self.ex.lib.bmc_stats_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def stats(executor, d, hz, req: StatsRequest, hist_cap: int = 1 << 16) -> dict:
    """One call over existing device outputs (bmc_cuda_stats)."""
    out = StatsOut(req, hist_cap)
    executor._check(executor.lib.bmc_cuda_stats(
        executor.ctx, C.c_void_p(d.data_ptr()), C.c_void_p(hz.data_ptr()) if hz is not None else None,
        int(d.numel()), C.byref(req.c()), C.byref(out.s)))
    return out.result()
