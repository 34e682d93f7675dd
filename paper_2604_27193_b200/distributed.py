"""Sharded statistics: one process per GPU, contiguous index shards.

Product path: ``TorchMerge`` -- the bmc_merge hooks of the fused statistics
stage (stats.StatsStage.finish(..., merge=TorchMerge(dist))) over
torch.distributed: three merge points per step (P1 partials SUM + extrema
MIN, P2 partials SUM, candidate counts + keys all-gather), every collective
on device buffers in the stage's stream (NCCL), and exact partials (integer
counts, u64 limbs of exact sums), so every rank finishes with the
single-device answer bit for bit.  bench.py uses it under torchrun.

The quantity-by-quantity merge below (Collective / HostShard / DeviceShard:
one small collective per quantity, radix select with one allreduce per
8-bit pass) is the round-1 path, kept for callers that want one statistic
and as a second, independent implementation the tests cross-check.

SURVEY.md section 8(e): sample i depends only on (seed, i) (sampling.hpp:3-6),
so rank r owns [r*N/G, (r+1)*N/G) and nothing crosses devices on the data
path.  The statistics of analysis.cpp combine with one small allreduce per
quantity:

* counts (horizon, exceedance per headway, histogram bins, radix-select
  digit histograms) add exactly -> integer results are bit-identical to a
  single-device run for any world size;
* extrema take MIN / MAX exactly;
* double-double sums are all-gathered and merged in rank order on every rank
  (deterministic; within a few ulp of the exact sum -- the reference's own
  sequential sum is within n*eps of it).

Order statistics (median, min_safe_headway) use distributed radix select:
each 8-bit pass allreduces the per-target digit histograms, and every rank
walks the same global histogram to the same digit, so the selected value is
the exact global order statistic.

The merge logic is written against a small "shard" protocol so the CUDA
shard (``DeviceShard``, the product path) and a NumPy shard (``HostShard``,
used by the CPU multi-process tests) run the identical code.
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence

import numpy as np

MAX_TARGETS = 16


def shard_range(n_total: int, rank: int, world: int):
    """Contiguous shard [begin, end) of rank r (same split as run_cuda)."""
    return n_total * rank // world, n_total * (rank + 1) // world


# ------------------------------------------------------------ collectives

class Collective:
    """Allreduce / allgather of small host vectors over torch.distributed.
    ``device`` is where the staging tensors live ("cuda:k" for NCCL, "cpu"
    for gloo).  dist=None (a single process) is a no-op; a process group of
    size 1 still runs the collectives (so torchrun at N=1 exercises them)."""

    def __init__(self, dist=None, device: str = "cpu"):
        self.dist = dist
        self.device = device
        self.world = dist.get_world_size() if dist is not None else 1

    def _t(self, arr, dtype):
        import torch
        return torch.as_tensor(np.ascontiguousarray(arr), dtype=dtype).to(self.device)

    def sum_u64(self, arr) -> np.ndarray:
        arr = np.asarray(arr, dtype=np.uint64)
        if self.dist is None:
            return arr.copy()
        import torch
        assert int(arr.max(initial=0)) < 2 ** 63
        t = self._t(arr.astype(np.int64), torch.int64)
        self.dist.all_reduce(t)
        return t.cpu().numpy().astype(np.uint64)

    def min_f64(self, x: float) -> float:
        return self._reduce_f64(x, "min")

    def max_f64(self, x: float) -> float:
        return self._reduce_f64(x, "max")

    def _reduce_f64(self, x: float, op: str) -> float:
        if self.dist is None:
            return float(x)
        import torch
        t = self._t([x], torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN if op == "min" else self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather_f64(self, vec) -> np.ndarray:
        """rank-ordered all-gather: returns shape (world, len(vec))."""
        vec = np.asarray(vec, dtype=np.float64)
        if self.dist is None:
            return vec[None, :].copy()
        import torch
        t = self._t(vec, torch.float64)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t)
        return np.stack([o.cpu().numpy() for o in out])


# ------------------------------------------- merge hooks of the stats stage

_SIGN = -(1 << 63)  # int64 bit pattern 0x8000...: flips unsigned <-> signed order


class _CudaWords:
    """A raw device pointer seen as an int64 tensor (no copy)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class TorchMerge:
    """bmc_merge over torch.distributed (brakemc_cuda.h): the statistics
    stage calls these hooks at its merge points with buffers of its own
    memory -- device pointers for the CUDA engine (NCCL: the collective is
    enqueued on the stage's stream), host pointers for the host twin used by
    the gloo tests.  u64 words ride as int64: SUM is the same bits either
    way; MIN/MAX of unsigned keys run on keys with the sign bit flipped."""

    def __init__(self, dist, device: str = "cuda", world: Optional[int] = None,
                 rank: Optional[int] = None, via_host: bool = False):
        from . import _native as N
        self.N = N
        self.dist = dist
        self.device = device
        # gloo between ranks that hold device buffers: stage through host memory
        self.via_host = via_host
        self.world = world if world is not None else dist.get_world_size()
        self.rank = rank if rank is not None else dist.get_rank()
        self.error = None
        self.calls = 0
        self._ar = N.ALLREDUCE_FN(self._allreduce)
        self._ag = N.ALLGATHER_FN(self._allgather)
        self._s = N.Merge(None, self.world, self.rank, self._ar, self._ag)

    def struct(self):
        return self._s

    def raise_pending(self):
        if self.error is not None:
            e, self.error = self.error, None
            raise e

    def _view(self, ptr, n):
        import torch
        if self.device == "cpu":
            import ctypes
            arr = np.frombuffer((ctypes.c_int64 * n).from_address(ptr), dtype=np.int64)
            return torch.from_numpy(arr)
        return torch.as_tensor(_CudaWords(ptr, n), device=self.device)

    def _stream_ctx(self, stream):
        import contextlib
        import torch
        if self.device == "cpu" or not stream:
            return contextlib.nullcontext()
        return torch.cuda.stream(torch.cuda.ExternalStream(stream, device=self.device))

    def _allreduce(self, user, buf, count, op, stream):
        try:
            self.calls += 1
            dev = self._view(buf, count)
            with self._stream_ctx(stream):
                t = dev.cpu() if self.via_host else dev
                if op == self.N.MERGE_SUM:
                    self.dist.all_reduce(t)
                else:
                    t.bitwise_xor_(_SIGN)
                    self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN if op == self.N.MERGE_MIN
                                         else self.dist.ReduceOp.MAX)
                    t.bitwise_xor_(_SIGN)
                if self.via_host:
                    dev.copy_(t)
            return 0
        except Exception as e:  # noqa: BLE001 -- reported after the C call returns
            self.error = e
            return 1

    def _allgather(self, user, send, recv, count, stream):
        try:
            self.calls += 1
            src = self._view(send, count)
            dst = self._view(recv, count * self.world)
            with self._stream_ctx(stream):
                if self.device == "cpu" or self.via_host:
                    hdst = dst.cpu() if self.via_host else dst
                    self.dist.all_gather(list(hdst.chunk(self.world)), src.cpu())
                    if self.via_host:
                        dst.copy_(hdst)
                else:
                    self.dist.all_gather_into_tensor(dst, src)
            return 0
        except Exception as e:  # noqa: BLE001
            self.error = e
            return 1


# ---------------------------------------------------------- dd arithmetic

def dd_merge(a, b):
    """(hi, lo) + (hi, lo) with TwoSum on the high parts (IEEE doubles)."""
    s = a[0] + b[0]
    bb = s - a[0]
    err = (a[0] - (s - bb)) + (b[0] - bb)
    return (s, a[1] + err + b[1])


def dd_merge_rows(rows):
    acc = (0.0, 0.0)
    for r in rows:
        acc = dd_merge(acc, (float(r[0]), float(r[1])))
    return acc


# --------------------------------------------------------------- shards

def order_key(d: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(d, dtype=np.float64).view(np.uint64)
    neg = (b >> np.uint64(63)) != 0
    return np.where(neg, ~b, b | np.uint64(1 << 63))


def key_value(k: int) -> float:
    k = int(k)
    b = (k & 0x7FFFFFFFFFFFFFFF) if (k >> 63) else (~k & 0xFFFFFFFFFFFFFFFF)
    return float(np.array([b], dtype=np.uint64).view(np.float64)[0])


class HostShard:
    """NumPy shard with the device kernels' exact semantics (test backend)."""

    def __init__(self, stop_distance: np.ndarray, hit_horizon: np.ndarray):
        self.d = np.ascontiguousarray(stop_distance, dtype=np.float64)
        self.hz = np.ascontiguousarray(hit_horizon, dtype=np.uint8)

    def partials(self):
        n = self.d.size
        return dict(count=n, horizon_count=int((self.hz != 0).sum()),
                    min=float(self.d.min()) if n else math.inf,
                    max=float(self.d.max()) if n else -math.inf,
                    sum=(math.fsum(self.d.tolist()), 0.0))

    def moments(self, mean: float):
        dev = self.d - mean
        sq = dev * dev
        return (math.fsum(sq.tolist()), 0.0), (math.fsum((sq * dev).tolist()), 0.0)

    def histogram(self, origin: float, bw: float, bins: int) -> np.ndarray:
        if self.d.size == 0:
            return np.zeros(bins, dtype=np.uint64)
        idx = ((self.d - origin) / bw).astype(np.uint64)
        idx = np.minimum(idx, np.uint64(bins - 1))
        return np.bincount(idx.astype(np.int64), minlength=bins).astype(np.uint64)

    def exceedance(self, headways) -> np.ndarray:
        h = np.asarray(headways, dtype=np.float64)
        hz = self.hz != 0
        return np.array([int((hz | (self.d > x)).sum()) for x in h], dtype=np.uint64)

    def select_pass(self, exclude_horizon: bool, shift: int, prefixes) -> np.ndarray:
        keys = order_key(self.d[self.hz == 0] if exclude_horizon else self.d)
        mask = np.uint64(0) if shift >= 56 else np.uint64((~0 << (shift + 8)) & 0xFFFFFFFFFFFFFFFF)
        digit = ((keys >> np.uint64(shift)) & np.uint64(0xFF)).astype(np.int64)
        out = np.zeros((len(prefixes), 256), dtype=np.uint64)
        for t, p in enumerate(prefixes):
            sel = (keys & mask) == np.uint64(p)
            out[t] = np.bincount(digit[sel], minlength=256).astype(np.uint64)
        return out


class DeviceShard:
    """The product shard: device-resident outputs of this rank's rollout."""

    def __init__(self, executor, stop_distance, hit_horizon):
        self.ex = executor
        self.d = stop_distance
        self.hz = hit_horizon

    def partials(self):
        p = self.ex.partials(self.d, self.hz)
        return dict(count=p["count"], horizon_count=p["horizon_count"], min=p["min"],
                    max=p["max"], sum=(p["sum_hi"], p["sum_lo"]))

    def moments(self, mean: float):
        m = self.ex.moments(self.d, mean)
        return (m[0], m[1]), (m[2], m[3])

    def histogram(self, origin: float, bw: float, bins: int) -> np.ndarray:
        return self.ex.histogram(self.d, origin, bw, bins)

    def exceedance(self, headways) -> np.ndarray:
        return self.ex.exceedance_counts(self.d, self.hz, headways)

    def select_pass(self, exclude_horizon: bool, shift: int, prefixes) -> np.ndarray:
        return self.ex.select_pass(self.d, self.hz, exclude_horizon, shift, prefixes)

    def exceedance_ttc_noise(self, ttc, closing_speed, sigma, noise_seed, first) -> np.ndarray:
        return self.ex.exceedance_ttc_noise(self.d, self.hz, ttc, closing_speed, sigma,
                                            noise_seed, first)


# ------------------------------------------------------ merged statistics

def order_stats(shard, coll: Collective, ranks: Sequence[int], exclude_horizon: bool):
    """Exact global order statistics (1-based ranks); NaN for ranks outside
    [1, count].  Returns (values, candidate count)."""
    ranks = [int(r) for r in ranks]
    vals: List[float] = [math.nan] * len(ranks)
    count = 0
    for t0 in range(0, max(1, len(ranks)), MAX_TARGETS):
        part = ranks[t0:t0 + MAX_TARGETS]
        if not part:
            break
        prefix = [0] * len(part)
        resid = list(part)
        valid = [True] * len(part)
        for shift in range(56, -8, -8):
            h = coll.sum_u64(shard.select_pass(exclude_horizon, shift, prefix).reshape(-1))
            h = h.reshape(len(part), 256)
            if shift == 56:
                count = int(h[0].sum())
                valid = [1 <= r <= count for r in resid]
            for t in range(len(part)):
                if not valid[t]:
                    continue
                cum = np.cumsum(h[t].astype(np.int64))
                digit = int(np.searchsorted(cum, resid[t]))
                resid[t] -= int(cum[digit - 1]) if digit > 0 else 0
                prefix[t] |= digit << shift
        for t in range(len(part)):
            vals[t0 + t] = key_value(prefix[t]) if valid[t] else math.nan
    return vals, count


def summarize(shard, coll: Collective, bin_width: float = 2.0) -> dict:
    """summarize (analysis.cpp:13-76) over all ranks' shards."""
    if not bin_width > 0.0:
        raise ValueError("outputs.bin_width: must be > 0")
    p = shard.partials()
    cnt = coll.sum_u64([p["count"], p["horizon_count"]])
    n, horizon = int(cnt[0]), int(cnt[1])
    if n == 0:
        raise ValueError("summarize: needs at least one result")
    mn = coll.min_f64(p["min"])
    mx = coll.max_f64(p["max"])
    s = dd_merge_rows(coll.gather_f64(list(p["sum"])))
    mean = (s[0] + s[1]) / float(n)
    m2l, m3l = shard.moments(mean)
    g = coll.gather_f64([m2l[0], m2l[1], m3l[0], m3l[1]])
    m2 = dd_merge_rows(g[:, 0:2])
    m3 = dd_merge_rows(g[:, 2:4])
    M2, M3 = m2[0] + m2[1], m3[0] + m3[1]
    sd = math.sqrt(M2 / (n - 1.0)) if n > 1 else 0.0
    var_pop = M2 / n
    skew = (M3 / n) / math.pow(var_pop, 1.5) if var_pop > 0.0 else 0.0
    ranks = [n // 2 + 1] if n % 2 == 1 else [n // 2, n // 2 + 1]
    med, _ = order_stats(shard, coll, ranks, exclude_horizon=False)
    median = med[0] if n % 2 == 1 else 0.5 * (med[0] + med[1])
    lo, hi = math.floor(mn), math.ceil(mx)
    bins = max(1, int(math.ceil((hi - lo) / bin_width)))
    hist = coll.sum_u64(shard.histogram(lo, bin_width, bins))
    return dict(n=n, horizon_count=horizon, mean=mean, sd=sd, min=mn, max=mx, median=median,
                skewness=skew, right_skewed=mean > median, origin=lo, bin_width=bin_width,
                bins=bins, histogram=hist)


def exceedance_counts(shard, coll: Collective, headways) -> np.ndarray:
    for h in headways:
        if not h >= 0.0:
            raise ValueError("risk.headway: must be >= 0")
    return coll.sum_u64(shard.exceedance(headways))


def exceedance_ttc_noise_counts(shard, coll: Collective, ttc, closing_speed: float, sigma: float,
                                noise_seed: int, first: int) -> np.ndarray:
    """Sensor-noise TTC sweep over all ranks: each rank's noise draws use its
    global sample indices (first = its shard start), so the sum equals a
    single-device run exactly."""
    return coll.sum_u64(shard.exceedance_ttc_noise(ttc, closing_speed, sigma, noise_seed, first))


def min_safe_headways(shard, coll: Collective, n_total: int, risks: Sequence[float]):
    """min_safe_headway (analysis.cpp:161-194) for several risk levels."""
    ranks = []
    for r in risks:
        if not (0.0 < r < 1.0):
            raise ValueError("risk.level: must be strictly between 0 and 1")
        raw = (1.0 - r) * float(n_total)
        ranks.append(int(math.ceil(raw - raw * 1e-12)))
    vals, stopped = order_stats(shard, coll, ranks, exclude_horizon=True)
    return [math.inf if rk > stopped else v for rk, v in zip(ranks, vals)]


def build_risk_curve(shard, coll: Collective, n_total: int, grid, levels, closing_speed: float):
    """build_risk_curve (analysis.cpp:203-228) over all shards."""
    counts = exceedance_counts(shard, coll, grid)
    probs = counts.astype(np.float64) / float(n_total)
    lv = sorted(levels, reverse=True)
    heads = min_safe_headways(shard, coll, n_total, lv)
    if not closing_speed > 0.0:
        raise ValueError("risk.closing_speed: must be > 0")
    return probs, [(r, h, h / closing_speed) for r, h in zip(lv, heads)]
