"""Fused statistics stage on CPU: the product's orchestration and arithmetic
(csrc/bmc_stats_pipeline.h, csrc/bmc_stats_core.h) run by the host test
backend (tests/cpp/stats_host.cpp), checked against the reference's own
analysis functions (/root/reference/proj/src/analysis.cpp via oracle/_ref)
and merged across gloo ranks through the same bmc_merge hooks the CUDA
engine calls (distributed.TorchMerge).

Bars: counts, extrema, median, histogram, collision numerators and
min_safe_headway are bit-identical to the reference; the stage's sums are
exact (correctly rounded), so mean/sd/skewness are within the reference's
own summation error of it, and every shard split gives identical bits.
"""
import json
import math
import os
import socket
import sys
import tempfile

import numpy as np
import pytest

from oracle.pyoracle import Model, World
from paper_2604_27193_b200.stats import StatsRequest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from hoststats import exact_sum, hist_index_mismatches, host_stats  # noqa: E402

RISKS = [0.05, 0.01, 0.001, 0.5]
EPS = 2.0 ** -52


def _grid(d):
    lo, hi = math.floor(float(d.min())) - 5.0, math.ceil(float(d.max())) + 5.0
    return [lo + k for k in range(int(hi - lo) + 1)]


def _results(ref, model, n):
    samples, _ = ref.draw_batch(model, n)
    res, _, _ = ref.run(samples, World(), "parallel")
    return res


def _request(res, bin_width=2.0, risks=RISKS):
    return StatsRequest(headways=_grid(res["stop_distance"]), risk_levels=risks, summarize=True,
                        bin_width=bin_width)


def check_vs_reference(ref, res, out, req):
    """The stage's answer vs the reference's analysis.cpp on the same results."""
    n = res.shape[0]
    d = res["stop_distance"]
    want = ref.summarize(res, req.bin_width)
    got = out["summary"]
    for k in ("n", "horizon_count", "bins"):
        assert got[k] == want[k], k
    for k in ("min", "max", "median", "origin"):
        assert got[k] == want[k], (k, got[k], want[k])
    assert np.array_equal(got["histogram"], np.asarray(want["histogram"], dtype=np.uint64))
    # exact sum vs the reference's sequential sum: within (n-1) eps sum|d|
    bound = (n - 1) * EPS * float(np.abs(d).sum()) / n + abs(want["mean"]) * EPS
    assert abs(got["mean"] - want["mean"]) <= bound
    assert got["sd"] == pytest.approx(want["sd"], rel=1e-12)
    assert got["skewness"] == pytest.approx(want["skewness"], rel=1e-9, abs=1e-12)
    if abs(want["mean"] - want["median"]) > 4 * bound:
        assert got["right_skewed"] == want["right_skewed"]
    # collision_probability numerators (analysis.cpp:145-159), bit for bit
    for h, c in zip(req.headways, out["exceed"]):
        assert float(c) / n == ref.collision_probability(res, h), h
    # min_safe_headway (analysis.cpp:161-194), exact incl. the +inf tail
    for r, v in zip(req.risk_levels, out["min_safe_headway"]):
        assert v == ref.min_safe_headway(res, r), r


# -------------------------------------------------- exact superaccumulator

def test_exact_sum_is_correctly_rounded():
    rng = np.random.default_rng(5)
    cases = [
        rng.normal(80.0, 12.0, 100000),
        np.concatenate([rng.normal(0, 1, 5000), -rng.normal(0, 1, 5000)]),
        np.array([1e16, 1.0, -1e16, 1e-300, 5e-324, -5e-324, 3.0]),
        np.array([1.7976931348623157e308, -1.7976931348623157e308, 1e308, 1e-308]),
        np.array([2.0 ** -1074] * 7 + [2.0 ** -1022]),
        rng.standard_cauchy(20000),
        np.array([0.1] * 10),
        np.array([1.0, 2.0 ** -53, 2.0 ** -53]),          # ties: rounds to even
        np.array([1.0, 2.0 ** -53, 2.0 ** -105]),          # just above the tie
        np.array([-0.0, -0.0]),
    ]
    for v in cases:
        assert exact_sum(v) == math.fsum(v.tolist()), v[:5]
    assert math.isnan(exact_sum(np.array([1.0, np.nan])))
    assert exact_sum(np.array([1.0, np.inf])) == np.inf
    assert math.isnan(exact_sum(np.array([np.inf, -np.inf])))
    assert exact_sum(np.array([1e308, 1e308])) == np.inf  # past DBL_MAX


def test_exact_sum_is_order_independent():
    rng = np.random.default_rng(9)
    v = rng.normal(50.0, 30.0, 50000) * np.exp(rng.normal(0, 8, 50000))
    s = exact_sum(v)
    for _ in range(3):
        rng.shuffle(v)
        assert exact_sum(v) == s


@pytest.mark.parametrize("lo,bw", [(20.0, 2.0), (20.0, 0.37), (-5.0, 0.1), (0.0, 1e-3),
                                   (37.0, 3.0), (1e6, 0.7)])
def test_division_free_histogram_index_is_exact(lo, bw):
    # the kernels' hist_index_fast must equal (size_t)((d - lo) / bw) on every
    # value, above all on the bin edges lo + k*bw and their neighbours
    rng = np.random.default_rng(3)
    k = np.arange(0, 5000, dtype=np.float64)
    edges = lo + k * bw
    v = np.concatenate([edges, np.nextafter(edges, np.inf), np.nextafter(edges, -np.inf),
                        lo + (k + 0.5) * bw, lo + rng.uniform(0, 5000 * bw, 200000),
                        [lo, np.nextafter(lo, np.inf), lo + 1e-300]])
    assert hist_index_mismatches(v, lo, bw, 4000) == 0


# ----------------------------------------------------- single rank vs ref

@pytest.mark.parametrize("model,n", [(Model(seed=3), 12000), (Model.mixed(7), 8000),
                                     (Model(seed=11), 9999)])
@pytest.mark.parametrize("bw", [2.0, 0.37])
def test_host_stage_matches_reference(ref, model, n, bw):
    res = _results(ref, model, n)
    req = _request(res, bw)
    out = host_stats(res["stop_distance"], res["hit_horizon"], req)
    check_vs_reference(ref, res, out, req)
    assert out["fallbacks"] == 0


def test_candidate_overflow_takes_exact_fallback(ref):
    res = _results(ref, Model.mixed(5), 6000)
    req = _request(res)
    want = host_stats(res["stop_distance"], res["hit_horizon"], req)
    got = host_stats(res["stop_distance"], res["hit_horizon"], req, cand_cap=3)
    assert got["fallbacks"] > 0
    check_vs_reference(ref, res, got, req)
    for k in ("median", "mean", "sd", "min", "max"):
        assert got["summary"][k] == want["summary"][k]
    assert np.array_equal(got["min_safe_headway"], want["min_safe_headway"])


def _mk(d, hz=None):
    d = np.asarray(d, dtype=np.float64)
    hz = np.zeros(d.size, np.uint8) if hz is None else np.asarray(hz, np.uint8)
    res = np.zeros(d.size, dtype=[("stop_distance", "<f8"), ("stop_time", "<f8"),
                                  ("steps", "<i8"), ("hit_horizon", "u1"), ("pad_", "V7")])
    res["stop_distance"] = d
    res["hit_horizon"] = hz
    res["steps"] = 1
    res["stop_time"] = 0.001
    return res


@pytest.mark.parametrize("d,hz", [
    ([42.0], None),                                   # n = 1
    ([3.0, 1.0], None),                               # even n: two median ranks
    ([5.5] * 1000, None),                             # span 0: one bucket, exact
    ([1.0, 2.0, 3.0, 4.0], [0, 0, 1, 1]),             # half the batch in the tail
    ([7.0, 8.0, 9.0], [1, 1, 1]),                     # all horizon: +inf headways
    (list(np.linspace(0.0, 1e-300, 777)), None),      # subnormal-scale spread
    ([-3.0, -1.0, 2.0, 2.0, 2.0, 1e4], None),         # negatives; > 8192 bins (fallback)
])
def test_edge_batches_match_reference(ref, d, hz):
    res = _mk(d, hz)
    req = StatsRequest(headways=[0.0, 1.0, 2.0, 2.5, 100.0], risk_levels=RISKS, summarize=True,
                       bin_width=0.5)
    out = host_stats(res["stop_distance"], res["hit_horizon"], req)
    check_vs_reference(ref, res, out, req)


def test_right_skewed_tie_is_exact():
    # mean == median exactly (symmetric values): the exact sum gives the
    # mathematically exact mean, so right_skewed is false, like the reference
    # whose sequential sum is exact here too
    d = np.array([1.0, 2.0, 3.0, 4.0, 5.0] * 200)
    out = host_stats(d, None, StatsRequest(summarize=True, bin_width=1.0))
    assert out["summary"]["mean"] == out["summary"]["median"] == 3.0
    assert out["summary"]["right_skewed"] is False


def test_request_validation():
    from paper_2604_27193_b200._native import BmcError, ConfigError
    d = np.array([1.0, 2.0])
    with pytest.raises(ConfigError, match="risk.headway"):
        host_stats(d, None, StatsRequest(headways=[-1.0]))
    with pytest.raises(ConfigError, match="risk.level"):
        host_stats(d, None, StatsRequest(risk_levels=[1.0]))
    with pytest.raises(ConfigError, match="outputs.bin_width"):
        host_stats(d, None, StatsRequest(summarize=True, bin_width=0.0))
    with pytest.raises(BmcError, match="at most 16"):
        host_stats(d, None, StatsRequest(risk_levels=[0.5] * 17))
    with pytest.raises(ConfigError, match="summarize: needs at least one result"):
        host_stats(np.zeros(0), None, StatsRequest(summarize=True))


# --------------------------------------------------------- gloo world 2/3

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _jsonable(out):
    o = {"n": out["n"], "horizon_count": out["horizon_count"],
         "exceed": [int(x) for x in out["exceed"]],
         "msh": [float(x) for x in out["min_safe_headway"]]}
    sm = dict(out["summary"])
    sm["histogram"] = [int(x) for x in sm["histogram"]]
    o["summary"] = {k: (float(v).hex() if isinstance(v, float) else v) for k, v in sm.items()}
    return o


def _worker(rank, world, outdir, port, cand_cap):
    import torch.distributed as dist
    from paper_2604_27193_b200.distributed import TorchMerge, shard_range
    from oracle.pyoracle import Reference
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        res = _results(Reference(), Model.mixed(13), 7001)
        b, e = shard_range(res.shape[0], rank, world)
        merge = TorchMerge(dist, "cpu")
        out = host_stats(res["stop_distance"][b:e], res["hit_horizon"][b:e], _request(res),
                         merge=merge, cand_cap=cand_cap)
        with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
            json.dump({"out": _jsonable(out), "calls": merge.calls}, f)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cand_cap", [(2, 0), (3, 0), (3, 5)])
def test_gloo_merge_equals_single_rank_bitwise(ref, world, cand_cap):
    import torch.multiprocessing as mp
    res = _results(ref, Model.mixed(13), 7001)
    req = _request(res)
    single = host_stats(res["stop_distance"], res["hit_horizon"], req)
    check_vs_reference(ref, res, single, req)
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, tmp, _free_port(), cand_cap), nprocs=world, join=True)
        outs = [json.load(open(os.path.join(tmp, f"rank{r}.json"))) for r in range(world)]
    for o in outs:
        # every rank holds the single-device answer, bit for bit (exact sums)
        assert o["out"] == _jsonable(single)
    # three merge points: P1 (SUM + MIN), P2 (SUM), candidates (counts + keys)
    assert outs[0]["calls"] >= 5


def test_infinite_range_histogram_refused():
    """+inf stop distances make the reference's bin count (size_t)ceil(inf / bw)
    undefined (analysis.cpp:61-63); the stage refuses with BMC_E_RANGE rather
    than sizing a 2^64-bin histogram."""
    from paper_2604_27193_b200 import BmcError
    req = StatsRequest(headways=[1.0], risk_levels=[0.05], summarize=True, bin_width=2.0)
    with pytest.raises(BmcError) as e:
        host_stats(np.array([1.0, 2.0, np.inf]), None, req)
    assert e.value.code == -5 and "bins" in str(e.value)
