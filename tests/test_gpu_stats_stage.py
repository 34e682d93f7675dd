"""GPU: the fused statistics stage (bmc_stats_* / bmc_cuda_rollout_stats).

Every device answer is compared bit for bit with the host twin of the same
stage (tests/cpp/stats_host.cpp: the product's orchestration and arithmetic
on CPU) and with the reference's own analysis functions
(/root/reference/proj/src/analysis.cpp via oracle/_ref) on the reference's
own rollout results.  Bars as in tests/test_stats_stage.py.
"""
import json
import math
import os
import socket
import sys
import tempfile

import numpy as np
import pytest

import paper_2604_27193_b200 as bmc
from oracle.pyoracle import Model, World
from paper_2604_27193_b200.stats import StatsRequest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from hoststats import host_stats  # noqa: E402
from test_stats_stage import RISKS, _grid, _mk, _request, _results, check_vs_reference  # noqa: E402

pytestmark = pytest.mark.gpu


def _dev(res):
    import torch
    d = torch.from_numpy(np.ascontiguousarray(res["stop_distance"])).cuda()
    hz = torch.from_numpy(np.ascontiguousarray(res["hit_horizon"]).astype(np.uint8)).cuda()
    return d, hz


def _same(a, b):
    """Bitwise equality of two stage results (exact sums make every field exact)."""
    assert a["n"] == b["n"] and a["horizon_count"] == b["horizon_count"]
    assert np.array_equal(a["exceed"], b["exceed"])
    assert np.array_equal(a["min_safe_headway"].view(np.uint64), b["min_safe_headway"].view(np.uint64))
    if "summary" in a:
        for k, v in a["summary"].items():
            if k == "histogram":
                assert np.array_equal(v, b["summary"][k])
            elif isinstance(v, float):
                assert np.float64(v).view(np.uint64) == np.float64(b["summary"][k]).view(np.uint64), k
            else:
                assert v == b["summary"][k], k


@pytest.mark.parametrize("model,n", [(Model(seed=3), 12000), (Model.mixed(7), 30000),
                                     (Model(seed=1), 100001)])
@pytest.mark.parametrize("bw", [2.0, 0.37])
def test_device_stage_matches_host_twin_and_reference(ref, executor, model, n, bw):
    res = _results(ref, model, n)
    req = _request(res, bw)
    d, hz = _dev(res)
    got = executor.stats(d, hz, req.headways, req.risk_levels, True, bw)
    _same(got, host_stats(res["stop_distance"], res["hit_horizon"], req))
    check_vs_reference(ref, res, got, req)
    assert got["fallbacks"] == 0


@pytest.mark.parametrize("d,hz", [
    ([42.0], None), ([3.0, 1.0], None), ([5.5] * 1000, None),
    ([1.0, 2.0, 3.0, 4.0], [0, 0, 1, 1]), ([7.0, 8.0, 9.0], [1, 1, 1]),
    (list(np.linspace(0.0, 1e-300, 777)), None), ([-3.0, -1.0, 2.0, 2.0, 2.0, 1e4], None),
])
def test_device_edge_batches(ref, executor, d, hz):
    res = _mk(d, hz)
    req = StatsRequest(headways=[0.0, 1.0, 2.0, 2.5, 100.0], risk_levels=RISKS, summarize=True,
                       bin_width=0.5)
    dd, hh = _dev(res)
    got = executor.stats(dd, hh, req.headways, req.risk_levels, True, 0.5)
    check_vs_reference(ref, res, got, req)
    _same(got, host_stats(res["stop_distance"], res["hit_horizon"], req))


def test_device_candidate_overflow_fallback(ref, executor):
    res = _results(ref, Model.mixed(5), 20000)
    req = _request(res)
    d, hz = _dev(res)
    want = executor.stats(d, hz, req.headways, req.risk_levels, True, 2.0)
    got = executor.stats(d, hz, req.headways, req.risk_levels, True, 2.0, cand_cap=3)
    assert got["fallbacks"] > 0 and want["fallbacks"] == 0
    _same(got, want)
    check_vs_reference(ref, res, got, req)


@pytest.mark.parametrize("opts", [dict(), dict(ilp=2, block_threads=640), dict(ilp=1, test_block=1),
                                  dict(schedule="index"), dict(table="global"),
                                  dict(table="none", block_threads=256)])
def test_rollout_fused_pass1(ref, executor, opts):
    """Pass 1 in the rollout epilogue == pass 1 over the finished outputs."""
    import torch
    samples, _ = ref.draw_batch(Model.mixed(23), 40000)
    res, _, _ = ref.run(samples, World(), "parallel")
    terms = bmc.stage_terms(samples)
    dev = [torch.from_numpy(terms[i]).cuda() for i in range(4)]
    n = samples.shape[0]
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.empty(n, dtype=torch.int32, device="cuda")
    hz = torch.empty(n, dtype=torch.uint8, device="cuda")
    req = _request(res)
    stage = executor.stats_stage(n, req.headways, req.risk_levels, True, 2.0)
    stage.begin()
    executor.rollout_device(dev, (d, st, hz), stats=stage, **opts)
    got = stage.finish(d, hz)
    assert np.array_equal(d.cpu().numpy().view(np.uint64), res["stop_distance"].view(np.uint64))
    _same(got, host_stats(res["stop_distance"], res["hit_horizon"], req))
    check_vs_reference(ref, res, got, req)
    # the stage is reusable: a second begin/rollout/finish gives the same bits
    stage.begin()
    executor.rollout_device(dev, (d, st, hz), stats=stage, **opts)
    _same(stage.finish(d, hz), got)
    stage.close()


def test_rollout_fused_stats_only(ref, executor):
    """No per-sample outputs except what the stage's later passes read."""
    import torch
    samples, _ = ref.draw_batch(Model(seed=8), 5000)
    res, _, _ = ref.run(samples, World(), "parallel")
    terms = bmc.stage_terms(samples)
    dev = [torch.from_numpy(terms[i]).cuda() for i in range(4)]
    n = samples.shape[0]
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    hz = torch.empty(n, dtype=torch.uint8, device="cuda")
    req = StatsRequest(headways=[60.0, 80.0, 100.0])
    stage = executor.stats_stage(n, req.headways)
    stage.begin()
    executor.rollout_device(dev, (d, None, hz), stats=stage)
    got = stage.finish(d, hz)
    for h, c in zip(req.headways, got["exceed"]):
        assert float(c) / n == ref.collision_probability(res, h)


def test_decision_graph_returns_statistics(ref, executor):
    n = 25000
    ttc = [1.0 + 0.25 * k for k in range(21)]
    req = StatsRequest(headways=[t * 30.0 for t in ttc], risk_levels=[0.05, 0.01, 0.001],
                       summarize=True, bin_width=2.0)
    g = executor.graph(n, stats=req)
    try:
        for seed in (1, 2):
            samples, _ = ref.draw_batch(Model(seed=seed), n)
            want, _, _ = ref.run(samples, World(), "parallel")
            rep = g.run(samples)
            assert np.array_equal(rep.results["stop_distance"].view(np.uint64),
                                  want["stop_distance"].view(np.uint64))
            got = g.stats()
            _same(got, host_stats(want["stop_distance"], want["hit_horizon"], req))
            check_vs_reference(ref, want, got, req)
            assert rep.launches >= 8  # bin (3) + rollout + unpermute + stage kernels
        # model-driven decisions (sampling inside the graph) carry statistics too
        rep = g.run_model(bmc.UncertaintyModel(seed=4))
        samples, _ = ref.draw_batch(Model(seed=4), n)
        want, _, _ = ref.run(samples, World(), "parallel")
        _same(g.stats(), host_stats(want["stop_distance"], want["hit_horizon"], req))
    finally:
        g.close()


def test_summarize_and_legacy_entry_points_agree(ref, executor):
    res = _results(ref, Model.mixed(31), 20000)
    d, hz = _dev(res)
    s = executor.summarize(d, hz, 0.37)
    want = ref.summarize(res, 0.37)
    for k in ("n", "horizon_count", "bins", "min", "max", "median", "origin"):
        assert s[k] == want[k]
    assert np.array_equal(s["histogram"], np.asarray(want["histogram"], dtype=np.uint64))
    assert executor.min_safe_headway(d, hz, 0.01) == ref.min_safe_headway(res, 0.01)


# ------------------------------------------- two ranks sharing one B200

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, outdir, port):
    import torch
    import torch.distributed as dist
    from paper_2604_27193_b200.distributed import TorchMerge, shard_range
    from oracle.pyoracle import Reference
    from test_stats_stage import _jsonable
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        ref = Reference()
        samples, _ = ref.draw_batch(Model.mixed(13), 7001)
        res, _, _ = ref.run(samples, World(), "parallel")
        b, e = shard_range(res.shape[0], rank, world)
        ex = bmc.CudaExecutor(0)
        terms = bmc.stage_terms(samples[b:e])
        dev = [torch.from_numpy(terms[i]).cuda() for i in range(4)]
        n = e - b
        d = torch.empty(n, dtype=torch.float64, device="cuda")
        st = torch.empty(n, dtype=torch.int32, device="cuda")
        hz = torch.empty(n, dtype=torch.uint8, device="cuda")
        req = _request(res)
        stage = ex.stats_stage(n, req.headways, req.risk_levels, True, 2.0)
        stage.begin()
        ex.rollout_device(dev, (d, st, hz), stats=stage)
        merge = TorchMerge(dist, "cuda", via_host=True)
        out = stage.finish(d, hz, merge=merge)
        with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
            json.dump(_jsonable(out), f)
        stage.close()
        ex.close()
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_merge_bitwise(ref):
    import torch.multiprocessing as mp
    from test_stats_stage import _jsonable
    res = _results(ref, Model.mixed(13), 7001)
    single = host_stats(res["stop_distance"], res["hit_horizon"], _request(res))
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(2, tmp, _free_port()), nprocs=2, join=True)
        outs = [json.load(open(os.path.join(tmp, f"rank{r}.json"))) for r in range(2)]
    for o in outs:
        assert o == _jsonable(single)


def test_run_model_stream_with_fused_statistics(ref, executor):
    """bmc_cuda_run_model_stats: pass 1 in every chunk's rollout (every slot
    streams), the rest after the stream -- equal to the one-call stage."""
    import torch
    m = Model.mixed(19)
    n = 50001
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.empty(n, dtype=torch.int32, device="cuda")
    hz = torch.empty(n, dtype=torch.uint8, device="cuda")
    samples, _ = ref.draw_batch(m, n)
    want, _, _ = ref.run(samples, World(), "parallel")
    req = _request(want)
    stage = executor.stats_stage(n, req.headways, req.risk_levels, True, 2.0)
    stage.begin()
    executor.run_model(bmc.UncertaintyModel(m.seed, *zip(m.mean, m.sd)), n,
                       device_out=(d, st, hz), stats=stage, chunk=7000)
    got = stage.finish(d, hz)
    assert np.array_equal(d.cpu().numpy().view(np.uint64), want["stop_distance"].view(np.uint64))
    _same(got, host_stats(want["stop_distance"], want["hit_horizon"], req))
    check_vs_reference(ref, want, got, req)
    stage.close()


def _pass2_batch(kind):
    """Data aimed at pass 2's paths: the 128-bit fixed-point sums (terms on
    the grid), their superaccumulator fallback (values within a few ulps of
    the batch mean, so dev*dev lies far below the grid), both signs of m3
    terms, zero deviations, bin edges and their neighbours for the
    power-of-two histogram index, and non-finite values that switch the fast
    path off."""
    rng = np.random.default_rng(11)
    x = np.round(rng.normal(0.0, 12.0, 150000) * 2.0 ** 20) / 2.0 ** 20
    edges = np.arange(20.0, 140.0, 0.5)
    base = np.concatenate([80.0 + x, 80.0 - x, edges, np.nextafter(edges, 0.0), [900.0, -150.0]])
    m = math.fsum(base) / base.size          # the batch mean (pairs about it keep it)
    k = np.arange(1, 200) * np.spacing(m)
    d = np.concatenate([base, np.full(3000, m), m + k, m - k])
    if kind == "nan":
        d = np.concatenate([d, [np.nan] * 5])
    elif kind == "inf":
        d = np.concatenate([d, [np.inf, 3.0]])
    rng.shuffle(d)
    hz = (rng.random(d.shape[0]) < 0.01).astype(np.uint8)
    return d, hz


@pytest.mark.parametrize("kind", ["finite", "nan", "inf"])
@pytest.mark.parametrize("bw", [2.0, 0.5, 0.37])
def test_device_pass2_fast_paths_exact(ref, executor, kind, bw):
    d, hz = _pass2_batch(kind)
    res = _mk(d, hz)
    req = StatsRequest(headways=[50.0, 80.0, 100.0], risk_levels=RISKS, summarize=True,
                       bin_width=bw)
    dd, hh = _dev(res)
    if kind == "inf":
        # +inf makes the reference's bin count (size_t)ceil(inf / bw) undefined: both the
        # device stage and its host twin refuse with BMC_E_RANGE instead of allocating
        with pytest.raises(bmc.BmcError) as e_dev:
            executor.stats(dd, hh, req.headways, req.risk_levels, True, bw)
        with pytest.raises(bmc.BmcError) as e_host:
            host_stats(res["stop_distance"], res["hit_horizon"], req)
        assert e_dev.value.code == e_host.value.code == -5 and "bins" in str(e_dev.value)
        return
    got = executor.stats(dd, hh, req.headways, req.risk_levels, True, bw)
    _same(got, host_stats(res["stop_distance"], res["hit_horizon"], req))
    if kind == "finite":
        check_vs_reference(ref, res, got, req)
