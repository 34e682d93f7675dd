"""GPU parity at the headline scale ("what's weak" 1).

* 1e7 default-model samples (BASELINE C5 shape, seed 3): the fused
  statistics stage vs the reference's own host functions over the GPU's
  results -- summarize at bin widths 2.0 and 0.37, the 171-point
  build_risk_curve, min_safe_headway at {0.05, 0.01, 0.001}
  (analysis.cpp:13-76, 161-228) -- plus 200k random rollouts re-simulated by
  the reference bit for bit;
* 1e6 mixed-model samples (C4, ~27% horizon hits): every rollout vs the
  reference run_parallel, and the same statistics;
* 2^27 + 7 samples (past 1e8) drawn on the device: windows at the start,
  middle and end of the batch bit-identical to the reference, and the
  statistics equal a host recount -- exercises the 32-bit work counter,
  inverse permutation, bucket cursors and unpermute above the bench size.
"""
import math
import os
import sys

import numpy as np
import pytest

import paper_2604_27193_b200 as bmc
from oracle.pyoracle import Model, World

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from hoststats import host_stats  # noqa: E402
from test_gpu_stats_stage import _same  # noqa: E402
from test_stats_stage import check_vs_reference  # noqa: E402
from paper_2604_27193_b200.stats import StatsRequest  # noqa: E402

pytestmark = pytest.mark.gpu
RISKS = [0.05, 0.01, 0.001]


def _to_model(m: Model) -> bmc.UncertaintyModel:
    return bmc.UncertaintyModel(m.seed, *zip(m.mean, m.sd))


def _results_array(d, st, hz, dt=1e-3):
    n = d.shape[0]
    res = np.zeros(n, dtype=bmc.RESULT_DTYPE)
    res["stop_distance"] = d
    res["steps"] = st
    res["stop_time"] = st.astype(np.float64) * dt
    res["hit_horizon"] = hz
    return res


def _fused_run(executor, samples, req):
    import torch
    terms = bmc.stage_terms(samples)
    dev = [torch.from_numpy(terms[i]).cuda() for i in range(4)]
    del terms
    n = samples.shape[0]
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.empty(n, dtype=torch.int32, device="cuda")
    hz = torch.empty(n, dtype=torch.uint8, device="cuda")
    stage = executor.stats_stage(n, req.headways, req.risk_levels, req.summarize, req.bin_width)
    stage.begin()
    executor.rollout_device(dev, (d, st, hz), stats=stage)
    out = stage.finish(d, hz)
    stage.close()
    return out, d, st, hz


def _grid171(d):
    lo = math.floor(float(d.min())) - 5.0
    return [lo + k for k in range(171)]


def test_default_model_1e7_statistics_vs_reference(ref, executor):
    n = 10_000_000
    samples, _ = bmc.draw_batch(bmc.UncertaintyModel(seed=3), n)
    # probe the range for the grid with a first, statistics-free run
    out0, d, st, hz = _fused_run(executor, samples, StatsRequest(summarize=True, bin_width=2.0))
    grid = _grid171(np.array([out0["summary"]["min"]]))
    hd, hs, hh = d.cpu().numpy(), st.cpu().numpy(), hz.cpu().numpy()
    res = _results_array(hd, hs, hh)
    # 200k random rollouts re-simulated by the reference, bit for bit
    rng = np.random.default_rng(7)
    idx = np.sort(rng.choice(n, size=200_000, replace=False))
    want, _, _ = ref.run(np.ascontiguousarray(samples[idx]), World(), "parallel")
    assert np.array_equal(hd[idx].view(np.uint64), want["stop_distance"].view(np.uint64))
    assert np.array_equal(hs[idx].astype(np.int64), want["steps"])
    assert np.array_equal(hh[idx], want["hit_horizon"].astype(np.uint8))
    for bw in (2.0, 0.37):
        req = StatsRequest(headways=grid, risk_levels=RISKS, summarize=True, bin_width=bw)
        dev = executor.stats(d, hz, req.headways, req.risk_levels, True, bw)
        check_vs_reference(ref, res, dev, req)
        _same(dev, host_stats(hd, hh, req))
    # the 171-point risk curve as the reference builds it (analysis.cpp:203-228)
    probs, thr = ref.build_risk_curve(res, grid, RISKS, 30.0)
    dev = executor.stats(d, hz, grid, RISKS)
    assert np.array_equal(dev["exceed"].astype(np.float64) / n, np.asarray(probs))
    lv = sorted(RISKS, reverse=True)
    got = dict(zip(RISKS, dev["min_safe_headway"]))
    assert [(r, got[r], got[r] / 30.0) for r in lv] == [tuple(t) for t in thr]


def test_mixed_model_1e6_every_rollout_and_statistics(ref, executor):
    n = 1_000_000
    samples, _ = ref.draw_batch(Model.mixed(3), n)
    want, _, _ = ref.run(samples, World(), "parallel")
    assert want["hit_horizon"].mean() > 0.2
    req = StatsRequest(headways=_grid171(want["stop_distance"]), risk_levels=RISKS, summarize=True,
                       bin_width=0.37)
    out, d, st, hz = _fused_run(executor, samples, req)
    assert np.array_equal(d.cpu().numpy().view(np.uint64), want["stop_distance"].view(np.uint64))
    assert np.array_equal(st.cpu().numpy().astype(np.int64), want["steps"])
    assert np.array_equal(hz.cpu().numpy(), want["hit_horizon"].astype(np.uint8))
    check_vs_reference(ref, want, out, req)
    _same(out, host_stats(want["stop_distance"], want["hit_horizon"], req))


def test_beyond_1e8_samples_device_sampler(ref, executor):
    import torch
    if not bmc.device_sampler_available():
        pytest.skip("device sampler gate closed on this host")
    n = (1 << 27) + 7
    model = Model(seed=3)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.empty(n, dtype=torch.int32, device="cuda")
    hz = torch.empty(n, dtype=torch.uint8, device="cuda")
    rep, clamps = executor.run_model(_to_model(model), n, device_out=(d, st, hz), sampler="device")
    assert rep.total_steps > 0
    hd = d.cpu().numpy()
    hs = st.cpu().numpy()
    hh = hz.cpu().numpy()
    w = 20_000
    for first in (0, 1 << 24, (1 << 26) + 12345, n - w):
        smp, _ = bmc.draw_batch(_to_model(model), w, first=first)
        want, _, _ = ref.run(smp, World(), "parallel")
        assert np.array_equal(hd[first:first + w].view(np.uint64),
                              want["stop_distance"].view(np.uint64)), first
        assert np.array_equal(hs[first:first + w].astype(np.int64), want["steps"]), first
        assert np.array_equal(hh[first:first + w], want["hit_horizon"].astype(np.uint8)), first
    # statistics over all 2^27 + 7 results vs a host recount
    headways = [30.0 * (1.0 + 0.25 * k) for k in range(21)]
    out = executor.stats(d, hz, headways, RISKS, True, 2.0)
    hb = hh != 0
    assert out["n"] == n and out["horizon_count"] == int(hb.sum())
    for h, c in zip(headways, out["exceed"]):
        assert int(c) == int(np.count_nonzero(hb | (hd > h))), h
    sm = out["summary"]
    assert sm["min"] == hd.min() and sm["max"] == hd.max()
    srt = np.partition(hd, [n // 2])
    assert sm["median"] == srt[n // 2]  # n odd
    stopped = hd[~hb]
    for r, v in zip(RISKS, out["min_safe_headway"]):
        raw = (1.0 - r) * float(n)
        rank = int(math.ceil(raw - raw * 1e-12))
        assert v == (math.inf if rank > stopped.size else np.partition(stopped, rank - 1)[rank - 1])


def test_host_pipeline_above_8m_bitwise(ref, executor):
    """bmc_cuda_run above 8M samples (four pipeline chunks on two slot
    streams): results equal a run with other chunk sizes bit for bit, and the
    reference on a random subset."""
    n = 9_000_001
    samples, _ = bmc.draw_batch(bmc.UncertaintyModel(seed=5), n)
    dflt = executor.run(samples)
    assert dflt.chunks == 4
    other = executor.run(samples, chunk=1 << 21)
    assert np.array_equal(dflt.results.view(np.uint8), other.results.view(np.uint8))
    rng = np.random.default_rng(11)
    idx = np.sort(rng.choice(n, size=50_000, replace=False))
    want, _, _ = ref.run(np.ascontiguousarray(samples[idx]), World(), "parallel")
    got = dflt.results[idx]
    assert np.array_equal(got["stop_distance"].view(np.uint64), want["stop_distance"].view(np.uint64))
    assert np.array_equal(got["steps"], want["steps"])
    assert np.array_equal(got["stop_time"].view(np.uint64), want["stop_time"].view(np.uint64))


def test_streamed_model_head_chunk_schedule(ref, executor):
    """bmc_cuda_run_model with the automatic schedule at >= 8 chunks: a
    chunk/4 first piece, then 4M-sample chunks over three slot streams with
    direct chunk outputs.  Windows across every chunk boundary equal the
    reference, and the whole output equals an explicit fixed-chunk run."""
    n = 8 * (1 << 22) + 12345
    model = _to_model(Model(seed=6))
    rep, _ = executor.run_model(model, n)
    head = (1 << 22) // 4
    assert rep.chunks == 1 + (n - head + (1 << 22) - 1) // (1 << 22)
    got = rep.results
    w = 4_000
    bounds = [head] + [head + k * (1 << 22) for k in range(1, rep.chunks - 1)]
    for b in [0] + bounds + [n - w // 2]:
        first = max(0, min(n - w, b - w // 2))
        smp, _ = bmc.draw_batch(model, w, first=first)
        want, _, _ = ref.run(smp, World(), "parallel")
        g = got[first:first + w]
        assert np.array_equal(g["stop_distance"].view(np.uint64),
                              want["stop_distance"].view(np.uint64)), first
        assert np.array_equal(g["steps"], want["steps"]), first
    fixed, _ = executor.run_model(model, n, chunk=1 << 22)
    assert fixed.chunks == (n + (1 << 22) - 1) // (1 << 22)
    assert np.array_equal(fixed.results.view(np.uint8), got.view(np.uint8))
