"""GPU statistics parity vs the reference's analysis.cpp.

Exact (bit / integer) for counts, histogram, extrema, median, order
statistics, exceedance probabilities and risk thresholds.  mean / sd /
skewness: the reference sums sequentially (analysis.cpp:34-45) so any other
summation order differs in the last bits; the device uses double-double
accumulation.  Tolerance: 1e-12 relative (the reference's own test allows
1e-9 vs a Kahan oracle, test_analysis.cpp:61-62).
"""
import math

import numpy as np
import pytest

import paper_2604_27193_b200 as bmc
from oracle.pyoracle import RESULT_DTYPE, Model, World

pytestmark = pytest.mark.gpu
REL = 1e-12


def device(res):
    import torch
    d = torch.from_numpy(np.ascontiguousarray(res["stop_distance"])).cuda()
    hz = torch.from_numpy(np.ascontiguousarray(res["hit_horizon"])).cuda()
    return d, hz


def check_summary(got, want):
    for k in ("n", "horizon_count", "bins"):
        assert got[k] == want[k], k
    for k in ("min", "max", "median", "origin"):
        assert got[k] == want[k], k
    for k in ("mean", "sd"):
        assert got[k] == pytest.approx(want[k], rel=REL, abs=1e-300), k
    assert got["skewness"] == pytest.approx(want["skewness"], rel=1e-9, abs=1e-12)
    assert got["right_skewed"] == want["right_skewed"]
    assert np.array_equal(got["histogram"], want["histogram"])


@pytest.fixture(scope="module")
def readme(ref):
    samples, _ = ref.draw_batch(Model(seed=3), 12000)
    res, _, _ = ref.run(samples, World(), "parallel")
    return res


@pytest.fixture(scope="module")
def mixed(ref):
    samples, _ = ref.draw_batch(Model.mixed(3), 60000)
    res, _, _ = ref.run(samples, World(), "parallel")
    return res


@pytest.mark.parametrize("bw", [2.0, 0.37, 5.0])
def test_summarize(ref, executor, readme, mixed, bw):
    for res in (readme, mixed):
        d, hz = device(res)
        check_summary(executor.summarize(d, hz, bw, hist_cap=1 << 16), ref.summarize(res, bw))


def test_summarize_small_and_degenerate(ref, executor):
    for dist in ([75.0, 75.0, 75.0], [70.0, 80.0, 90.0], [42.0], [1.5, 2.5], list(range(1, 101))):
        res = np.zeros(len(dist), dtype=RESULT_DTYPE)
        res["stop_distance"] = dist
        d, hz = device(res)
        check_summary(executor.summarize(d, hz, 2.0), ref.summarize(res, 2.0))


def test_exceedance_and_risk_curve(ref, executor, readme, mixed):
    for res in (readme, mixed):
        d, hz = device(res)
        finite = res["stop_distance"]
        grid = ref.headway_grid(math.floor(finite.min()) - 5.0, math.ceil(finite.max()) + 5.0, 1.0)
        levels = [0.05, 0.01, 0.001, 0.3]
        probs, thr = ref.build_risk_curve(res, grid, levels, 30.0)
        gp, gthr = executor.build_risk_curve(d, hz, grid, levels, 30.0)
        assert np.array_equal(gp, probs)
        assert [tuple(t) for t in gthr] == [tuple(t) for t in thr]
        for h in (0.0, 77.7, float(finite[5]), 1e9):
            assert executor.collision_probability(d, hz, h) == ref.collision_probability(res, h)


def test_min_safe_headway_ties_and_horizon(ref, executor):
    rng = np.random.default_rng(123)
    dist = np.abs(rng.normal(79.0, 12.0, 1000))
    dist[[10, 20, 30]] = 90.0
    res = np.zeros(1000, dtype=RESULT_DTYPE)
    res["stop_distance"] = dist
    res["hit_horizon"][::97] = 1
    d, hz = device(res)
    for risk in (0.5, 0.25, 1.0 / 3.0, 0.05, 0.011, 0.002, 0.0101):
        assert executor.min_safe_headway(d, hz, risk) == ref.min_safe_headway(res, risk)
    with pytest.raises(bmc.ConfigError):
        executor.min_safe_headway(d, hz, 1.0)


def test_order_stats_exact(executor):
    import torch
    rng = np.random.default_rng(5)
    x = rng.normal(0.0, 50.0, 100001)
    x[:7] = [0.0, -0.0, 1e-300, -1e-300, 3.5, 3.5, -7.25]
    d = torch.from_numpy(x).cuda()
    ranks = [1, 2, 500, 50001, 99999, 100001]
    vals, cnt = executor.order_stats(d, None, ranks, exclude_horizon=False)
    srt = np.sort(x)
    assert cnt == x.size
    for r, v in zip(ranks, vals):
        assert v == srt[r - 1]
    vals, _ = executor.order_stats(d, None, [0, 100002], exclude_horizon=False)
    assert np.isnan(vals).all()


TTC = [1.0 + 0.25 * k for k in range(21)]


@pytest.mark.parametrize("sigma", [0.0, 0.05, 0.3, 1.5])
def test_sensor_noise_ttc_sweep(ref, executor, readme, mixed, sigma):
    # BASELINE C4's sensor-noise TTC sweep: device counts equal the C oracle
    # exactly (same glibc Box-Muller stream); sigma = 0 equals the plain
    # exceedance counts at T * v (the reference's collision_probability)
    from oracle.pyoracle import Port
    port = Port()
    v = 30.0
    for res in (readme, mixed):
        d, hz = device(res)
        got = executor.exceedance_ttc_noise(d, hz, TTC, v, sigma, noise_seed=7, first=1000)
        want = port.exceed_ttc_noise(res, TTC, v, sigma, noise_seed=7, first=1000)
        assert got.tolist() == want.tolist()
        if sigma == 0.0:
            assert got.tolist() == executor.exceedance_counts(d, hz, [t * v for t in TTC]).tolist()


def test_sensor_noise_ttc_shards_add_up(executor, mixed):
    # rank shards draw their noise at their global indices: the sum over
    # shards equals the single-device sweep, bit for bit
    d, hz = device(mixed)
    n = d.numel()
    whole = executor.exceedance_ttc_noise(d, hz, TTC[::-1], 30.0, 0.2, noise_seed=11, first=0)
    cut = n // 3
    a = executor.exceedance_ttc_noise(d[:cut], hz[:cut], TTC[::-1], 30.0, 0.2, noise_seed=11, first=0)
    b = executor.exceedance_ttc_noise(d[cut:], hz[cut:], TTC[::-1], 30.0, 0.2, noise_seed=11,
                                      first=cut)
    assert (a + b).tolist() == whole.tolist()


@pytest.mark.parametrize("sigma", [0.05, 0.3])
def test_sensor_noise_sweep_on_the_reference_normal_stream(ref, executor, mixed, sigma):
    # pins the noisy sweep to the REFERENCE itself, not only the C oracle:
    # eps_i = sigma * standard_normal_at(noise_seed, first + i) from the
    # unmodified reference (sampling.cpp:48-53 via oracle/_ref), then the
    # collision rule d > (T + eps_i) * v (IEEE, in the kernel's op order) and
    # horizon hits always colliding (analysis.cpp:152-157)
    n = 20000
    res = mixed[:n]
    first, seed, v = 4321, 0x5EED, 30.0
    z = np.array([ref.standard_normal_at(seed, first + i) for i in range(n)])
    eps = sigma * z
    d_host = res["stop_distance"]
    hz_host = res["hit_horizon"] != 0
    want = [int(np.count_nonzero(hz_host | (d_host > (t + eps) * v))) for t in TTC]
    d, hz = device(res)
    got = executor.exceedance_ttc_noise(d, hz, TTC, v, sigma, noise_seed=seed, first=first)
    assert got.tolist() == want
