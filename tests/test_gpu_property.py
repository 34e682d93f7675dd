"""Randomised parity: random SimConfig / VehicleGeometry / PhysicalConstants
and random uncertainty models (wide, clamping, horizon-heavy), CUDA executor
vs the reference library on identical samples, bit for bit.  Also the
device statistics on the same random results."""
import math

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import paper_2604_27193_b200 as bmc
from oracle.pyoracle import Model, World, results_bitwise_equal

pytestmark = pytest.mark.gpu

worlds = st.builds(
    World,
    dt=st.sampled_from([5e-4, 1e-3, 2e-3, 2.5e-3, 4e-3]),
    t_max=st.sampled_from([0.5, 2.0, 4.0, 10.0, 12.0]),
    brake_cmd=st.floats(-11.0, -1.0),
    cg_height=st.floats(0.2, 1.0),
    wheelbase=st.floats(2.0, 3.5),
    actuator_tau=st.floats(0.02, 0.8),
    gravity=st.floats(9.0, 10.5),
    air_density=st.floats(0.0, 1.6),
    frontal_area=st.floats(1.5, 3.5),
)

models = st.builds(
    lambda seed, v0, mu, th, m, cd: Model(seed=seed, mean=(v0[0], mu[0], th[0], m[0], cd[0]),
                                          sd=(v0[1], mu[1], th[1], m[1], cd[1])),
    st.integers(0, 2**63),
    st.tuples(st.floats(5.0, 45.0), st.floats(0.0, 8.0)),
    st.tuples(st.floats(0.06, 1.2), st.floats(0.0, 0.4)),
    st.tuples(st.floats(-0.2, 0.2), st.floats(0.0, 0.3)),
    st.tuples(st.floats(600.0, 3000.0), st.floats(0.0, 400.0)),
    st.tuples(st.floats(0.0, 0.6), st.floats(0.0, 0.2)),
)


@settings(max_examples=25, deadline=None, suppress_health_check=list(HealthCheck))
@given(w=worlds, m=models, n=st.integers(1, 3000))
def test_random_worlds_bit_exact(ref, executor, w, m, n):
    samples, _ = ref.draw_batch(m, n)
    want, _, _ = ref.run(samples, w, "parallel")
    sw = bmc.SimWorld(*w.as_array().tolist())
    got = executor.run(samples, sw).results
    assert results_bitwise_equal(want, got)
    v = ref.verify_consistency(want, got)
    assert v["passed"] and v["max_abs_deviation"] == 0.0


@settings(max_examples=15, deadline=None, suppress_health_check=list(HealthCheck))
@given(m=models, n=st.integers(2, 4000), bw=st.floats(0.25, 7.0))
def test_random_statistics(ref, executor, m, n, bw):
    import torch
    samples, _ = ref.draw_batch(m, n)
    res, _, _ = ref.run(samples, World(), "parallel")
    d = torch.from_numpy(np.ascontiguousarray(res["stop_distance"])).cuda()
    hz = torch.from_numpy(np.ascontiguousarray(res["hit_horizon"])).cuda()
    want = ref.summarize(res, bw)
    got = executor.summarize(d, hz, bw, hist_cap=1 << 20)
    for k in ("n", "horizon_count", "bins", "min", "max", "median", "origin"):
        assert got[k] == want[k], k
    assert np.array_equal(got["histogram"], want["histogram"])
    assert got["mean"] == pytest.approx(want["mean"], rel=1e-12)
    for risk in (0.5, 0.1, 0.01):
        a, b = executor.min_safe_headway(d, hz, risk), ref.min_safe_headway(res, risk)
        assert a == b or (math.isinf(a) and math.isinf(b))


# every rollout loop variant the planner can pick (chains per thread, block
# size, termination-test block, table placement) on random worlds / models
variants = st.sampled_from([
    dict(ilp=1, block_threads=1024, test_block=8), dict(ilp=1, block_threads=256, test_block=1),
    dict(ilp=2, block_threads=640, test_block=8), dict(ilp=2, block_threads=512, test_block=1),
    dict(ilp=2, block_threads=768, test_block=8, table="global"),
    dict(ilp=1, block_threads=512, test_block=8, table="global"),
])


@settings(max_examples=25, deadline=None, suppress_health_check=list(HealthCheck))
@given(w=worlds, m=models, n=st.integers(1, 5000), opts=variants)
def test_random_loop_variants_bit_exact(ref, executor, w, m, n, opts):
    samples, _ = ref.draw_batch(m, n)
    want, _, _ = ref.run(samples, w, "parallel")
    sw = bmc.SimWorld(*w.as_array().tolist())
    got = executor.run(samples, sw, **opts).results
    assert results_bitwise_equal(want, got), opts


@settings(max_examples=20, deadline=None, suppress_health_check=list(HealthCheck))
@given(m=models, first=st.integers(0, 2**40), n=st.integers(1, 20000))
def test_random_device_draws_bit_exact(executor, m, first, n):
    # the glibc-port device sampler vs the host pool (itself pinned to the
    # reference's draw_batch) on random models and index windows
    if not bmc.device_sampler_available():
        pytest.skip("device sampler gate closed on this host")
    model = bmc.UncertaintyModel(m.seed, *zip(m.mean, m.sd))
    terms, samples, clamps = executor.draw_device(model, n, first=first)
    host, hclamps = bmc.draw_batch(model, n, first=first)
    assert np.array_equal(samples.cpu().numpy().view(np.uint64),
                          np.ascontiguousarray(host).view(np.uint64).reshape(n, 5))
    assert clamps == hclamps
    assert np.array_equal(terms.cpu().numpy().view(np.uint64), bmc.stage_terms(host).view(np.uint64))


@settings(max_examples=20, deadline=None, suppress_health_check=list(HealthCheck))
@given(m=models, n=st.integers(1, 4000), sigma=st.floats(0.0, 3.0),
       seed=st.integers(0, 2**64 - 1), first=st.integers(0, 2**40),
       ttc=st.lists(st.floats(0.0, 8.0), min_size=1, max_size=40))
def test_random_sensor_noise_sweeps(ref, executor, m, n, sigma, seed, first, ttc):
    import torch
    from oracle.pyoracle import Port
    samples, _ = ref.draw_batch(m, n)
    res, _, _ = ref.run(samples, World(), "parallel")
    d = torch.from_numpy(np.ascontiguousarray(res["stop_distance"])).cuda()
    hz = torch.from_numpy(np.ascontiguousarray(res["hit_horizon"])).cuda()
    got = executor.exceedance_ttc_noise(d, hz, ttc, 27.5, sigma, seed, first)
    want = Port().exceed_ttc_noise(res, ttc, 27.5, sigma, seed, first)
    assert got.tolist() == want.tolist()
