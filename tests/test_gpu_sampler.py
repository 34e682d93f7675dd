"""GPU parity of the on-device sampler (csrc/bmc_sampler.cu + bmc_libm.h).

draw_batch (sampling.cpp:67-100) and RolloutTerms::from (dynamics.cpp:57-68)
run on the B200 through the op-for-op port of glibc's FMA libm variants; the
bar is bitwise equality with the reference library (oracle/_ref) drawing the
same indices on the same host, including the clamp count.  Model-driven runs
(run_model, decision graphs) must give identical results whichever sampler
fed them.
"""
import math

import numpy as np
import pytest

import paper_2604_27193_b200 as bmc
from oracle.pyoracle import Model, World, results_bitwise_equal

pytestmark = pytest.mark.gpu


def to_model(m: Model) -> bmc.UncertaintyModel:
    return bmc.UncertaintyModel(m.seed, *zip(m.mean, m.sd))


def to_world(w: World) -> bmc.SimWorld:
    return bmc.SimWorld(*w.as_array().tolist())


MODELS = [
    Model(seed=3),                                                   # C1/C5 default
    Model.mixed(4),                                                  # C4 wet/icy, +-6 % grade
    # every clamp fires: v0 < 0.1, mu < 0.05, m < 500, c_d < 0, |grade| > 1.5
    Model(seed=77, mean=(2.0, 0.1, 0.0, 600.0, 0.05), sd=(3.0, 0.2, 1.2, 300.0, 0.1)),
    Model(seed=2**64 - 5, mean=(30.0, 0.8, 0.3, 1500.0, 0.3), sd=(2.0, 0.1, 0.5, 100.0, 0.05)),
]


def as_u64(x):
    return np.ascontiguousarray(x).view(np.uint64)


@pytest.mark.parametrize("m", MODELS, ids=["default", "mixed", "clamps", "bigseed"])
@pytest.mark.parametrize("first,n", [(0, 200000), (987654321, 65537)])
def test_device_draw_equals_reference(ref, executor, m, first, n):
    terms, samples, clamps = executor.draw_device(to_model(m), n, first=first)
    # product host pool (itself pinned to the reference's prefix slices in
    # tests/test_native_cpu.py); the reference draws from index 0 only
    host, hclamps = bmc.draw_batch(to_model(m), n, first=first)
    if first == 0:
        want, wclamps = ref.draw_batch(m, n)                          # the reference itself
        assert np.array_equal(as_u64(want), as_u64(host)) and wclamps == hclamps
    got = samples.cpu().numpy()
    assert np.array_equal(as_u64(got), as_u64(host).reshape(n, 5))
    assert clamps == hclamps
    want_terms = bmc.stage_terms(host)
    assert np.array_equal(as_u64(terms.cpu().numpy()), as_u64(want_terms))
    if m.seed == 77:
        assert clamps > 0.05 * n


def test_device_terms_match_reference_rollout_terms(ref, executor):
    m = Model.mixed(21)
    for w in (World(), World(gravity=9.7, air_density=1.3, frontal_area=2.5, cg_height=0.6)):
        terms, _, _ = executor.draw_device(to_model(m), 3000, world=to_world(w), samples=False)
        t = terms.cpu().numpy()
        samples, _ = ref.draw_batch(m, 3000)
        for i in range(0, 3000, 41):
            r = ref.rollout_terms(samples[i], w)
            assert np.array_equal(as_u64(t[1:, i]), as_u64(r[:3])), i


def test_device_draw_domain_error(executor):
    with pytest.raises(bmc.DomainError):
        executor.draw_device(bmc.UncertaintyModel(), 1000, world=bmc.SimWorld(wheelbase=-0.2))
    with pytest.raises(bmc.ConfigError, match="samples: must be >= 1"):
        executor.draw_device(bmc.UncertaintyModel(), 0)


@pytest.mark.parametrize("sampler", ["host", "device"])
@pytest.mark.parametrize("first,n", [(0, 20000), (123457, 9001)])
def test_run_model_either_sampler_matches_reference(ref, executor, sampler, first, n):
    m = Model.mixed(13)
    full, _ = ref.draw_batch(m, first + n)
    want, _, _ = ref.run(full[first:], World(), "parallel")
    rep, clamps = executor.run_model(to_model(m), n, first=first, chunk=4096, sampler=sampler)
    v = ref.verify_consistency(want, rep.results)
    assert v["passed"] and v["max_abs_deviation"] == 0.0, v
    prefix = ref.draw_batch(m, first)[1] if first else 0
    assert clamps == ref.draw_batch(m, first + n)[1] - prefix
    assert rep.h2d_bytes == (0 if sampler == "device" else 32 * n)


def test_run_model_device_sampler_stats_only(executor):
    import torch
    n = 1_000_003
    outs = []
    for sampler in ("host", "device"):
        d = torch.empty(n, dtype=torch.float64, device="cuda")
        st = torch.empty(n, dtype=torch.int32, device="cuda")
        hz = torch.empty(n, dtype=torch.uint8, device="cuda")
        rep, clamps = executor.run_model(bmc.UncertaintyModel(seed=8), n, first=5 * 10**8,
                                         device_out=(d, st, hz), sampler=sampler)
        outs.append((d, st, hz, clamps, rep.total_steps))
    (a, b) = outs
    assert torch.equal(a[0].view(torch.int64), b[0].view(torch.int64))
    assert torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    assert a[3] == b[3] and a[4] == b[4]


def test_graph_decisions_on_device_sampler(ref, executor):
    for sampler in ("device", "host"):
        g = executor.graph(25000, sampler=sampler)
        try:
            for seed, first in ((5, 0), (6, 10**9)):
                rep = g.run_model(to_model(Model(seed=seed)), first=first)
                s, _ = bmc.draw_batch(to_model(Model(seed=seed)), 25000, first=first)
                want, _, _ = ref.run(s, World(), "parallel")
                assert results_bitwise_equal(want, rep.results)
                assert rep.h2d_bytes == (96 if sampler == "device" else 32 * 25000)
        finally:
            g.close()


def test_forced_device_sampler_reports_availability(executor):
    assert bmc.device_sampler_available()
    rep, _ = executor.run_model(bmc.UncertaintyModel(), 1000, sampler="device")
    assert rep.results.shape[0] == 1000
