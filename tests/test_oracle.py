"""Pins the oracle (CPU, no GPU needed).

The C restatement (oracle/bmc_oracle.c) must be bit-identical to the
reference library itself (oracle/_ref, compiled from /root/reference/proj/src)
on identical inputs, and both must reproduce the known-answer constants the
reference's own tests freeze and the committed golden vectors.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle.pyoracle import Model, World, results_bitwise_equal

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def f64(hexbits: str) -> float:
    return float(np.array([int(hexbits, 16)], dtype=np.uint64).view(np.float64)[0])


def bits(x: float) -> int:
    return int(np.array([x], dtype=np.float64).view(np.uint64)[0])


# ---------------------------------------------------------------- sampler

def test_stream_goldens(ref, port):
    for rec in GOLDEN["stream"]:
        s, c = rec["seed"], rec["counter"]
        assert port.stream_word(s, c) == int(rec["word"], 16) == ref.stream_word(s, c)
        assert bits(port.stream_uniform(s, c)) == int(rec["uniform"], 16)
        assert bits(port.standard_normal_at(s, c)) == int(rec["normal"], 16)
        assert bits(ref.standard_normal_at(s, c)) == int(rec["normal"], 16)


def test_survey_sampler_goldens(port):
    # SURVEY.md 8c golden vectors (seed 3)
    assert port.stream_word(3, 0) == 0x1D0B14E4DB018FED
    assert port.stream_uniform(3, 0) == 0.11345034205715454
    assert port.standard_normal_at(3, 0) == -0.64105156952623799


@pytest.mark.parametrize("model", [Model(seed=1), Model(seed=3), Model.mixed(7)])
def test_draw_matches_reference_and_shards(ref, port, model):
    full, clamps = ref.draw_batch(model, 3000)
    mine, c2 = port.draw_range(model, 0, 3000)
    assert np.array_equal(full.view(np.uint64), mine.view(np.uint64))
    assert clamps == c2
    # counter-based stream: any shard equals the slice (sampling.hpp:3-6)
    shard, _ = port.draw_range(model, 1234, 500)
    assert np.array_equal(full[1234:1734].view(np.uint64), shard.view(np.uint64))


def test_clamp_accounting(ref, port):
    wild = Model(seed=5, mean=(0.5, 0.06, 0.0, 600.0, 0.01), sd=(1.0, 0.05, 2.0, 200.0, 0.1))
    a, ca = ref.draw_batch(wild, 2000)
    b, cb = port.draw_range(wild, 0, 2000)
    assert ca == cb > 0
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert a["friction"].min() >= 0.05 and abs(a["grade"]).max() <= 1.5


# --------------------------------------------------------------- dynamics

def test_terms_match_reference(ref, port):
    samples, _ = ref.draw_batch(Model.mixed(11), 200)
    for s in samples:
        assert np.array_equal(ref.rollout_terms(s, World()).view(np.uint64),
                              port.rollout_terms(s, World()).view(np.uint64))
    nom = GOLDEN["nominal"]
    assert [bits(x) for x in port.rollout_terms(nom["sample"])] == [int(t, 16) for t in nom["terms"]]


def test_friction_limit_known_answers(port):
    # test_dynamics.cpp:25-39
    hi = port.rollout_terms((30.0, 0.8, 0.0, 1500.0, 0.3))[0]
    lo = port.rollout_terms((30.0, 0.5, 0.0, 1500.0, 0.3))[0]
    assert hi == pytest.approx(-6.8353, rel=1e-4)
    assert lo == pytest.approx(-4.4893, rel=1e-4)


# ------------------------------------------------------------- integrator

def test_nominal_known_answers(ref, port):
    nom = GOLDEN["nominal"]
    r = port.run(np.array([tuple(nom["sample"])], dtype=ref_dtype()))[0]
    assert bits(r["stop_distance"]) == int(nom["result"]["stop_distance"], 16)
    assert r["steps"] == nom["result"]["steps"] == 5079
    # test_integrator.cpp:20 (fine-step oracle value, frozen in the reference)
    fine = port.fine_stopping_distance(nom["sample"], World(), 1e-5)
    assert fine == pytest.approx(77.78395990740091, rel=1e-9)
    assert abs(r["stop_distance"] - fine) < 0.05
    assert ref.oracle_stopping_distance(nom["sample"]) == fine


def ref_dtype():
    from oracle.pyoracle import SAMPLE_DTYPE
    return SAMPLE_DTYPE


def test_horizon_known_answer(port):
    # test_integrator.cpp:238-248
    h = GOLDEN["horizon_case"]
    r = port.run(np.array([tuple(h["sample"])], dtype=ref_dtype()))[0]
    assert r["hit_horizon"] == 1 and r["steps"] == 10000 and r["stop_distance"] > 300.0
    assert bits(r["stop_distance"]) == int(h["result"]["stop_distance"], 16)
    assert r["stop_time"] == pytest.approx(10.0)


def test_constant_deceleration_known_answer(port):
    # test_integrator.cpp:106-119: 75 m within 0.01 m, 5 s
    c = GOLDEN["constant_decel_case"]
    w = World(*c["world"])
    r = port.run(np.array([tuple(c["sample"])], dtype=ref_dtype()), w)[0]
    assert r["stop_distance"] == pytest.approx(75.0, abs=0.01)
    assert r["stop_time"] == pytest.approx(5.0, rel=1e-3)
    assert bits(r["stop_distance"]) == int(c["result"]["stop_distance"], 16)
    assert r["steps"] == c["result"]["steps"]


def test_mu_threshold_flat_region(port):
    # test_integrator.cpp:185-215
    lo, hi = 0.1, 1.2
    for _ in range(100):
        mid = 0.5 * (lo + hi)
        if mid * 9.81 / (1.0 + mid * 0.5 / 2.7) < 6.0:
            lo = mid
        else:
            hi = mid
    thr = 0.5 * (lo + hi)
    assert thr == pytest.approx(0.6897432622301698, rel=1e-10)
    s = np.array([(30.0, thr + 0.01, 0.0, 1500.0, 0.3), (30.0, 1.2, 0.0, 1500.0, 0.3)],
                 dtype=ref_dtype())
    r = port.run(s)
    assert r[0]["stop_distance"] == r[1]["stop_distance"]


@pytest.mark.parametrize("name", ["seed1", "seed2", "seed3", "mixed3"])
def test_golden_batches(port, name):
    case = next(c for c in GOLDEN["batches"] if c["name"] == name)
    m = Model(seed=case["seed"], mean=tuple(case["mean"]), sd=tuple(case["sd"]))
    samples, _ = port.draw_range(m, 0, 64)
    want = np.array([[int(b, 16) for b in s] for s in case["samples"]], dtype=np.uint64)
    assert np.array_equal(samples.view(np.uint64).reshape(64, 5), want)
    res = port.run(samples)
    for r, g in zip(res, case["results"]):
        assert bits(r["stop_distance"]) == int(g["stop_distance"], 16)
        assert bits(r["stop_time"]) == int(g["stop_time"], 16)
        assert r["steps"] == g["steps"] and bool(r["hit_horizon"]) == g["hit_horizon"]


@pytest.mark.parametrize("model", [Model(seed=2), Model.mixed(5)])
def test_port_rollouts_match_reference(ref, port, model):
    samples, _ = ref.draw_batch(model, 1500)
    want, _, _ = ref.run(samples, World(), "sequential")
    got = port.run(samples, World(), threads=4)
    assert results_bitwise_equal(want, got)
    assert ref.verify_consistency(want, got)["passed"]


def test_port_nondefault_worlds(ref, port):
    samples, _ = ref.draw_batch(Model.mixed(9), 200)
    for w in [World(dt=0.002, t_max=6.0), World(actuator_tau=0.4, brake_cmd=-8.0),
              World(dt=0.0005, t_max=3.0, gravity=9.7, air_density=1.1)]:
        want, _, _ = ref.run(samples, w, "sequential")
        assert results_bitwise_equal(want, port.run(samples, w))


# ------------------------------------------------------------- statistics

def test_readme_statistics(ref, port):
    g = GOLDEN["readme_12000"]
    samples, _ = port.draw_range(Model(seed=3), 0, 12000)
    res = port.run(samples, World(), threads=8)
    assert int(res["steps"].sum()) == g["total_steps"]
    sm = port.summarize(res)
    for k in ("mean", "sd", "min", "max", "median", "skewness", "origin"):
        assert bits(sm[k]) == int(g["summary"][k], 16), k
    assert [int(x) for x in sm["histogram"]] == g["histogram"]
    # README.md:165-171: mean ~79.3, sd ~12.2, 100.7 / 111.7 / 123.8 m
    assert sm["mean"] == pytest.approx(79.3, abs=0.1) and sm["sd"] == pytest.approx(12.2, abs=0.1)
    grid = [f64(x) for x in g["grid"]]
    assert np.array_equal(port.headway_grid(grid[0], grid[-1], 1.0), np.array(grid))
    assert [port.exceed_count(res, h) for h in grid] == g["exceed_counts"]
    for row in g["thresholds"]:
        risk = f64(row[0])
        assert bits(port.min_safe_headway(res, risk)) == int(row[1], 16)


def test_min_safe_headway_with_horizons(ref, port):
    from oracle.pyoracle import RESULT_DTYPE
    d = [60, 65, 70, 75, 80, 85, 90, 95, 400, 410]
    res = np.zeros(10, dtype=RESULT_DTYPE)
    res["stop_distance"] = d
    res["hit_horizon"][8:] = 1
    # test_analysis.cpp:179-191
    assert port.min_safe_headway(res, 0.1) == math.inf == ref.min_safe_headway(res, 0.1)
    assert port.min_safe_headway(res, 0.2) == 95.0 == ref.min_safe_headway(res, 0.2)
    assert port.exceed_count(res, 1e9) == 2


TTC = [1.0 + 0.25 * k for k in range(21)]


def test_sensor_noise_ttc_oracle(ref, port):
    # the C4 extension's oracle: sigma = 0 is the reference's own
    # collision_probability at T * v; sigma > 0 follows the reference's
    # standard_normal_at on the noise stream sample by sample
    samples, _ = ref.draw_batch(Model.mixed(8), 3000)
    res, _, _ = ref.run(samples, World(), "parallel")
    v = 30.0
    zero = port.exceed_ttc_noise(res, TTC, v, 0.0, noise_seed=99, first=0)
    want = [int(round(ref.collision_probability(res, t * v) * len(res))) for t in TTC]
    assert zero.tolist() == want
    seed, first, sigma = 0xABCDEF, 123456, 0.3
    got = port.exceed_ttc_noise(res, TTC, v, sigma, noise_seed=seed, first=first)
    eps = [sigma * ref.standard_normal_at(seed, first + i) for i in range(len(res))]
    brute = [sum(1 for i in range(len(res))
                 if res["hit_horizon"][i] or res["stop_distance"][i] > (t + eps[i]) * v)
             for t in TTC]
    assert got.tolist() == brute
    assert got.tolist() != zero.tolist()
