"""Generate tests/golden/golden.json from the reference itself.

Runs the UNMODIFIED reference (oracle/_ref/libbrakemc_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile) and records:
  * the reference tests' own known-answer constants, re-derived
    (test_integrator.cpp:20, 46-58, 185-215, 238-248; test_dynamics.cpp:25-95);
  * sampler words / uniforms / deviates (sampling.cpp:36-53);
  * per-sample results (bits) for the first samples of seeds 1..3 and the
    mixed model, plus the nominal fixed sample;
  * summary / risk statistics at the README scenario (seed 3, n = 12000,
    README.md:165-171) -- integer and order-statistic outputs exactly.
Sampled-input goldens depend on glibc 2.39's libm (log/cos/sin) on an
FMA-capable x86 host; parity tests always re-run the oracle on
the same host and use these only as a pinned cross-check.

Usage: python tests/golden/make_golden.py  (needs oracle/_ref built)
"""
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.pyoracle import Model, Reference, World  # noqa: E402


def bits(x: float) -> str:
    return "0x%016x" % np.array([x], dtype=np.float64).view(np.uint64)[0]


def result_rec(r):
    return {"stop_distance": bits(r["stop_distance"]), "stop_time": bits(r["stop_time"]),
            "steps": int(r["steps"]), "hit_horizon": bool(r["hit_horizon"]),
            "stop_distance_value": float(r["stop_distance"])}


def main():
    ref = Reference()
    w = World()
    g = {"generator": "tests/golden/make_golden.py via oracle/_ref (reference sources)"}

    g["stream"] = [{"seed": s, "counter": c, "word": "0x%016x" % ref.stream_word(s, c),
                    "uniform": bits(ref.stream_uniform(s, c)),
                    "normal": bits(ref.standard_normal_at(s, c))}
                   for s in (1, 3, 42) for c in (0, 1, 2, 1234567)]

    nominal = (30.0, 0.8, 0.0, 1500.0, 0.3)
    g["nominal"] = {"sample": nominal, "result": result_rec(ref.simulate_rollout(nominal, w)),
                    "terms": [bits(x) for x in ref.rollout_terms(nominal, w)],
                    "fine_stop_distance": ref.oracle_stopping_distance(nominal, w, 1e-5)}
    # known-answer tests of the reference suite, re-derived
    ice = (30.0, 0.05, -0.3, 1500.0, 0.3)
    g["horizon_case"] = {"sample": ice, "result": result_rec(ref.simulate_rollout(ice, w))}
    inst = World(air_density=0.0, actuator_tau=1e-6, dt=1e-6)
    g["constant_decel_case"] = {"world": inst.as_array().tolist(), "sample": nominal,
                                "result": result_rec(ref.simulate_rollout(nominal, inst))}
    weak = (30.0, 0.5, 0.0, 1500.0, 0.3)
    g["weak_grip_case"] = {"sample": weak, "result": result_rec(ref.simulate_rollout(weak, w))}

    cases = []
    for name, model in [("seed1", Model(seed=1)), ("seed2", Model(seed=2)),
                        ("seed3", Model(seed=3)), ("mixed3", Model.mixed(3))]:
        samples, clamps = ref.draw_batch(model, 64)
        res, _, _ = ref.run(samples, w, "sequential")
        cases.append({"name": name, "seed": model.seed, "mean": model.mean, "sd": model.sd,
                      "clamp_count_64": clamps,
                      "samples": [[bits(v) for v in s.tolist()] for s in samples],
                      "results": [result_rec(r) for r in res]})
    g["batches"] = cases

    samples, _ = ref.draw_batch(Model(seed=3), 12000)
    res, _, _ = ref.run(samples, w, "parallel")
    sm = ref.summarize(res, 2.0)
    grid = ref.headway_grid(math.floor(sm["min"]) - 5.0, math.ceil(sm["max"]) + 5.0, 1.0)
    levels = [0.05, 0.01, 0.001]
    closing = 30.0
    probs, thr = ref.build_risk_curve(res, grid, levels, closing)
    g["readme_12000"] = {
        "summary": {k: (bits(v) if isinstance(v, float) else v) for k, v in sm.items()
                    if k != "histogram"},
        "summary_values": {k: v for k, v in sm.items() if isinstance(v, float)},
        "histogram": [int(x) for x in sm["histogram"]],
        "total_steps": int(res["steps"].sum()),
        "grid": [bits(x) for x in grid],
        "exceed_counts": [int(round(p * 12000)) for p in probs],
        "thresholds": [[bits(x) for x in row] for row in thr],
        "threshold_values": thr.tolist(),
    }
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
