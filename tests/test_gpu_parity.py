"""GPU parity: the CUDA executor vs the reference, bit for bit.

Every test calls the product through the C-ABI (libbrakemc_b200.so) and
compares with the reference library (oracle/_ref) run on the SAME samples on
the same host, so glibc-libm variance cannot leak in.  Bar: bitwise equality
of all four RolloutResult fields (backends.cpp:24-30), i.e. the reference's
verify_consistency verdict `pass` with max_abs_deviation == 0.0.
"""
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2604_27193_b200 as bmc
from oracle.pyoracle import Model, World, results_bitwise_equal

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def to_model(m: Model) -> bmc.UncertaintyModel:
    return bmc.UncertaintyModel(m.seed, *zip(m.mean, m.sd))


def to_world(w: World) -> bmc.SimWorld:
    return bmc.SimWorld(*w.as_array().tolist())


def assert_parity(ref, want, got):
    v = ref.verify_consistency(want, got)
    assert v["passed"] and v["max_abs_deviation"] == 0.0, v
    assert results_bitwise_equal(want, got)


# acceptance_main.cpp:65-107 -- criterion 1 matrix
@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("n", [1000, 12000, 100000])
def test_criterion1_matrix(ref, executor, seed, n):
    samples, _ = ref.draw_batch(Model(seed=seed), n)
    want, _, _ = ref.run(samples, World(), "parallel")
    rep = executor.run(samples)
    assert_parity(ref, want, rep.results)
    assert rep.total_steps == int(want["steps"].sum())


def test_large_batch_default_plan(ref, executor):
    # >= 2^20 samples per launch: the planner's two-chains-per-thread rollout
    n = (1 << 20) + 12345
    samples, _ = ref.draw_batch(Model.mixed(41), n)
    want, _, _ = ref.run(samples, World(), "parallel")
    import torch
    terms = bmc.stage_terms(samples)
    dev = [torch.from_numpy(terms[i]).cuda() for i in range(4)]
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.empty(n, dtype=torch.int32, device="cuda")
    hz = torch.empty(n, dtype=torch.uint8, device="cuda")
    executor.rollout_device(dev, (d, st, hz))
    executor.sync()
    assert np.array_equal(d.cpu().numpy().view(np.uint64), want["stop_distance"].view(np.uint64))
    assert np.array_equal(st.cpu().numpy(), want["steps"].astype(np.int32))
    assert np.array_equal(hz.cpu().numpy(), want["hit_horizon"].astype(np.uint8))


def test_mixed_model_with_horizons(ref, executor):
    samples, _ = ref.draw_batch(Model.mixed(3), 100000)
    want, _, _ = ref.run(samples, World(), "parallel")
    assert want["hit_horizon"].mean() > 0.2  # divergence-heavy: ~27% horizon
    rep = executor.run(samples)
    assert_parity(ref, want, rep.results)


@pytest.mark.parametrize("schedule", ["index", "binned"])
@pytest.mark.parametrize("table", ["shared", "global", "none"])
@pytest.mark.parametrize("block", [256, 512, 1024])
def test_scheduling_knobs_never_change_bits(ref, executor, schedule, table, block):
    samples, _ = ref.draw_batch(Model.mixed(17), 6000)
    want, _, _ = ref.run(samples, World(), "parallel")
    rep = executor.run(samples, schedule=schedule, table=table, block_threads=block,
                       chunk=2500)
    assert_parity(ref, want, rep.results)


@pytest.mark.parametrize("ilp,block,tb", [(1, 1024, 1), (1, 768, 1), (2, 640, 1), (2, 512, 1),
                                          (1, 1024, 8), (1, 512, 8), (2, 640, 8), (2, 768, 8)])
@pytest.mark.parametrize("table", ["shared", "global"])
@pytest.mark.parametrize("w", [World(), World(t_max=3.0), World(actuator_tau=30.0),
                               World(t_max=0.0005), World(t_max=0.003)],
                         ids=["default", "tmax3", "tau30", "one_step", "three_steps"])
def test_loop_variants_never_change_bits(ref, executor, ilp, block, tb, table, w):
    # odd/even step counts, stops inside each warp-uniform phase, horizons
    samples, _ = ref.draw_batch(Model.mixed(29), 5000)
    want, _, _ = ref.run(samples, w, "parallel")
    rep = executor.run(samples, to_world(w), table=table, block_threads=block, ilp=ilp,
                       test_block=tb)
    assert_parity(ref, want, rep.results)


# Grades around the point where the final brake just holds the car (F ~ G):
# warps mix chains whose every stage acceleration is <= 0 (blocks past
# monotone_from test only their last speed) with chains that never get there,
# plus near-zero initial speeds that stop inside the first block.
BOUNDARY_MODELS = [
    Model(seed=41, mean=(12.0, 0.12, 0.10, 1500.0, 0.3), sd=(6.0, 0.06, 0.08, 300.0, 0.1)),
    Model(seed=42, mean=(25.0, 0.10, -0.10, 1500.0, 0.3), sd=(8.0, 0.05, 0.10, 300.0, 0.1)),
    Model(seed=43, mean=(0.3, 0.8, 0.0, 1500.0, 0.3), sd=(0.4, 0.2, 0.2, 100.0, 0.05)),
]


@pytest.mark.parametrize("m", BOUNDARY_MODELS, ids=["uphill", "downhill", "slow"])
@pytest.mark.parametrize("ilp,block,tb,table", [(2, 640, 8, "shared"), (2, 768, 8, "global"),
                                                (1, 1024, 8, "shared")])
@pytest.mark.parametrize("w", [World(), World(t_max=2.0, actuator_tau=0.5)], ids=["default", "short"])
def test_monotone_blocks_at_the_holding_boundary(ref, executor, m, ilp, block, tb, table, w):
    samples, _ = ref.draw_batch(m, 6000)
    want, _, _ = ref.run(samples, w, "parallel")
    rep = executor.run(samples, to_world(w), table=table, block_threads=block, ilp=ilp,
                       test_block=tb)
    assert_parity(ref, want, rep.results)


def test_monotone_blocks_equal_per_step_test():
    """The last-speed-only block test vs the per-step running minimum
    (BMC_PER_STEP_TEST=1, a separate process: the switch is read once)."""
    code = (
        "import hashlib, sys; sys.path.insert(0, %r)\n"
        "import paper_2604_27193_b200 as bmc\n"
        "ex = bmc.CudaExecutor(0)\n"
        "h = hashlib.sha256()\n"
        "for mdl in (bmc.UncertaintyModel.mixed(7), bmc.UncertaintyModel(seed=9)):\n"
        "    s, _ = bmc.draw_batch(mdl, 300000)\n"
        "    for t in ('shared', 'global'):\n"
        "        h.update(ex.run(s, table=t).results.tobytes())\n"
        "print(h.hexdigest())\n" % ROOT)
    outs = []
    for env in ({}, {"BMC_PER_STEP_TEST": "1"}):
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                           env={**os.environ, **env})
        assert p.returncode == 0, p.stderr
        outs.append(p.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1]


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 257])
def test_ragged_sizes(ref, executor, n):
    samples, _ = ref.draw_batch(Model.mixed(n), n)
    want, _, _ = ref.run(samples, World(), "sequential")
    assert_parity(ref, want, executor.run(samples).results)


def test_empty_batch_is_config_error(executor):
    with pytest.raises(bmc.ConfigError, match="batch: must be non-empty"):
        executor.run(np.zeros(0, dtype=bmc.SAMPLE_DTYPE))


def test_domain_error(executor):
    s = np.zeros(1, dtype=bmc.SAMPLE_DTYPE)
    s[0] = (30.0, 0.8, 0.0, 1500.0, 0.3)
    with pytest.raises(bmc.DomainError):
        executor.run(s, bmc.SimWorld(wheelbase=-0.2))


WORLDS = [
    World(t_max=3.0),                               # horizon before the actuator fixed point
    World(dt=0.002, brake_cmd=-8.0),
    World(actuator_tau=0.4),
    World(actuator_tau=30.0),                       # no fixed point inside the horizon
    World(dt=0.0005, t_max=6.0, gravity=9.7, air_density=1.1, frontal_area=2.6),
    World(t_max=0.0005),                            # llround(0.5) = 1 step
    World(t_max=0.0),                               # zero steps: all horizon
]


@pytest.mark.parametrize("w", WORLDS, ids=lambda w: f"dt{w.dt}_tmax{w.t_max}_tau{w.actuator_tau}")
def test_nondefault_worlds(ref, executor, w):
    samples, _ = ref.draw_batch(Model.mixed(23), 3000)
    want, _, _ = ref.run(samples, w, "parallel")
    assert_parity(ref, want, executor.run(samples, to_world(w)).results)


def test_known_answer_cases(ref, executor):
    # test_integrator.cpp: nominal (5079 steps), weak grip, glare ice horizon,
    # mu threshold flat region, extreme clamps
    rows = [(30.0, 0.8, 0.0, 1500.0, 0.3), (30.0, 0.5, 0.0, 1500.0, 0.3),
            (30.0, 0.05, -0.3, 1500.0, 0.3), (30.0, 0.6997432622301698, 0.0, 1500.0, 0.3),
            (30.0, 1.2, 0.0, 1500.0, 0.3), (0.1, 0.05, 1.5, 500.0, 0.0),
            (45.0, 0.05, -1.5, 500.0, 0.6), (0.1, 3.0, 0.0, 4000.0, 0.0)]
    s = np.array(rows, dtype=bmc.SAMPLE_DTYPE)
    want, _, _ = ref.run(s, World(), "sequential")
    got = executor.run(s).results
    assert_parity(ref, want, got)
    assert got[0]["steps"] == 5079 and got[2]["hit_horizon"] == 1
    assert got[3]["stop_distance"] == got[4]["stop_distance"]


def test_constant_deceleration_long_rollout(ref, executor):
    # test_integrator.cpp:106-119: dt = tau = 1e-6, 5,000,002 steps
    w = World(air_density=0.0, actuator_tau=1e-6, dt=1e-6)
    s = np.array([(30.0, 0.8, 0.0, 1500.0, 0.3)], dtype=bmc.SAMPLE_DTYPE)
    want, _, _ = ref.run(s, w, "sequential")
    got = executor.run(s, to_world(w)).results
    assert_parity(ref, want, got)
    assert got[0]["stop_distance"] == pytest.approx(75.0, abs=0.01)


def test_host_sampler_feeds_gpu(ref, executor):
    # product sampler (host pool) -> GPU == reference sampler -> reference
    mine, _ = bmc.draw_batch(bmc.UncertaintyModel(seed=9), 20000)
    theirs, _ = ref.draw_batch(Model(seed=9), 20000)
    assert np.array_equal(mine.view(np.uint64), theirs.view(np.uint64))
    want, _, _ = ref.run(theirs, World(), "parallel")
    assert_parity(ref, want, executor.run(mine).results)


def test_device_resident_path(ref, executor):
    import torch
    samples, _ = ref.draw_batch(Model.mixed(31), 50000)
    want, _, _ = ref.run(samples, World(), "parallel")
    terms = bmc.stage_terms(samples)
    dev = [torch.from_numpy(terms[i].copy()).cuda() for i in range(4)]
    n = samples.shape[0]
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.empty(n, dtype=torch.int32, device="cuda")
    hz = torch.empty(n, dtype=torch.uint8, device="cuda")
    total = torch.zeros(1, dtype=torch.int64, device="cuda")
    executor.rollout_device(dev, (d, st, hz), total_steps=total)
    executor.sync()
    assert np.array_equal(d.cpu().numpy().view(np.uint64), want["stop_distance"].view(np.uint64))
    assert np.array_equal(st.cpu().numpy().astype(np.int64), want["steps"])
    assert np.array_equal(hz.cpu().numpy(), want["hit_horizon"])
    assert int(total.item()) == int(want["steps"].sum())
    rms, pms = executor.last_kernel_ms()
    assert rms > 0.0
    # predict, scan, scatter, rollout, unpermute (BMC_DIRECT_OUTPUTS=1: the
    # rollout writes each sample's outputs at its index, no unpermute pass)
    assert executor.last_launches() == (4 if os.environ.get("BMC_DIRECT_OUTPUTS") == "1" else 5)


def test_cpp_executor_api():
    """The reference's own C++ parity checks through brakemc::run_cuda."""
    exe = os.path.join(ROOT, "build", "parity_cpp")
    assert os.path.exists(exe), "build/parity_cpp missing (built by __graft_entry__.build())"
    p = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr


def test_reference_dispatch_sites_patched_for_cuda():
    """INTEGRATION.md's edits applied to a copy of the reference's own
    dispatch sites (tools/integrate_reference.py): config_from_json "cuda",
    run_configured_executor's body, convergence_table and
    max_samples_within_budget run the B200 executor; "gpu" still throws."""
    exe = os.path.join(ROOT, "build", "integration_test")
    assert os.path.exists(exe), "build/integration_test missing (built by __graft_entry__.build())"
    p = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert p.stdout.count("[PASS]") == 5


# ------------------------------------------------ streaming / real-time modes

@pytest.mark.parametrize("first,n", [(0, 20000), (123457, 9001)])
def test_run_model_matches_reference(ref, executor, first, n):
    """Sampler fused into the pipeline: samples [first, first+n) of the
    counter-based stream, never materialised as AoS."""
    m = Model.mixed(13)
    full, _ = ref.draw_batch(m, first + n)
    want, _, _ = ref.run(full[first:], World(), "parallel")
    rep, clamps = executor.run_model(to_model(m), n, first=first, chunk=4096)
    assert_parity(ref, want, rep.results)
    _, ref_clamps_prefix = ref.draw_batch(m, first) if first else (None, 0)
    assert clamps == ref.draw_batch(m, first + n)[1] - ref_clamps_prefix
    assert rep.chunks == (n + 4095) // 4096


def test_run_model_device_outputs(ref, executor):
    import torch
    n = 30000
    m = Model(seed=4)
    samples, _ = ref.draw_batch(m, n)
    want, _, _ = ref.run(samples, World(), "parallel")
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.empty(n, dtype=torch.int32, device="cuda")
    hz = torch.empty(n, dtype=torch.uint8, device="cuda")
    rep, _ = executor.run_model(to_model(m), n, device_out=(d, st, hz), chunk=7000)
    assert rep.results is None and rep.d2h_bytes == 0
    assert np.array_equal(d.cpu().numpy().view(np.uint64), want["stop_distance"].view(np.uint64))
    assert np.array_equal(st.cpu().numpy().astype(np.int64), want["steps"])
    assert np.array_equal(hz.cpu().numpy(), want["hit_horizon"])


def test_graph_mode_decisions(ref, executor):
    g = executor.graph(25000)
    try:
        for seed in (1, 2):
            s, _ = ref.draw_batch(Model(seed=seed), 25000)
            want, _, _ = ref.run(s, World(), "parallel")
            rep = g.run(s)
            assert_parity(ref, want, rep.results)
            assert rep.total_steps == int(want["steps"].sum())
        # sampling inside the decision (feasibility convention)
        rep = g.run_model(to_model(Model(seed=5)))
        s, _ = ref.draw_batch(Model(seed=5), 25000)
        want, _, _ = ref.run(s, World(), "parallel")
        assert_parity(ref, want, rep.results)
        # an unrelated larger call must not disturb the graph's buffers
        big, _ = ref.draw_batch(Model.mixed(2), 50000)
        executor.run(big, bmc.SimWorld(actuator_tau=0.3))
        assert_parity(ref, want, g.run(s).results)
    finally:
        g.close()


def test_verify_against_csv_flow(ref, executor, tmp_path):
    """cmd_verify --against (cli.cpp:82-116): CUDA results written as the
    reference's results.csv, parsed by the reference, steps rebuilt, then
    verify_consistency against run_sequential -> PASS."""
    samples, _ = ref.draw_batch(Model(seed=3), 12000)
    gpu = executor.run(samples).results
    path = str(tmp_path / "results.csv")
    bmc.engine.write_results_csv(path, gpu)
    back = ref.read_results_csv(path, 0.001)
    seq, _, _ = ref.run(samples, World(), "sequential")
    assert_parity(ref, seq, back)


def test_feasibility_search_logic():
    # analysis.cpp:258-318 with the reference test's synthetic linear machine
    # t(n) = 0.01 + 1e-6 n (test_analysis.cpp:235-266)
    n, capped = bmc.engine.max_feasible_n(lambda k: 0.01 + 1e-6 * k, 0.53, 1000, 1 << 22)
    assert not capped and abs(n - 520000) <= 520000 // 64 + 1
    n, capped = bmc.engine.max_feasible_n(lambda k: 0.0, 0.53, 1000, 4096)
    assert capped and n == 4096
    assert bmc.engine.max_feasible_n(lambda k: 1.0, 0.53, 1000, 4096) == (0, False)


def test_interleaved_worlds_never_rewrite_a_table_in_flight(ref, executor):
    """a device-resident rollout for world A, then -- before
    any synchronisation -- one for world B with a different actuator table.
    Tables are immutable per-world cache entries, so A's in-flight kernel
    keeps reading A's table; both results equal the reference."""
    import torch
    wa, wb = World(), World(actuator_tau=0.4, t_max=8.0)
    sa, _ = ref.draw_batch(Model(seed=41), 300000)
    sb, _ = ref.draw_batch(Model(seed=42), 4000)
    want_a, _, _ = ref.run(sa, wa, "parallel")
    want_b, _, _ = ref.run(sb, wb, "parallel")

    def dev(samples, w):
        t = bmc.stage_terms(samples, to_world(w))
        n = samples.shape[0]
        return ([torch.from_numpy(t[i]).cuda() for i in range(4)],
                (torch.empty(n, dtype=torch.float64, device="cuda"),
                 torch.empty(n, dtype=torch.int32, device="cuda"),
                 torch.empty(n, dtype=torch.uint8, device="cuda")))

    ta, oa = dev(sa, wa)
    tb, ob = dev(sb, wb)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    executor.rollout_device(ta, oa, to_world(wa), stream=s1)   # long, in flight
    executor.rollout_device(tb, ob, to_world(wb), stream=s2)   # new world, no sync
    for _ in range(3):                                         # churn the table cache
        executor.rollout_device(tb, ob, to_world(World(actuator_tau=0.1 + 0.05 * _)), stream=s2)
    executor.rollout_device(tb, ob, to_world(wb), stream=s2)
    torch.cuda.synchronize()
    assert np.array_equal(oa[0].cpu().numpy().view(np.uint64), want_a["stop_distance"].view(np.uint64))
    assert np.array_equal(ob[0].cpu().numpy().view(np.uint64), want_b["stop_distance"].view(np.uint64))


_PIPE_DIGEST = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_2604_27193_b200 as bmc
samples, _ = bmc.draw_batch(bmc.UncertaintyModel.mixed(23), 50000)
ex = bmc.CudaExecutor(0)
rep = ex.run(samples, chunk=6000)          # 9 chunks: three slots wrap three times
r = rep.results
h = hashlib.sha256()
for f in ("stop_distance", "steps", "hit_horizon"):
    h.update(np.ascontiguousarray(r[f]).tobytes())
print(rep.chunks, rep.launches, h.hexdigest())
"""


def test_pipeline_output_paths_identical(ref):
    """The streamed pipeline writes chunk outputs directly at each sample's
    index (forward map); BMC_DIRECT_OUTPUTS=0 forces the packed-record +
    unpermute path.  Both -- and the reference -- give the same bits.  (The
    switch is read once per process, hence the subprocesses.)"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for mode in ("1", "0"):
        env = dict(os.environ, BMC_DIRECT_OUTPUTS=mode)
        p = subprocess.run([sys.executable, "-c", _PIPE_DIGEST.format(root=root)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        chunks, launches, digest = p.stdout.split()[-3:]
        outs[mode] = (int(chunks), int(launches), digest)
    assert outs["1"][0] == outs["0"][0] == 9
    # per chunk: predict, scan, scatter, rollout (+ unpermute on the packed path)
    assert outs["1"][1] == 9 * 4 and outs["0"][1] == 9 * 5
    assert outs["1"][2] == outs["0"][2]
    samples, _ = ref.draw_batch(Model.mixed(23), 50000)
    want, _, _ = ref.run(samples, World(), "parallel")
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(want["stop_distance"]).tobytes())
    h.update(np.ascontiguousarray(want["steps"].astype(np.int64)).tobytes())
    h.update(np.ascontiguousarray(want["hit_horizon"].astype(np.uint8)).tobytes())
    assert outs["1"][2] == h.hexdigest()
