"""CPU-side checks of the product library (no GPU required).

* libbrakemc_b200.so loads and exports every entry point include/brakemc_cuda.h
  declares;
* the host producers inside it (sampler shard + RolloutTerms staging) are
  bit-identical to the reference on identical inputs;
* without a device the compute entry points fail loudly (no CPU fallback).
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2604_27193_b200 as bmc
from paper_2604_27193_b200 import _native as N
from oracle.pyoracle import Model, World

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "brakemc_cuda.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bmc_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = N.load()
    names = declared_symbols()
    assert len(names) >= 17
    for name in names:
        assert hasattr(lib, name), name
    assert {n for n, _, _ in N.SIGNATURES} == set(names)
    assert lib.bmc_abi_version() == 1


def test_cpp_executor_header_declares_run_cuda():
    hpp = open(os.path.join(ROOT, "include", "brakemc", "cuda_executor.hpp")).read()
    assert "ExecutionReport run_cuda(" in hpp


def to_model(m: Model) -> bmc.UncertaintyModel:
    return bmc.UncertaintyModel(m.seed, *zip(m.mean, m.sd))


@pytest.mark.parametrize("model", [Model(seed=3), Model.mixed(4)])
@pytest.mark.parametrize("threads", [1, 3, 0])
def test_host_sampler_matches_reference(ref, model, threads):
    want, clamps = ref.draw_batch(model, 4000)
    got, c2 = bmc.draw_batch(to_model(model), 4000, threads=threads)
    assert np.array_equal(want.view(np.uint64), got.view(np.uint64))
    assert clamps == c2
    shard, _ = bmc.draw_batch(to_model(model), 777, first=1500, threads=threads)
    assert np.array_equal(want[1500:2277].view(np.uint64), shard.view(np.uint64))


def test_sampler_rejects_empty():
    with pytest.raises(bmc.ConfigError, match="samples: must be >= 1"):
        bmc.draw_batch(bmc.UncertaintyModel(), 0)


def test_stage_terms_match_reference(ref):
    samples, _ = ref.draw_batch(Model.mixed(21), 500)
    for w in (World(), World(gravity=9.7, air_density=1.3, frontal_area=2.5)):
        sw = bmc.SimWorld(*w.as_array().tolist())
        terms = bmc.stage_terms(samples, sw, threads=4)
        for i in range(0, 500, 37):
            t = ref.rollout_terms(samples[i], w)
            got = np.array([terms[1, i], terms[2, i], terms[3, i]])
            assert np.array_equal(got.view(np.uint64), t[:3].view(np.uint64))
            assert terms[0, i] == samples[i]["initial_speed"]


def test_stage_terms_domain_error():
    s = np.zeros(1, dtype=bmc.SAMPLE_DTYPE)
    s[0] = (30.0, 0.8, 0.0, 1500.0, 0.3)
    with pytest.raises(bmc.DomainError):
        bmc.stage_terms(s, bmc.SimWorld(wheelbase=-0.1))


def test_results_csv_matches_reference_io(ref, tmp_path):
    """results.csv (io.cpp:17-31) byte-identical; parse (io.cpp:94-123) + step
    rebuild (cli.cpp:96-100) round-trips every field bit for bit."""
    from oracle.pyoracle import results_bitwise_equal
    samples, _ = ref.draw_batch(Model.mixed(3), 2500)
    res, _, _ = ref.run(samples, World(), "parallel")
    mine, theirs = str(tmp_path / "mine.csv"), str(tmp_path / "ref.csv")
    bmc.engine.write_results_csv(mine, res, threads=3)
    ref.write_results_csv(res, theirs)
    assert open(mine, "rb").read() == open(theirs, "rb").read()
    assert results_bitwise_equal(bmc.engine.read_results_csv(theirs, 0.001), res)
    assert results_bitwise_equal(ref.read_results_csv(mine, 0.001), res)
    bad = tmp_path / "bad.csv"
    bad.write_text("index,d,t,h\n0,1,2,0\n")
    with pytest.raises(bmc.BmcError, match="unexpected header"):
        bmc.engine.read_results_csv(str(bad), 0.001)
    gap = tmp_path / "gap.csv"
    gap.write_text("index,d_stop_m,t_stop_s,horizon_flag\n0,1,2,0\n2,1,2,0\n")
    with pytest.raises(bmc.BmcError, match="non-contiguous"):
        bmc.engine.read_results_csv(str(gap), 0.001)


def test_no_cpu_fallback_without_device():
    if bmc.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(bmc.CudaError):
        bmc.CudaExecutor(0)


def test_cpp_statistics_merge_fake_collective():
    """C++ CPU test (tests/cpp/merge_main.cpp): the statistics stage's merge
    orchestration over brakemc::Collective with an in-process fake, worlds
    1/2/3, against the reference's analysis functions (built here when the
    reference tree is present)."""
    import subprocess
    exe = os.path.join(ROOT, "build", "merge_cpp")
    if not os.path.exists(exe):
        pytest.skip("build/merge_cpp not built (needs the reference headers)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
