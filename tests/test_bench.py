"""bench.py contract checks (small sizes).

CPU: the reference arm prints one JSON line with impl=reference.
GPU: the B200 arm at N=1, and a 2-rank torchrun launch (gloo collectives,
both ranks on cuda:0) exercising the sharded path the driver's scaling run
uses with NCCL.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches"]


def _json_lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_reference_arm_contract():
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "1", "--ref-seconds", "2"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    lines = _json_lines(p.stdout)
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    for k in KEYS:
        assert k in line, k


@pytest.mark.gpu
def test_b200_arm_single_gpu():
    p = subprocess.run([sys.executable, "bench.py", "--samples", "3e5", "--steps", "2",
                        "--warmup", "3", "--skip-cpu", "--latency-reps", "20"], cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    (line,) = _json_lines(p.stdout)
    for k in KEYS + ["roofline", "clocks", "latency_25k", "feasibility_530ms"]:
        assert k in line, k
    assert line["value"] > 0 and line["gpu_launches"] > 0 and line["n_gpus"] == 1
    assert line["roofline"]["bound"] == "fp64" and line["roofline"]["frac"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 32 * 300000
    ds = line["device_sampler"]
    assert ds["available"] and ds["bit_identical_to_host_draw"] and ds["verified_samples"] == 300000
    assert ds["e2e_model"]["h2d_bytes_per_step"] == 0 and ds["e2e_model"]["value"] > 0


@pytest.mark.gpu
def test_b200_arm_two_ranks_gloo():
    env = dict(os.environ, BMC_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--samples", "2e5", "--steps", "2", "--warmup", "3", "--skip-cpu",
           "--skip-latency"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1  # rank 0 only
    assert lines[0]["n_gpus"] == 2 and lines[0]["value"] > 0
    assert lines[0]["config"]["parallelism"] == "shard2"
    assert lines[0]["device_sampler"]["bit_identical_to_host_draw"]
    # both ranks' spot checks against the reference, summed over ranks
    assert lines[0]["parity"]["rollout_mismatches"] == 0
    assert lines[0]["parity"]["rollouts_checked"] == 200000  # 1e5 per rank
    # the merged statistics equal a one-process run of the same samples, bit
    # for bit (exact partials), through five merge calls per step
    st2 = lines[0]["statistics"]
    assert st2["merge_calls_per_step"] == 5 and st2["fallbacks"] == 0
    one = subprocess.run([sys.executable, "bench.py", "--samples", "2e5", "--steps", "2",
                          "--warmup", "3", "--skip-cpu", "--skip-latency", "--skip-e2e"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert one.returncode == 0, one.stderr[-3000:]
    (l1,) = _json_lines(one.stdout)
    for k in ("n", "horizon_count", "collision_probability", "min_safe_headway_m", "mean", "sd",
              "median", "skewness"):
        assert st2[k] == l1["statistics"][k], k


@pytest.mark.gpu
def test_b200_arm_nccl_torchrun_one_rank():
    # the driver's scaling launch (torchrun, NCCL process group, device_id
    # bound, collectives on CUDA tensors) at world size 1: every allreduce /
    # allgather of the merged statistics goes through NCCL on the B200
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "1", "--samples", "2e5", "--steps", "2", "--warmup", "3", "--skip-cpu",
           "--skip-latency"]
    env = dict(os.environ)
    env.pop("BMC_DIST_BACKEND", None)
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    (line,) = _json_lines(p.stdout)
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["config"]["parallelism"] == "shard1"
    assert line["statistics"]["merge_calls_per_step"] == 5  # NCCL through the stage's hooks
    assert line["parity"]["rollout_mismatches"] == 0
