"""Multi-rank (sharded) statistics: world_size 2/3 over gloo on CPU.

The merge logic in paper_2604_27193_b200/distributed.py is exercised with
the NumPy shard backend (same semantics as the device kernels) in real
torch.distributed processes, and compared with the reference's analysis
functions on the unsharded results.  The GPU variant (two processes sharing
cuda:0, DeviceShard) is in test_gpu_distributed below.
"""
import json
import math
import os
import socket
import tempfile

import numpy as np
import pytest

from paper_2604_27193_b200 import distributed as D
from oracle.pyoracle import RESULT_DTYPE, Model, World

N_RESULTS = 4000
LEVELS = [0.05, 0.01, 0.001, 0.5]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dataset():
    """Deterministic mixed-model results (with horizon hits) from the C oracle."""
    from oracle.pyoracle import Port
    port = Port()
    samples, _ = port.draw_range(Model.mixed(7), 0, N_RESULTS)
    return port.run(samples, World(), threads=4)


def _grid(res):
    d = res["stop_distance"]
    return [math.floor(d.min()) - 5.0 + k for k in range(int(math.ceil(d.max()) - math.floor(d.min())) + 11)]


def _compute(shard, coll, n_total, grid):
    summ = D.summarize(shard, coll, 2.0)
    probs, thr = D.build_risk_curve(shard, coll, n_total, grid, LEVELS, 30.0)
    return {
        "summary": {k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in summ.items()},
        "probs": probs.tolist(),
        "thr": thr,
    }


def _worker(rank, world, outdir, port, device_kind):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        res = _dataset()
        b, e = D.shard_range(res.shape[0], rank, world)
        if device_kind == "cuda":
            import torch
            import paper_2604_27193_b200 as bmc
            ex = bmc.CudaExecutor(0)
            d = torch.from_numpy(np.ascontiguousarray(res["stop_distance"][b:e])).cuda()
            hz = torch.from_numpy(np.ascontiguousarray(res["hit_horizon"][b:e])).cuda()
            shard = D.DeviceShard(ex, d, hz)
        else:
            shard = D.HostShard(res["stop_distance"][b:e], res["hit_horizon"][b:e])
        out = _compute(shard, D.Collective(dist, "cpu"), res.shape[0], _grid(res))
        with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
            json.dump(out, f)
    finally:
        dist.destroy_process_group()


def _run_world(world, device_kind="host"):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, tmp, _free_port(), device_kind), nprocs=world, join=True)
        outs = [json.load(open(os.path.join(tmp, f"rank{r}.json"))) for r in range(world)]
    for o in outs[1:]:
        assert o == outs[0]  # every rank holds the identical merged answer
    return outs[0]


def _check_against_reference(ref, out):
    res = _dataset()
    want = ref.summarize(res, 2.0)
    got = out["summary"]
    for k in ("n", "horizon_count", "bins"):
        assert got[k] == want[k], k
    for k in ("min", "max", "median", "origin"):
        assert got[k] == want[k], k
    assert got["mean"] == pytest.approx(want["mean"], rel=1e-12)
    assert got["sd"] == pytest.approx(want["sd"], rel=1e-12)
    assert got["skewness"] == pytest.approx(want["skewness"], rel=1e-9)
    assert got["histogram"] == [int(x) for x in want["histogram"]]
    probs, thr = ref.build_risk_curve(res, _grid(res), LEVELS, 30.0)
    assert out["probs"] == probs.tolist()
    assert [tuple(t) for t in out["thr"]] == [tuple(t) for t in thr]


def test_shard_ranges_cover_exactly():
    for n in (1, 7, 100, 12345):
        for world in (1, 2, 3, 8):
            spans = [D.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_single_rank_host_shard_matches_reference(ref):
    res = _dataset()
    out = _compute(D.HostShard(res["stop_distance"], res["hit_horizon"]), D.Collective(),
                   res.shape[0], _grid(res))
    _check_against_reference(ref, out)


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_world_matches_reference(ref, world):
    _check_against_reference(ref, _run_world(world))


@pytest.mark.gpu
def test_gpu_shards_over_gloo(ref):
    """Two ranks on one B200 (own contexts), DeviceShard + gloo collectives."""
    _check_against_reference(ref, _run_world(2, "cuda"))
