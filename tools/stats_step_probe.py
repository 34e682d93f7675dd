"""Where does a bench step's time go with the fused statistics stage?

Times (CUDA events on the engine's stream + host wall) for: the rollout
alone, the rollout with pass 1 fused, and the full step (rollout + finish),
at --n samples of the default model.  Diagnostic only.
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_27193_b200 as bmc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=2e7)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n = int(a.n)
samples, _ = bmc.draw_batch(bmc.UncertaintyModel(seed=3), n)
terms = bmc.stage_terms(samples)
dev = [torch.from_numpy(terms[i]).cuda() for i in range(4)]
d = torch.empty(n, dtype=torch.float64, device="cuda")
st = torch.empty(n, dtype=torch.int32, device="cuda")
hz = torch.empty(n, dtype=torch.uint8, device="cuda")
ex = bmc.CudaExecutor(0)
stream = torch.cuda.ExternalStream(ex.stream_handle)
headways = [30.0 * (1.0 + 0.25 * k) for k in range(21)]
stage = ex.stats_stage(n, headways, [0.05, 0.01, 0.001], summarize=True, bin_width=2.0)


def timed(label, fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(a.reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / a.reps * 1e3
    print(f"{label:40s} events {e0.elapsed_time(e1) / a.reps:9.3f} ms   wall {wall:9.3f} ms  "
          f"stages(bin, roll, unperm) {tuple(round(x, 3) for x in ex.last_stage_ms())}", flush=True)


timed("rollout only", lambda: (ex.rollout_device(dev, (d, st, hz)), ex.sync()))
timed("rollout + fused pass 1", lambda: (stage.begin(), ex.rollout_device(dev, (d, st, hz), stats=stage), ex.sync()))


def full():
    stage.begin()
    ex.rollout_device(dev, (d, st, hz), stats=stage)
    ex.last_stage_ms()
    stage.finish(d, hz)


timed("rollout + stage finish", full)
timed("finish only (after a fused rollout)", lambda: stage.finish(d, hz))
timed("bmc_cuda_stats (standalone pass 1)", lambda: ex.stats(d, hz, headways, [0.05, 0.01, 0.001], True, 2.0))
timed("summarize (legacy API via stage)", lambda: ex.summarize(d, hz, 2.0))
