"""Host/device timeline of bench.py's step (diagnostic): per step, the
device span (CUDA events on the engine's stream around the whole step) and
the host time of each phase, to find time that is neither kernel nor
statistics.  Same calls as bench.py's step."""
import argparse
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_27193_b200 as bmc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=2e7)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--total-steps", type=int, default=1)
a = ap.parse_args()
n = int(a.n)
samples, _ = bmc.draw_batch(bmc.UncertaintyModel(seed=3), n)
terms = bmc.stage_terms(samples)
dev = [torch.from_numpy(terms[i]).cuda() for i in range(4)]
del terms
d = torch.empty(n, dtype=torch.float64, device="cuda")
st = torch.empty(n, dtype=torch.int32, device="cuda")
hz = torch.empty(n, dtype=torch.uint8, device="cuda")
total = torch.zeros(1, dtype=torch.int64, device="cuda")
ex = bmc.CudaExecutor(0)
stream = torch.cuda.ExternalStream(ex.stream_handle)
headways = [30.0 * (1.0 + 0.25 * k) for k in range(21)]
stage = ex.stats_stage(n, headways, [0.05, 0.01, 0.001], summarize=True, bin_width=2.0)
sw = bmc.SimWorld()


def step(evs, host):
    t = [time.perf_counter()]
    if a.total_steps:
        total.zero_()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    stage.begin()
    t.append(time.perf_counter())
    ex.rollout_device(dev, (d, st, hz), sw, total_steps=total if a.total_steps else None,
                      stats=stage)
    t.append(time.perf_counter())
    stages = ex.last_stage_ms()
    t.append(time.perf_counter())
    out = stage.finish(d, hz)
    t.append(time.perf_counter())
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(stream)
    if a.total_steps:
        int(total.item())
    t.append(time.perf_counter())
    evs.append((e0, e1, stages))
    host.append([1e3 * (t[i + 1] - t[i]) for i in range(len(t) - 1)])


for _ in range(2):
    step([], [])
torch.cuda.synchronize()
gc.collect()
gc.disable()
evs, host = [], []
E0 = torch.cuda.Event(enable_timing=True)
E1 = torch.cuda.Event(enable_timing=True)
E0.record(stream)
for _ in range(a.steps):
    step(evs, host)
E1.record(stream)
torch.cuda.synchronize()
print(f"n={n}: whole {E0.elapsed_time(E1) / a.steps:.3f} ms/step")
for k, ((e0, e1, sg), h) in enumerate(zip(evs, host)):
    gap = evs[k + 1][0].elapsed_time(e0) if False else (e1.elapsed_time(evs[k + 1][0]) if k + 1 < len(evs) else float("nan"))
    print(f"step {k}: device span {e0.elapsed_time(e1):9.3f} ms  (bin {sg[0]:.3f} roll {sg[1]:.3f} "
          f"unperm {sg[2]:.3f})  gap to next {gap:7.3f} ms  host phases "
          f"[zero+begin, rollout enqueue, stage_ms wait, finish, item] = "
          f"{', '.join(f'{x:.3f}' for x in h)}")
