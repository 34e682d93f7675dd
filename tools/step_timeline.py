"""Per-step device timeline of the bench step (events on the engine stream):
rollout launch (bin + rollout + unpermute) vs statistics vs gaps.
python tools/step_timeline.py [--samples 4e7] [--steps 6]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_27193_b200 as bmc  # noqa: E402
from paper_2604_27193_b200 import distributed as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--samples", type=float, default=4e7)
ap.add_argument("--steps", type=int, default=6)
a = ap.parse_args()
n = int(a.samples)
ex = bmc.CudaExecutor(0)
terms, _, _ = ex.draw_device(bmc.UncertaintyModel(seed=3), n, samples=False)
dev = [terms[i] for i in range(4)]
d = torch.empty(n, dtype=torch.float64, device="cuda")
st = torch.empty(n, dtype=torch.int32, device="cuda")
hz = torch.empty(n, dtype=torch.uint8, device="cuda")
total = torch.zeros(1, dtype=torch.int64, device="cuda")
stream = torch.cuda.ExternalStream(ex.stream_handle, device="cuda:0")
shard = D.DeviceShard(ex, d, hz)
coll = D.Collective(None, "cuda:0")
heads = [30.0 * (1.0 + 0.25 * k) for k in range(21)]
sw = bmc.SimWorld()
for i in range(a.steps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    h0 = time.perf_counter()
    e[0].record(stream)
    total.zero_()
    ex.rollout_device(dev, (d, st, hz), sw, total_steps=total)
    e[1].record(stream)
    h1 = time.perf_counter()
    b_ms, r_ms, u_ms = ex.last_stage_ms()
    h2 = time.perf_counter()
    D.exceedance_counts(shard, coll, heads)
    D.summarize(shard, coll, 2.0)
    e[2].record(stream)
    torch.cuda.synchronize()
    h3 = time.perf_counter()
    launch = e[0].elapsed_time(e[1])
    stats = e[1].elapsed_time(e[2])
    print(f"step {i}: device {e[0].elapsed_time(e[2]):8.2f} ms = rollout launch {launch:8.2f} "
          f"(bin {b_ms:.2f} + rollout {r_ms:.2f} + unpermute {u_ms:.2f}) + stats {stats:6.2f} | host: "
          f"enqueue {1e3*(h1-h0):.2f} wait {1e3*(h2-h1):.2f} stats {1e3*(h3-h2):.2f} ms", flush=True)
ex.close()
