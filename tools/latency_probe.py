"""Where a 25k-sample decision's time goes (diagnostic): host wall per
decision through the CUDA graph (sim-only and with the statistics stage),
and the device-resident pieces timed with CUDA events -- binning, rollout,
unpermute -- for the same batch.  Run under ncu for per-kernel durations."""
import argparse
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_27193_b200 as bmc  # noqa: E402
from paper_2604_27193_b200.stats import StatsRequest  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=25000)
ap.add_argument("--reps", type=int, default=300)
ap.add_argument("--model", default="default", choices=["default", "mixed"])
a = ap.parse_args()
ex = bmc.CudaExecutor(0)
mk = bmc.UncertaintyModel.mixed if a.model == "mixed" else (lambda s: bmc.UncertaintyModel(seed=s))
batches = [bmc.draw_batch(mk(s), a.n)[0] for s in range(1, 9)]
heads = [30.0 * (1.0 + 0.25 * k) for k in range(21)]
for label, g in [("graph sim-only", ex.graph(a.n)),
                 ("graph + statistics", ex.graph(a.n, stats=StatsRequest(heads, [0.05, 0.01, 0.001])))]:
    for b in batches:
        g.run(b)
    ts = []
    for k in range(a.reps):
        t = time.perf_counter()
        g.run(batches[k % len(batches)])
        if g.req is not None:
            g.stats()
        ts.append(1e3 * (time.perf_counter() - t))
    print(f"{label:22s} p50 {statistics.median(ts):.4f} ms  p99 {np.percentile(ts, 99):.4f} ms  "
          f"min {min(ts):.4f} ms", flush=True)
    g.close()
# device-resident pieces for batch 0
terms = bmc.stage_terms(batches[0])
dev = [torch.from_numpy(terms[i]).cuda() for i in range(4)]
d = torch.empty(a.n, dtype=torch.float64, device="cuda")
st = torch.empty(a.n, dtype=torch.int32, device="cuda")
hz = torch.empty(a.n, dtype=torch.uint8, device="cuda")
ms = []
for _ in range(50):
    ex.rollout_device(dev, (d, st, hz))
    ms.append(ex.last_stage_ms())
ms = np.array(ms[5:])
print(f"device-resident: bin {np.median(ms[:, 0]):.4f} ms  rollout {np.median(ms[:, 1]):.4f} ms  "
      f"unpermute {np.median(ms[:, 2]):.4f} ms  longest rollout {int(st.max().item())} steps")
t0 = time.perf_counter()
for _ in range(100):
    bmc.stage_terms(batches[0])
print(f"host RolloutTerms staging of {a.n}: {10 * (time.perf_counter() - t0):.4f} ms")
