"""bmc_cuda_run end to end (host AoS samples -> host AoS results) at --n,
default schedule (edge-ramped chunks) vs fixed chunks; wall time per call and
the run's own breakdown.  Diagnostic only."""
import argparse
import gc
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27193_b200 as bmc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=1e8)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n = int(a.n)
samples, _ = bmc.draw_batch(bmc.UncertaintyModel(seed=3), n)
ex = bmc.CudaExecutor(0)
out = np.empty(n, dtype=bmc.RESULT_DTYPE)
for label, opts in [("default (ramped)", {}), ("fixed 4M chunks", {"chunk": 1 << 22}),
                    ("fixed 8M chunks", {"chunk": 1 << 23}), ("default again", {})]:
    ex.run(samples, out=out, **opts)
    gc.collect()
    gc.disable()
    ts = []
    for _ in range(a.reps):
        t = time.perf_counter()
        rep = ex.run(samples, out=out, **opts)
        ts.append(time.perf_counter() - t)
    gc.enable()
    print(f"{label:20s} wall {min(ts)*1e3:9.2f} ms (min of {a.reps}) = {n/min(ts):.4e}/s  "
          f"chunks {rep.chunks}  kernel_ms {rep.kernel_ms:.1f}  predict_ms {rep.predict_ms:.1f}",
          flush=True)
