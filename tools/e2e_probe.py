"""bmc_cuda_run end to end (host AoS samples -> host AoS results) at --n:
wall time per call for a few host-thread counts and chunk sizes, with the
pipeline's own host-phase totals (BMC_PIPE_TRACE=1 prints them to stderr:
time spent waiting on the device, unpacking results, staging terms).
Diagnostic only."""
import argparse
import gc
import os
import sys
import time

os.environ.setdefault("BMC_PIPE_TRACE", "1")
import numpy as np  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27193_b200 as bmc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=1e8)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n = int(a.n)
print(f"host cores {os.cpu_count()}, affinity {len(os.sched_getaffinity(0))}", flush=True)
samples, _ = bmc.draw_batch(bmc.UncertaintyModel(seed=3), n)
ex = bmc.CudaExecutor(0)
out = np.empty(n, dtype=bmc.RESULT_DTYPE)
ncpu = len(os.sched_getaffinity(0))
variants = [("default", {}), ("threads/2", {"host_threads": max(1, ncpu // 2)}),
            ("threads x2", {"host_threads": 2 * ncpu}), ("fixed 8M chunks", {"chunk": 1 << 23}),
            ("fixed 2M chunks", {"chunk": 1 << 21}), ("default again", {})]
for label, opts in variants:
    ex.run(samples, out=out, **opts)
    gc.collect()
    gc.disable()
    ts = []
    for _ in range(a.reps):
        t = time.perf_counter()
        rep = ex.run(samples, out=out, **opts)
        ts.append(time.perf_counter() - t)
    gc.enable()
    print(f"{label:20s} wall min {min(ts)*1e3:9.2f} mean {np.mean(ts)*1e3:9.2f} ms = "
          f"{n/np.mean(ts):.4e}/s  chunks {rep.chunks}  kernel_ms {rep.kernel_ms:.1f}  "
          f"predict_ms {rep.predict_ms:.1f}", flush=True)
