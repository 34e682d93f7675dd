"""bmc_cuda_run end to end at --n for the library in BMC_LIB_PATH (or the
in-tree one): mean wall of --reps calls per chunk size.  Diagnostic only."""
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
ap.add_argument("--chunks", default="0,8388608")
a = ap.parse_args()
n = int(a.n)
samples, _ = bmc.draw_batch(bmc.UncertaintyModel(seed=3), n)
ex = bmc.CudaExecutor(0)
out = np.empty(n, dtype=bmc.RESULT_DTYPE)
tag = os.environ.get("BMC_LIB_PATH", "in-tree")
for ch in [int(c) for c in a.chunks.split(",")]:
    ex.run(samples, out=out, chunk=ch)
    gc.collect()
    gc.disable()
    ts = []
    for _ in range(a.reps):
        t = time.perf_counter()
        rep = ex.run(samples, out=out, chunk=ch)
        ts.append(time.perf_counter() - t)
    gc.enable()
    print(f"{tag}: chunk {ch or 'default'} wall mean {np.mean(ts)*1e3:.2f} min {min(ts)*1e3:.2f} ms "
          f"= {n/np.mean(ts):.4e}/s chunks {rep.chunks} kernel_ms {rep.kernel_ms:.1f}", flush=True)
