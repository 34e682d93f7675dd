"""C2 real-time decision latency (25k samples, CUDA graph replay, host wall
clock per decision, p50/p99 over replays on 16 fresh-seed batches) vs the
rollout plan: schedule (binned / index order), termination-test block,
block size.  python tools/latency_sweep.py [--n 25000] [--reps 300]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_27193_b200 as bmc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=25000)
ap.add_argument("--reps", type=int, default=300)
a = ap.parse_args()
ex = bmc.CudaExecutor(0)
batches = [bmc.draw_batch(bmc.UncertaintyModel(seed=s), a.n)[0] for s in range(1, 17)]
configs = [dict(schedule=s, test_block=tb, block_threads=bt)
           for s in ("binned", "index") for tb in (1, 8) for bt in (128 * 0 + 256, 512, 1024)]
for cfg in configs:
    try:
        g = ex.graph(a.n, **cfg)
    except Exception as e:  # noqa: BLE001
        print(f"{cfg}: {e}")
        continue
    for b in batches[:4]:
        g.run(b)
    ts = []
    for k in range(a.reps):
        t = time.perf_counter()
        g.run(batches[k % len(batches)])
        ts.append(1e3 * (time.perf_counter() - t))
    g.close()
    print(f"{str(cfg):60s} p50 {np.percentile(ts, 50):.3f} ms  p99 {np.percentile(ts, 99):.3f} ms",
          flush=True)
ex.close()
