"""run_cuda (host samples -> host results) wall time vs pipeline chunk size:
python tools/chunk_sweep.py -- median of 5 per (n, chunk)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_27193_b200 as bmc  # noqa: E402

ex = bmc.CudaExecutor(0)
m = bmc.UncertaintyModel(seed=3)
full, _ = bmc.draw_batch(m, 16_000_000)
out = np.empty(full.shape[0], dtype=bmc.RESULT_DTYPE)
for n in (250_000, 500_000, 1_000_000, 2_000_000, 4_000_000, 8_000_000, 16_000_000):
    s, o = full[:n], out[:n]
    row = []
    for div in (1, 2, 4, 8, 16):
        chunk = max(1, n // div)
        for sampler in ("run", "model"):
            f = (lambda: ex.run(s, out=o, chunk=chunk)) if sampler == "run" else \
                (lambda: ex.run_model(m, n, out=o, chunk=chunk, sampler="device"))
            f()
            ts = []
            for _ in range(5):
                t = time.perf_counter()
                f()
                ts.append(time.perf_counter() - t)
            row.append(f"{sampler}/{div}:{statistics.median(ts) * 1e3:7.2f}")
    print(f"n={n:>9}  " + "  ".join(row), flush=True)
ex.close()
