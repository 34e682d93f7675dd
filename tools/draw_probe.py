"""On-device sampler throughput probe (ncu target): draws n samples of the
default model straight into SoA rollout terms, twice (first = warm-up)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_27193_b200 as bmc  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
ex = bmc.CudaExecutor(0)
m = bmc.UncertaintyModel(seed=3)
for k in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    ex.draw_device(m, n, samples=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
print(f"draw {n} samples: {dt * 1e3:.2f} ms host-timed ({n / dt:.3e} samples/s)")
ex.close()
