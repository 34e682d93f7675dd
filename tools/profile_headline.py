"""One bench step at the headline configuration, for ncu.

1e8 default-model samples (seed 3) resident in HBM; one step = stats begin,
binning (predict, scan, scatter), the rollout with statistics pass 1 fused,
unpermute, and the statistics stage (finalize, pass 2, targets, compaction,
selection) -- the same calls bench.py times.  --warm runs one untimed step
first so the captured launches are the steady-state ones.

  ncu --set full --clock-control none -k regex:'rollout_kernel' -s 1 -c 1 \\
      python tools/profile_headline.py --warm
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_27193_b200 as bmc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--samples", type=float, default=1e8)
ap.add_argument("--warm", action="store_true")
a = ap.parse_args()
n = int(a.samples)
model = bmc.UncertaintyModel(seed=3)
samples, _ = bmc.draw_batch(model, n)
terms = bmc.stage_terms(samples)
del samples
dev = [torch.from_numpy(terms[i]).cuda() for i in range(4)]
del terms
d = torch.empty(n, dtype=torch.float64, device="cuda")
st = torch.empty(n, dtype=torch.int32, device="cuda")
hz = torch.empty(n, dtype=torch.uint8, device="cuda")
ex = bmc.CudaExecutor(0)
headways = [30.0 * (1.0 + 0.25 * k) for k in range(21)]
stage = ex.stats_stage(n, headways, [0.05, 0.01, 0.001], summarize=True, bin_width=2.0)
total = torch.zeros(1, dtype=torch.int64, device="cuda")


def step():
    total.zero_()
    stage.begin()
    ex.rollout_device(dev, (d, st, hz), total_steps=total, stats=stage)
    return stage.finish(d, hz)


if a.warm:
    step()
out = step()
torch.cuda.synchronize()
print(f"n={n} rk4_steps={int(total.item())} median={out['summary']['median']!r} "
      f"stage_kernels={out['launches']}")
