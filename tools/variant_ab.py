"""A/B of rollout-kernel variants on one device-resident batch (diagnostic):
interleaved repetitions of each variant, best and median kernel time, and a
bitwise comparison of every variant's outputs against the first one.

python tools/variant_ab.py --samples 2e7 --model default --variants "ilp=2,block_threads=640,test_block=8" ...

The digest line lets runs in separate processes (environment switches such as
BMC_PER_STEP_TEST=1) be compared bit for bit.
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_27193_b200 as bmc  # noqa: E402


def parse_opts(text):
    out = {}
    for kv in text.split(","):
        k, v = kv.split("=")
        out[k] = int(v) if v.lstrip("-").isdigit() else v
    return out


ap = argparse.ArgumentParser()
ap.add_argument("--samples", type=float, default=2e7)
ap.add_argument("--model", default="default")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--variants", nargs="+", required=True)
a = ap.parse_args()
n = int(a.samples)
model = bmc.UncertaintyModel.mixed(3) if a.model == "mixed" else bmc.UncertaintyModel(seed=3)
samples, _ = bmc.draw_batch(model, n)
terms = bmc.stage_terms(samples)
dev = [torch.from_numpy(terms[i]).cuda() for i in range(4)]
ex = bmc.CudaExecutor(0)
peak, _ = ex.fp64_peak()
tot = torch.zeros(1, dtype=torch.int64, device="cuda")
outs, times = [], {v: [] for v in a.variants}
bins = {v: [] for v in a.variants}
lanes = {}
ref_out = None
for rep in range(a.reps):
    for v in a.variants:
        d = torch.empty(n, dtype=torch.float64, device="cuda")
        st = torch.empty(n, dtype=torch.int32, device="cuda")
        tot.zero_()
        ex.rollout_device(dev, (d, st, None), total_steps=tot, **parse_opts(v))
        ex.sync()
        r, _ = ex.last_kernel_ms()
        times[v].append(r)
        bins[v].append(ex.last_stage_ms()[0])
        lanes[v] = ex.lane_efficiency()[2]
        if rep == 0:
            if ref_out is None:
                ref_out = (d.clone(), st.clone())
            same = torch.equal(d.view(torch.int64), ref_out[0].view(torch.int64)) and torch.equal(st, ref_out[1])
            import hashlib
            dig = hashlib.sha256(d.cpu().numpy().tobytes() + st.cpu().numpy().tobytes()).hexdigest()[:16]
            print(f"{v}: outputs bitwise equal to the first variant: {same}  digest {dig}", flush=True)
steps = int(tot.item())
for v in a.variants:
    b, m = min(times[v]), statistics.median(times[v])
    print(f"{a.model} n={n} {v:45s} best {b:9.3f} ms  median {m:9.3f} ms  "
          f"exec {32 * steps / (b * 1e-3) / peak:.4f} of probe  binning {min(bins[v]):.3f} ms  "
          f"lane efficiency {lanes[v]:.5f}", flush=True)
