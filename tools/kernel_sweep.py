"""Device-resident rollout timing sweep over the scheduling knobs.

python tools/kernel_sweep.py [--samples 4e6] [--model default|mixed] [--profile]
Prints one line per configuration: rollout-kernel ms (CUDA events on the
engine stream), predict/bin ms, RK4 steps/s and executed FP64 op rate.
--profile: run only the default configuration twice (for ncu -k rollout).
"""
import argparse
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2604_27193_b200 as bmc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=float, default=4e6)
    ap.add_argument("--model", default="default")
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--occupancy", action="store_true")
    ap.add_argument("--testblock", action="store_true", help="per-step vs blocked termination test")
    ap.add_argument("--ilpcmp", action="store_true", help="ilp 1 (1024) vs ilp 2 (640), blocked test")
    a = ap.parse_args()
    n = int(a.samples)
    model = bmc.UncertaintyModel.mixed(3) if a.model == "mixed" else bmc.UncertaintyModel(seed=3)
    samples, _ = bmc.draw_batch(model, n)
    terms = bmc.stage_terms(samples)
    dev = [torch.from_numpy(terms[i]).cuda() for i in range(4)]
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.empty(n, dtype=torch.int32, device="cuda")
    hz = torch.empty(n, dtype=torch.uint8, device="cuda")
    tot = torch.zeros(1, dtype=torch.int64, device="cuda")
    ex = bmc.CudaExecutor(0)
    peak, _ = ex.fp64_peak()
    print(f"fp64 probe peak: {peak/1e12:.3f} T op/s", flush=True)
    if a.profile:
        for _ in range(2):
            ex.rollout_device(dev, (d, st, hz), total_steps=tot)
            ex.sync()
        print("profile run done", ex.last_kernel_ms())
        return
    configs = [(s, t, b, 1, 1) for s, t, b in itertools.product(
        ["binned", "index"], ["shared", "global", "none"], [256, 512, 768, 1024])]
    configs += [(s, t, b, 2, 1) for s, t, b in itertools.product(
        ["binned"], ["shared", "global"], [512, 640, 768])]
    if a.quick:
        configs = [c for c in configs if c[0] == "binned" and c[2] >= 512 and c[1] != "none"]
    if a.occupancy:
        configs = [("binned", t, b, 1, 1) for t in ("shared", "global") for b in (256, 512, 768, 1024)]
    if a.testblock:
        configs = [("binned", "shared", b, 1, tb) for tb in (1, 8) for b in (768, 1024)]
        configs += [("binned", "shared", b, 2, 8) for b in (512, 640, 768)]
    if a.ilpcmp:
        configs = [("binned", "shared", 1024, 1, 8), ("binned", "shared", 640, 2, 8)]
    for sched, table, bt, ilp, tb in configs:
        if table == "none" and sched == "binned":
            continue
        best = None
        for _ in range(a.reps):
            tot.zero_()
            ex.rollout_device(dev, (d, st, hz), total_steps=tot, schedule=sched, table=table,
                              block_threads=bt, ilp=ilp, test_block=tb)
            ex.sync()
            r, p = ex.last_kernel_ms()
            if best is None or r + p < best[0] + best[1]:
                best = (r, p)
        steps = int(tot.item())
        r, p = best
        _, _, eff = ex.lane_efficiency()
        print(f"{a.model:7s} n={n} sched={sched:6s} table={table:6s} bt={bt:4d} ilp={ilp} tb={tb} "
              f"rollout {r:9.3f} ms  predict {p:7.3f} ms  steps/s {steps/(r*1e-3):.4e}  "
              f"exec-op/s {32*steps/(r*1e-3)/1e12:.3f} T ({32*steps/(r*1e-3)/peak:.3f} of probe)"
              f"  algo {57*steps/(r*1e-3)/peak:.3f}  lane-eff {eff:.4f}", flush=True)


if __name__ == "__main__":
    main()
