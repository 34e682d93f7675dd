#!/usr/bin/env python
"""bench.py -- BASELINE.json metric: MC rollouts/s at 1e8 samples (1/2/4/8 GPU),
plus p50/p99 latency of the real-time 25k-sample decision batch.

One JSON line on rank 0.  Arms:
  (default)          the B200 engine (libbrakemc_b200.so through its C-ABI)
  --impl reference   the reference's own CPU executor (run_parallel, all host
                     threads) from oracle/_ref, on a bounded prefix sample of
                     the same workload; rank 0 only.

A step = one pass of the hot path over the batch: predict/bin + RK4 rollout
of every sample on the rank's shard + the outcome statistics (exceedance
counts over the TTC-threshold grid, horizon count, extrema, moments, median,
histogram), then the NCCL allreduce of the count vectors when N > 1.
`value`: inputs resident in HBM (32 B/sample terms, 3.2 GB at 1e8 >> 126 MB
L2, so no flush is needed), device-timed with CUDA events on the engine's
stream, max over ranks.  `e2e`: the same rollouts through bmc_cuda_run (the
run_cuda core) from pageable host samples to host results, H2D/D2H inside.
Sample generation is excluded from both (backends.hpp:22-24), and reported.
`device_sampler`: the same shard drawn on the GPU by the op-for-op glibc port
(csrc/bmc_libm.h), checked bit for bit against the host-drawn terms over the
whole shard, and `e2e_model`: model -> host results through
bmc_cuda_run_model with the device sampler (sampling included, the
convention of the reference's feasibility search, analysis.cpp:331-338).
"""
import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALGO_FLOPS_PER_STEP = 57   # reference formulation, per RK4 step
# Algorithmic HBM bytes per sample of the streaming stages around the rollout:
#   sample stream = predict (reads v0, floor, drag, grade: 32 B; writes a 2-B key)
#                 + binning scatter (reads key + 32 B terms; writes the 32-B packed
#                   record + 4-B slot index)
#   result stream = unpermute (reads the 4-B slot + 16-B packed output; writes
#                   stop_distance 8 B + steps 4 B + hit_horizon 1 B)
SAMPLE_STREAM_BYTES = 32 + 2 + 2 + 32 + 32 + 4
RESULT_STREAM_BYTES = 4 + 16 + 8 + 4 + 1
EXEC_FLOPS_PER_STEP = 32   # this kernel (actuator table + exact-doubling FMA)
SPEC_FP64_OPS = 148 * 64 * 1.965e9  # nominal DADD/DMUL rate at max clock


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--samples", type=float, default=1e8)
    p.add_argument("--seed", type=int, default=3)
    p.add_argument("--latency-reps", type=int, default=1000)
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--ref-seconds", type=float, default=150.0)
    p.add_argument("--skip-e2e", action="store_true")
    p.add_argument("--skip-latency", action="store_true")
    p.add_argument("--skip-cpu", action="store_true")
    p.add_argument("--clock-ms", type=int, default=200, help="nvidia-smi sampling period (0: off)")
    p.add_argument("--parity-samples", type=float, default=2e5,
                   help="random indices of the timed batch re-simulated by the reference")
    p.add_argument("--skip-parity", action="store_true")
    return p.parse_args()


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every period_ms.  Started
    before the warm-up steps (nvidia-smi's NVML start-up can stall the
    driver for tens of ms, which must not land in the timed region) and
    summarised over the rows whose timestamps fall inside the timed window
    (mark_start / mark_end)."""
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period_ms: int = 200):
        self.index = index
        self.period_ms = period_ms
        self.rows = []
        self.proc = None
        self.thread = None
        self.t0 = None
        self.t1 = None

    def start(self):
        if self.period_ms <= 0:
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period_ms), "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def _read(self):
        import datetime
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) != 8:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            self.rows.append((ts, parts[1:]))

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=5)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, r in self.rows:
            if ts is not None and self.t0 is not None and not (self.t0 <= ts <= (self.t1 or ts)):
                continue
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for nm, v in zip(names, r[3:]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "window": "timed region only (rows filtered by timestamp)"}


# --------------------------------------------------------------- reference

def reference_arm(args, rank):
    if rank != 0:
        return
    from oracle.pyoracle import Model, Reference, World
    ref = Reference()
    cores = ref.hardware_concurrency()
    model = Model(seed=args.seed)
    probe, _ = ref.draw_batch(model, 2000)
    _, t_probe, _ = ref.run(probe, World(), "parallel", 0)
    per_sample = t_probe / 2000.0
    # whole run within minutes: --ref-seconds of CPU work split over all steps
    budget = max(0.05, args.ref_seconds / max(1, args.steps + args.warmup))
    n = int(min(args.samples, max(2000, budget / per_sample)))
    samples, _ = ref.draw_batch(model, n)
    for _ in range(args.warmup):
        ref.run(samples[: max(2000, n // 10)], World(), "parallel", 0)
    times = []
    for _ in range(args.steps):
        _, wall, wc = ref.run(samples, World(), "parallel", 0)
        times.append(wall)
    value = args.steps * n / sum(times)
    line = {
        "impl": "reference", "metric": "MC rollouts/s at 1e8 samples (1/2/4/8 GPU)",
        "value": value, "unit": "rollouts/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference draw_batch, default UncertaintyModel)",
        "config": {"workload": "C5 default model seed %d; bounded prefix sample of the 1e8 batch"
                   % args.seed, "samples_per_step": n, "executor": "run_parallel",
                   "worker_count": wc, "chunk_size": 256},
        "cpu_baseline": {"value": value, "unit": "rollouts/s", "cores": cores, "kind": "reference",
                         "sample": f"{n} samples (prefix of seed {args.seed}), run_parallel"},
        "e2e": {"value": value, "unit": "rollouts/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args, n_total):
    from oracle.pyoracle import Model, Reference, World
    ref = Reference()
    model = Model(seed=args.seed)
    probe, _ = ref.draw_batch(model, 2000)
    _, t_probe, _ = ref.run(probe, World(), "parallel", 0)
    n = int(min(n_total, max(2000, args.cpu_seconds * 2000.0 / t_probe)))
    samples, _ = ref.draw_batch(model, n)
    _, wall, wc = ref.run(samples, World(), "parallel", 0)
    # the reference's single-core executor too (run_sequential, backends.cpp:38-55)
    ns = min(n, 10000)
    _, wall_s, _ = ref.run(samples[:ns], World(), "sequential")
    return {"value": n / wall, "unit": "rollouts/s", "cores": wc, "kind": "reference",
            "sample": f"{n} samples (prefix of the seed-{args.seed} batch), reference "
                      f"run_parallel with {wc} threads, {wall:.1f} s",
            "sequential": {"value": ns / wall_s, "unit": "rollouts/s", "cores": 1,
                           "sample": f"{ns} samples, reference run_sequential, {wall_s:.1f} s"}}


# -------------------------------------------------------------------- b200

def _pct(v, p):
    return float(np.percentile(np.array(v), p))


def realtime(bmc, ex, sw, args, headways, risks):
    """C2: 25k-sample decision batches through the CUDA-graph mode, p50/p99
    over replays on fresh seeds: sim-only (samples given, per-sample results
    back), with the fused statistics stage in the graph (P(collision) per TTC
    threshold + min_safe_headway per decision), and with sampling inside the
    decision as well (the reference's feasibility convention,
    analysis.cpp:331-338)."""
    from paper_2604_27193_b200.stats import StatsRequest
    n = 25000
    req = StatsRequest(headways=headways, risk_levels=risks)
    g = ex.graph(n, sw)
    gs = ex.graph(n, sw, stats=req)
    try:
        batches = [bmc.draw_batch(bmc.UncertaintyModel(seed=s), n)[0] for s in range(1, 17)]
        for _ in range(2):
            for b in batches:
                g.run(b)
                gs.run(b)
                gs.stats()
            gs.run_model(bmc.UncertaintyModel(seed=999))  # first call captures its graph
        sim_ms, st_ms, full_ms, steps = [], [], [], []
        gc.collect()
        gc.disable()  # the engine's decision latency, not the interpreter's collector
        for k in range(args.latency_reps):
            t1 = time.perf_counter()
            rep = g.run(batches[k % len(batches)])
            sim_ms.append(1e3 * (time.perf_counter() - t1))
            steps.append(int(rep.results["steps"].max()))
        for k in range(args.latency_reps):
            t1 = time.perf_counter()
            gs.run(batches[k % len(batches)])
            dec = gs.stats()
            st_ms.append(1e3 * (time.perf_counter() - t1))
        for k in range(args.latency_reps):
            t1 = time.perf_counter()
            gs.run_model(bmc.UncertaintyModel(seed=1000 + k))
            gs.stats()
            full_ms.append(1e3 * (time.perf_counter() - t1))
        gc.enable()
        return {"samples": n, "budget_ms": 530.0, "mode": "CUDA graph (H2D, bin, rollout, D2H)",
                "with_sampling_mode": "CUDA graph (%s) + statistics stage" % (
                    "device sampler: params H2D, draw, bin, rollout, D2H"
                    if bmc.device_sampler_available() else "host sampler, terms H2D"),
                "sim_only_ms": {"p50": _pct(sim_ms, 50), "p99": _pct(sim_ms, 99),
                                "reps": len(sim_ms)},
                "with_statistics_ms": {"p50": _pct(st_ms, 50), "p99": _pct(st_ms, 99),
                                       "reps": len(st_ms),
                                       "returns": "per-sample results + collision probability at "
                                                  "%d TTC thresholds + min_safe_headway at %s"
                                                  % (len(headways), risks)},
                "with_sampling_ms": {"p50": _pct(full_ms, 50), "p99": _pct(full_ms, 99),
                                     "reps": len(full_ms)},
                "last_decision_collision_probability": [float(x) for x in
                                                        dec["collision_probability"]],
                "longest_rollout_steps_p50": _pct(steps, 50),
                "kernel_launches_per_decision": rep.launches,
                "kernel_launches_per_decision_with_statistics": dec["launches"]}
    finally:
        g.close()
        gs.close()


def device_sampler(bmc, ex, sw, args, model, n, begin, dev_terms, world, dist, cdev):
    """Draw the rank's shard on the device and prove it equals the host draw
    (all 4 x n terms, bitwise); time the draw kernel and the model-driven
    end-to-end path (sampling included)."""
    import torch
    if not bmc.device_sampler_available():
        return {"available": False,
                "why": bmc.load().bmc_last_error().decode(errors="replace")}
    ex.draw_device(model, min(n, 1 << 20), first=begin, world=sw, samples=False)  # warm-up
    torch.cuda.synchronize()
    t = time.perf_counter()
    terms, _, dclamps = ex.draw_device(model, n, first=begin, world=sw, samples=False)
    draw_s = time.perf_counter() - t
    same = all(torch.equal(terms[i].view(torch.int64), dev_terms[i].view(torch.int64))
               for i in range(4))
    del terms
    torch.cuda.empty_cache()
    out = np.empty(n, dtype=bmc.RESULT_DTYPE)
    ex.run_model(model, n, first=begin, world=sw, out=out, sampler="device")  # warm-up
    if dist is not None:
        dist.barrier()
    reps = max(1, min(args.steps, 3))
    gc.collect()
    gc.disable()
    tt = time.perf_counter()
    for _ in range(reps):
        rep, _ = ex.run_model(model, n, first=begin, world=sw, out=out, sampler="device")
    e2e_s = (time.perf_counter() - tt) / reps
    gc.enable()
    te = torch.tensor([e2e_s, 0.0 if same else 1.0], dtype=torch.float64, device=cdev)
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    return {"available": True, "bit_identical_to_host_draw": float(te[1].item()) == 0.0,
            "verified_samples": n, "clamp_count": dclamps, "draw_s": draw_s,
            "draw_samples_per_s": n / draw_s,
            "e2e_model": {"value": int(args.samples) / float(te[0].item()), "unit": "rollouts/s",
                          "h2d_bytes_per_step": rep.h2d_bytes,
                          "d2h_bytes_per_step": rep.d2h_bytes, "reps": reps,
                          "path": "bmc_cuda_run_model(sampler=device): UncertaintyModel -> "
                                  "device draw + RolloutTerms -> bin+rollout -> D2H -> AoS "
                                  "results (sampling included)"}}


def feasibility_search(bmc, ex, sw, args):
    """max_samples_within_budget (analysis.cpp:320-370) on the CUDA executor:
    the reference's doubling+bisection search, median-of-5 timings, budget
    700-120-50 = 530 ms, search cap raised from 2^22 to 2^27.  Probes run the
    streaming executor (host sampling overlapped with the GPU), i.e. the
    reference convention with sampling included."""
    budget = 0.530
    model = bmc.UncertaintyModel(seed=args.seed)
    holder = [np.empty(0, dtype=bmc.RESULT_DTYPE)]

    def timed_with_sampling(n):
        # results land in a reused host buffer (a deployed decision loop
        # preallocates; the untimed warm-up call absorbs first-touch faults)
        if holder[0].shape[0] < n:
            holder[0] = np.empty(n, dtype=bmc.RESULT_DTYPE)
        out = holder[0][:n]
        return bmc.engine.median_wall_time_s(lambda: ex.run_model(model, n, world=sw, out=out), 5, 1)

    n_max, capped = bmc.engine.max_feasible_n(timed_with_sampling, budget, 1000, 1 << 27)
    with_s = timed_with_sampling(n_max) if n_max else None
    return {"budget_ms": 530.0, "max_samples": n_max, "capped": capped,
            "search_cap": 1 << 27, "time_with_sampling_ms": with_s * 1e3 if with_s else None,
            "meets_convergence_threshold": n_max >= 12000,
            "path": "bmc_cuda_run_model (%s)" % (
                "device sampler: draw + rollout on the GPU" if bmc.device_sampler_available()
                else "host sampler -> pinned SoA -> H2D, overlapped")}


def parity_spot_check(bmc, args, samples, begin, d, st, hz, sw, out, dist, cdev, headways,
                      risks):
    """Checker leg (after the timed region): the headline run's own outputs
    against the reference.  (1) `--parity-samples` random indices of this
    rank's shard re-simulated by the unmodified reference (oracle/_ref,
    run_parallel) and compared bit for bit on all of (stop_distance, steps,
    hit_horizon); (2) at N=1 the step's statistics against a host recount
    over the full per-sample outputs with the reference's formulas
    (analysis.cpp:13-76, 145-194)."""
    import torch
    from oracle.pyoracle import Reference, World
    n = samples.shape[0]
    world = dist.get_world_size() if dist is not None else 1
    k = int(min(n, max(1, args.parity_samples // world)))  # the total is split over ranks
    rng = np.random.default_rng(20261017 + begin)
    idx = np.sort(rng.choice(n, size=k, replace=False)) if k < n else np.arange(n)
    ti = torch.from_numpy(idx).to(d.device)
    gd = d.index_select(0, ti).cpu().numpy()
    gs = st.index_select(0, ti).cpu().numpy()
    gh = hz.index_select(0, ti).cpu().numpy()
    t0 = time.perf_counter()
    ref = Reference()
    want, _, _ = ref.run(np.ascontiguousarray(samples[idx]), World(), "parallel", 0)
    ref_s = time.perf_counter() - t0
    mism = int(np.count_nonzero((gd.view(np.uint64) != want["stop_distance"].view(np.uint64)) |
                                (gs.astype(np.int64) != want["steps"]) |
                                (gh.astype(np.uint8) != want["hit_horizon"].astype(np.uint8))))
    te = torch.tensor([mism, k], dtype=torch.int64, device=cdev)
    if dist is not None:
        dist.all_reduce(te)
    res = {"rollouts_checked": int(te[1].item()), "rollout_mismatches": int(te[0].item()),
           "rollout_checker": "oracle/_ref run_parallel on random indices of the timed batch "
                              f"({ref_s:.1f} s on rank 0)"}
    if dist is None or dist.get_world_size() == 1:
        # statistics recount over all n outputs (integer / order quantities exact)
        t1 = time.perf_counter()
        hd = d.cpu().numpy()
        hh = hz.cpu().numpy() != 0
        bad = []
        hs = np.sort(np.asarray(headways))
        p = np.searchsorted(hs, hd, side="left")  # #{h < d}
        p[hh] = len(hs)
        cnt = np.bincount(p, minlength=len(hs) + 1)
        ex = np.cumsum(cnt[::-1])[::-1][1:]  # #{p > j}
        if not np.array_equal(ex.astype(np.uint64), out["exceed"][np.argsort(np.argsort(headways))]):
            bad.append("exceed")
        sm = out["summary"]
        if sm["horizon_count"] != int(hh.sum()):
            bad.append("horizon_count")
        if sm["min"] != float(hd.min()) or sm["max"] != float(hd.max()):
            bad.append("extrema")
        lo, hi = math.floor(hd.min()), math.ceil(hd.max())
        bins = max(1, int(math.ceil((hi - lo) / 2.0)))
        hidx = np.minimum(((hd - lo) / 2.0).astype(np.uint64), np.uint64(bins - 1))
        if not np.array_equal(np.bincount(hidx.astype(np.int64), minlength=bins).astype(np.uint64),
                              sm["histogram"]):
            bad.append("histogram")
        srt = np.partition(hd, [n // 2 - 1, n // 2])
        med = srt[n // 2] if n % 2 else 0.5 * (srt[n // 2 - 1] + srt[n // 2])
        if sm["median"] != med:
            bad.append("median")
        stopped = hd[~hh]
        for r, v in zip(risks, out["min_safe_headway"]):
            raw = (1.0 - r) * float(n)
            rank = int(math.ceil(raw - raw * 1e-12))
            w = math.inf if rank > stopped.size else float(np.partition(stopped, rank - 1)[rank - 1])
            if v != w:
                bad.append(f"min_safe_headway({r})")
        res.update({"statistics_recount": "exceedance counts, horizon count, min/max, histogram, "
                                          "median, min_safe_headway: host recount over all "
                                          f"{n} outputs with the reference formulas",
                    "statistics_mismatches": bad,
                    "mean_rel_dev_vs_numpy": abs(sm["mean"] - float(hd.mean())) / abs(sm["mean"]),
                    "recount_s": time.perf_counter() - t1})
    return res


def b200_arm(args, rank, world, local_rank, dist, coll_device=None):
    import torch
    import paper_2604_27193_b200 as bmc

    torch.cuda.set_device(local_rank)
    n_total = int(args.samples)
    begin = n_total * rank // world
    end = n_total * (rank + 1) // world
    n = end - begin
    model = bmc.UncertaintyModel(seed=args.seed)
    sw = bmc.SimWorld()

    t0 = time.perf_counter()
    samples, clamps = bmc.draw_batch(model, n, first=begin)
    sample_s = time.perf_counter() - t0
    terms = bmc.stage_terms(samples, sw)
    dev_terms = [torch.from_numpy(terms[i]).to(f"cuda:{local_rank}") for i in range(4)]
    del terms
    d = torch.empty(n, dtype=torch.float64, device=f"cuda:{local_rank}")
    st = torch.empty(n, dtype=torch.int32, device=f"cuda:{local_rank}")
    hz = torch.empty(n, dtype=torch.uint8, device=f"cuda:{local_rank}")
    total_steps = torch.zeros(1, dtype=torch.int64, device=f"cuda:{local_rank}")

    ex = bmc.CudaExecutor(local_rank)
    peak_ops, _ = ex.fp64_peak(reps=5)
    stream = torch.cuda.ExternalStream(ex.stream_handle, device=f"cuda:{local_rank}")

    # C4-style TTC threshold sweep: T in {1.0, 1.25, ..., 6.0} s, closing 30 m/s
    ttc = [1.0 + 0.25 * k for k in range(21)]
    headways = [t * model.initial_speed[0] for t in ttc]
    risks = [0.05, 0.01, 0.001]
    launches = [0]
    kernel_ms = []
    stage_ms = []
    stats_host_ms = []

    from paper_2604_27193_b200 import distributed as D
    cdev = coll_device or f"cuda:{local_rank}"
    merge = None
    if dist is not None:
        merge = D.TorchMerge(dist, f"cuda:{local_rank}", via_host=(cdev == "cpu"))
    # the fused statistics stage: pass 1 in the rollout epilogue, then one
    # streaming pass + compaction + selection (3 merge points under torchrun)
    stage = ex.stats_stage(n, headways, risks, summarize=True, bin_width=2.0)
    last = {}

    step_events = []

    def step(record=False):
        # warm-up and timed steps do the same host work (the first call of
        # anything lazy must not land in the timed region)
        total_steps.zero_()
        e_a = torch.cuda.Event(enable_timing=True)
        e_a.record(stream)
        stage.begin()
        ex.rollout_device(dev_terms, (d, st, hz), sw, total_steps=total_steps, stats=stage)
        nl = ex.last_launches()
        b_ms, r_ms, u_ms = ex.last_stage_ms()
        h0 = time.perf_counter()
        out = stage.finish(d, hz, merge=merge)
        h_ms = 1e3 * (time.perf_counter() - h0)
        e_b = torch.cuda.Event(enable_timing=True)
        e_b.record(stream)
        steps_done = int(total_steps.item())
        if record:
            kernel_ms.append(r_ms)
            stage_ms.append((b_ms, u_ms))
            launches[0] += nl + out["launches"]
            stats_host_ms.append(h_ms)
            step_events.append((e_a, e_b))
        last["out"] = out
        return steps_done

    clocks = ClockSampler(local_rank, args.clock_ms)
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # the statistics end in a host read back per step: keep the collector
    # from pausing the host inside the timed region
    gc.collect()
    gc.disable()
    ev0.record(stream)
    steps_sum = 0
    for _ in range(args.steps):
        steps_sum += step(record=True)
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks.mark_end()
    gc.enable()
    if dist is not None:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=cdev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    value = n_total / (ms_per_step * 1e-3)
    # device span of each timed step and the idle gap before the next one
    spans = [a.elapsed_time(b) for a, b in step_events]
    gaps = [step_events[k][1].elapsed_time(step_events[k + 1][0])
            for k in range(len(step_events) - 1)]

    parity = None
    if not args.skip_parity:
        parity = parity_spot_check(bmc, args, samples, begin, d, st, hz, sw, last["out"], dist,
                                   cdev, headways, risks)
    stats_out = last["out"]
    roll_ms = sum(kernel_ms) / len(kernel_ms)
    # DRAM traffic per kernel from the ncu --set full capture of this same
    # step at 1e8 (tools/profile_headline.py -> tools/ncu_traffic.py); the
    # capture's per-sample bytes scale to this launch when n differs
    traffic, traffic_detail, ncu_k = None, None, {}
    tpath = os.path.join(ROOT, "profiles", "round2_traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        ncu_k = tj["kernels"]
        if "rollout_kernel" in ncu_k:
            bps = ncu_k["rollout_kernel"]["bytes_per_sample"]
            traffic = bps * n
            traffic_detail = {"bytes_per_sample": bps, "algorithmic_bytes_per_sample": 48,
                              "source": tj["source"] + (
                                  "" if int(tj["samples"]) == n else
                                  ", scaled from %d samples to this launch's" % int(tj["samples"]))}
    steps_per_launch = steps_sum / args.steps
    hbm_peak, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
    ppath = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(ppath):
        hbm_peak, hbm_src = float(json.load(open(ppath))["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    bin_ms = sum(b for b, _ in stage_ms) / len(stage_ms)
    unp_ms = sum(u for _, u in stage_ms) / len(stage_ms)

    def stream(bytes_per_sample, ms, what, kernels):
        gbs = bytes_per_sample * n / (ms * 1e-3) / 1e9 if ms > 0 else None
        dram = [ncu_k[k]["bytes_per_sample"] for k in kernels if k in ncu_k]
        return {"what": what, "algorithmic_bytes_per_sample": bytes_per_sample, "ms": ms,
                "gb_per_s": gbs, "frac_of_hbm_peak": gbs / hbm_peak if gbs else None,
                "dram_bytes_per_sample_ncu": sum(dram) if len(dram) == len(kernels) else None}

    hbm_streams = {
        "peak_gb_per_s": hbm_peak, "peak_source": hbm_src,
        "sample_stream": stream(SAMPLE_STREAM_BYTES, bin_ms,
                                "predict + binning scatter: terms in, packed sorted records out",
                                ["predict_kernel", "bin_scatter_kernel"]),
        "rollout": stream(48.0, roll_ms,
                          "rollout kernel: packed records in, packed outputs out -- FP64-bound",
                          ["rollout_kernel"]),
        "result_stream": stream(RESULT_STREAM_BYTES, unp_ms,
                                "unpermute: packed sorted outputs -> index-order outputs",
                                ["unpermute_kernel"]),
        "statistics_passes": {"what": "pass 2 (d + hit_horizon) and compaction (d, hit_horizon "
                                      "on a hit): 18 algorithmic B/sample",
                              "dram_bytes_per_sample_ncu": (
                                  ncu_k["pass2_kernel"]["bytes_per_sample"] +
                                  ncu_k["compact_kernel"]["bytes_per_sample"])
                              if "pass2_kernel" in ncu_k and "compact_kernel" in ncu_k else None,
                              "ms_ncu": (ncu_k["pass2_kernel"]["time_ms"] +
                                         ncu_k["compact_kernel"]["time_ms"])
                              if "pass2_kernel" in ncu_k and "compact_kernel" in ncu_k else None},
    }
    achieved = ALGO_FLOPS_PER_STEP * steps_per_launch / (roll_ms * 1e-3)
    executed = EXEC_FLOPS_PER_STEP * steps_per_launch / (roll_ms * 1e-3)

    # ---- e2e through the run_cuda core (host samples -> host results)
    e2e = None
    if not args.skip_e2e:
        out = np.empty(n, dtype=bmc.RESULT_DTYPE)
        for _ in range(max(1, args.warmup // 2)):
            ex.run(samples, sw, out=out)
        if dist is not None:
            dist.barrier()
        gc.collect()
        gc.disable()
        tt = time.perf_counter()
        reps = max(1, min(args.steps, 3))
        for _ in range(reps):
            rep = ex.run(samples, sw, out=out)
        e2e_s = (time.perf_counter() - tt) / reps
        gc.enable()
        te = torch.tensor([e2e_s], dtype=torch.float64, device=cdev)
        if dist is not None:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": n_total / float(te.item()), "unit": "rollouts/s",
               "h2d_bytes_per_step": rep.h2d_bytes, "d2h_bytes_per_step": rep.d2h_bytes,
               "path": "bmc_cuda_run (run_cuda core): pageable AoS samples -> terms staging "
                       "(host pool) -> pinned -> H2D -> bin+rollout -> D2H -> AoS results",
               "reps": reps}
        del out

    # ---- on-device sampler: bit-identity over the shard + sampling-included e2e
    dsamp = None
    if not args.skip_e2e:
        dsamp = device_sampler(bmc, ex, sw, args, model, n, begin, dev_terms, world, dist, cdev)

    # ---- real-time decision batch (C2): 25k samples, p50/p99 over replays
    latency = None
    feasibility = None
    if rank == 0 and not args.skip_latency:
        latency = realtime(bmc, ex, sw, args, headways, risks)
        feasibility = feasibility_search(bmc, ex, sw, args)

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        cpu = cpu_baseline(args, n_total)

    if rank == 0:
        line = {
            "metric": "MC rollouts/s at 1e8 samples (1/2/4/8 GPU)",
            "value": value, "unit": "rollouts/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (host draw_batch, default UncertaintyModel, bit-identical to "
                    "the reference sampler)",
            "config": {"workload": "C5: %d default-model samples (seed %d), contiguous index "
                                   "shards per GPU; per step: bin + RK4 rollout with statistics "
                                   "pass 1 fused in its epilogue + statistics stage (21 TTC "
                                   "exceedance counts, summarize, 3 min_safe_headway levels) + "
                                   "merge across ranks" % (n_total, args.seed),
                       "samples": n_total, "dt": sw.dt, "t_max": sw.t_max,
                       "parallelism": f"shard{world}",
                       "l2": "no flush: inputs 32 B/sample = %.2f GB per GPU >> 126 MB L2"
                             % (32 * n / 1e9),
                       "sampling_s": sample_s, "clamp_count": clamps},
            "roofline": {"bound": "fp64", "achieved": executed / 1e12, "peak": peak_ops / 1e12,
                         "unit": "TFLOP/s", "frac": executed / peak_ops, "traffic": traffic,
                         "traffic_detail": traffic_detail,
                         "basis": "FP64 ops the kernel executes (DADD/DMUL/DFMA, %d per RK4 "
                                  "step) x RK4 steps executed in the launch (kernel counter) / "
                                  "rollout-kernel CUDA-event time on its stream"
                                  % EXEC_FLOPS_PER_STEP,
                         "kernel": "rollout_kernel", "kernel_ms": roll_ms,
                         "rk4_steps_per_launch": steps_per_launch,
                         "executed_flops_per_step": EXEC_FLOPS_PER_STEP,
                         "algorithmic_equivalent": {
                             "flops_per_step": ALGO_FLOPS_PER_STEP,
                             "tflops": achieved / 1e12, "ratio_to_peak": achieved / peak_ops,
                             "note": "SURVEY 8d counts 57 FP64 ops per step in the reference "
                                     "formulation; the exact per-batch actuator table (-21) and "
                                     "exact-doubling FMAs (-4) leave 32 executed, so this ratio "
                                     "is not a pipe fraction and may exceed 1"},
                         "peak_source": "measured in-run: unfused DADD/DMUL probe "
                                        "(MEASURED_PEAKS.json has no FP64 entry)",
                         "spec_peak_tflops": SPEC_FP64_OPS / 1e12},
            "parity": parity,
            "statistics": {
                "stage": "pass 1 fused into the rollout epilogue (per-CTA shared-memory partials: "
                         "count, horizon, extrema keys, exact sum, exceedance buckets); pass 2 "
                         "(exact m2/m3, histogram, order-statistic buckets); compaction + exact "
                         "selection; merges: %s" % ("torch.distributed (%s)" % (
                             "gloo via host" if cdev == "cpu" else "NCCL")
                                                    if dist is not None else "none (1 process)"),
                "stage_kernels_per_step": stats_out["launches"],
                "fallbacks": stats_out["fallbacks"],
                "merge_calls_per_step": (merge.calls // max(1, args.steps + args.warmup)
                                         if merge is not None else 0),
                "n": stats_out["n"], "horizon_count": stats_out["horizon_count"],
                "ttc_s": ttc,
                "collision_probability": [float(x) for x in stats_out["collision_probability"]],
                "risk_levels": risks,
                "min_safe_headway_m": [float(x) for x in stats_out["min_safe_headway"]],
                "mean": stats_out["summary"]["mean"], "sd": stats_out["summary"]["sd"],
                "median": stats_out["summary"]["median"],
                "skewness": stats_out["summary"]["skewness"]},
            "hbm_streams": hbm_streams,
            "step_breakdown_ms": {"binning": bin_ms, "rollout": roll_ms, "unpermute": unp_ms,
                                  "statistics_wall": sum(stats_host_ms) / len(stats_host_ms),
                                  "step": ms_per_step,
                                  "device_span_per_step": spans,
                                  "gap_between_steps": gaps},
            "e2e": e2e,
            "device_sampler": dsamp,
            "latency_25k": latency,
            "feasibility_530ms": feasibility,
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": launches[0],
        }
        print(json.dumps(line), flush=True)
    stage.close()
    ex.close()


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("BMC_DIST_BACKEND", "nccl")  # gloo: multi-rank tests on one GPU
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    dist = None
    # a process group whenever launched by torchrun (WORLD_SIZE set), also at
    # N=1, so the scaling run's collective path is the one measured
    if "WORLD_SIZE" in os.environ:
        if world > 1:
            # communicator lines ("Init COMPLETE ... nranks N") on stderr, so the
            # rank count of a scaling run can be read off the log tail
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch
        import torch.distributed as dist
        local_rank = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
        else:
            dist.init_process_group(backend)
    try:
        b200_arm(args, rank, world, local_rank, dist, "cpu" if backend == "gloo" else None)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
