"""Per-call cost of the device statistics at 2e7 samples and the bench step
timed as bench.py times it (python tools/stat_prof.py, on the B200)."""
import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2604_27193_b200 as bmc
from paper_2604_27193_b200 import distributed as D
n = 20_000_000
ex = bmc.CudaExecutor(0)
m = bmc.UncertaintyModel(seed=3)
terms, _, _ = ex.draw_device(m, n, samples=False)
dev = [terms[i] for i in range(4)]
d = torch.empty(n, dtype=torch.float64, device="cuda"); st = torch.empty(n, dtype=torch.int32, device="cuda"); hz = torch.empty(n, dtype=torch.uint8, device="cuda")
ex.rollout_device(dev, (d, st, hz)); ex.sync()
shard = D.DeviceShard(ex, d, hz); coll = D.Collective(None, "cuda:0")
heads = [30.0 * (1.0 + 0.25 * k) for k in range(21)]
def t(name, f, reps=5):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - a)
    print(f"{name:28s} {1e3*min(ts):8.3f} ms", flush=True)
t("rollout_device", lambda: (ex.rollout_device(dev, (d, st, hz)), ex.sync()))
t("exceedance_counts", lambda: D.exceedance_counts(shard, coll, heads))
t("partials", lambda: shard.partials())
t("moments", lambda: shard.moments(79.0))
t("histogram", lambda: shard.histogram(40.0, 2.0, 60))
t("select_pass", lambda: shard.select_pass(False, 56, [0]))
t("order_stats (median)", lambda: D.order_stats(shard, coll, [n // 2, n // 2 + 1], False))
t("summarize", lambda: D.summarize(shard, coll, 2.0))

# the bench step, timed as bench.py times it (events on the engine stream)
stream = torch.cuda.ExternalStream(ex.stream_handle, device="cuda:0")
total = torch.zeros(1, dtype=torch.int64, device="cuda")
sw = bmc.SimWorld()
def step():
    total.zero_()
    ex.rollout_device(dev, (d, st, hz), sw, total_steps=total)
    ex.last_stage_ms()
    D.exceedance_counts(shard, coll, heads)
    D.summarize(shard, coll, 2.0)
for _ in range(2):
    step()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
w = time.perf_counter()
e0.record(stream)
for _ in range(3):
    step()
    int(total.item())
e1.record(stream)
torch.cuda.synchronize()
print(f"bench-style step: events {e0.elapsed_time(e1) / 3:.3f} ms, wall {1e3 * (time.perf_counter() - w) / 3:.3f} ms")
# the same without the torch zero_ on the default stream
def step2():
    ex.rollout_device(dev, (d, st, hz), sw, total_steps=total)
    ex.last_stage_ms()
    D.exceedance_counts(shard, coll, heads)
    D.summarize(shard, coll, 2.0)
w = time.perf_counter()
e0.record(stream)
for _ in range(3):
    step2()
e1.record(stream)
torch.cuda.synchronize()
print(f"step without zero_/item: events {e0.elapsed_time(e1) / 3:.3f} ms, wall {1e3 * (time.perf_counter() - w) / 3:.3f} ms")
for name, pre, post in [("zero_ only", True, False), ("item only", False, True), ("both", True, True)]:
    for _ in range(2):
        step2()
    torch.cuda.synchronize()
    w = time.perf_counter()
    e0.record(stream)
    for _ in range(3):
        if pre:
            total.zero_()
        step2()
        if post:
            int(total.item())
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"{name:12s}: events {e0.elapsed_time(e1) / 3:.3f} ms, wall {1e3 * (time.perf_counter() - w) / 3:.3f} ms", flush=True)
# zero on the engine stream instead
with torch.cuda.stream(stream):
    w = time.perf_counter()
    e0.record(stream)
    for _ in range(3):
        total.zero_()
        step2()
        int(total.item())
    e1.record(stream)
    torch.cuda.synchronize()
print(f"zero_/item on engine stream: events {e0.elapsed_time(e1) / 3:.3f} ms, wall {1e3 * (time.perf_counter() - w) / 3:.3f} ms")
