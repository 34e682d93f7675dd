"""Small workload touching every kernel of the library, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):
    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
Checks results against the oracle too, so a sanitizer-clean run is also a
correct one."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_27193_b200 as bmc  # noqa: E402
from oracle.pyoracle import Port, World, results_bitwise_equal  # noqa: E402

ex = bmc.CudaExecutor(0)
port = Port()
n = 3000
samples, _ = bmc.draw_batch(bmc.UncertaintyModel.mixed(5), n)
want = port.run(samples, World(), threads=os.cpu_count() or 1)
# host pipeline: binned one-chain / two-chain, per-step and blocked test, index order, no table
for opts in (dict(), dict(ilp=2, block_threads=640), dict(test_block=1), dict(schedule="index"),
             dict(table="global", block_threads=256), dict(table="none"), dict(chunk=700)):
    rep = ex.run(samples, **opts)
    assert results_bitwise_equal(want, rep.results), opts
# device-resident rollout + statistics
terms = bmc.stage_terms(samples)
dev = [torch.from_numpy(terms[i].copy()).cuda() for i in range(4)]
d = torch.empty(n, dtype=torch.float64, device="cuda")
st = torch.empty(n, dtype=torch.int32, device="cuda")
hz = torch.empty(n, dtype=torch.uint8, device="cuda")
ex.rollout_device(dev, (d, st, hz))
ex.sync()
assert np.array_equal(d.cpu().numpy().view(np.uint64), want["stop_distance"].view(np.uint64))
s = ex.summarize(d, hz, 2.0)
c = ex.exceedance_counts(d, hz, [30.0 * (1 + 0.25 * k) for k in range(21)])
h = ex.min_safe_headways(d, hz, [0.05, 0.01])
noisy = ex.exceedance_ttc_noise(d, hz, [1.0 + 0.25 * k for k in range(21)], 30.0, 0.2, 9)
assert noisy.tolist() == port.exceed_ttc_noise(want, [1.0 + 0.25 * k for k in range(21)], 30.0,
                                               0.2, 9).tolist()
# fused statistics stage: pass 1 in the rollout epilogue (and standalone), pass 2,
# targets, compaction, selection, the exact fallbacks (tiny candidate capacity
# and a histogram wider than the device capacity), a statistics decision graph
heads = [30.0 * (1 + 0.25 * k) for k in range(21)]
stage = ex.stats_stage(n, heads, [0.05, 0.01, 0.001], summarize=True, bin_width=2.0)
stage.begin()
ex.rollout_device(dev, (d, st, hz), stats=stage)
fused = stage.finish(d, hz)
stage.close()
one = ex.stats(d, hz, heads, [0.05, 0.01, 0.001], True, 2.0)
assert fused["exceed"].tolist() == one["exceed"].tolist() == c.tolist()
assert fused["summary"]["median"] == one["summary"]["median"] == s["median"]
fb = ex.stats(d, hz, heads, [0.05, 0.01], True, 0.01, hist_cap=64, cand_cap=1)
assert fb["fallbacks"] > 0, fb["fallbacks"]
assert fb["summary"]["median"] == s["median"], (fb["summary"]["median"], s["median"])
assert fb["min_safe_headway"].tolist() == ex.min_safe_headways(d, hz, [0.05, 0.01])
from paper_2604_27193_b200.stats import StatsRequest  # noqa: E402
gs = ex.graph(2000, stats=StatsRequest(heads, [0.05], True, 2.0))
gs.run(samples[:2000])
gs.stats()
gs.close()
# device sampler, model-driven pipeline, decision graphs
ex.draw_device(bmc.UncertaintyModel(seed=3), 5000)
out = np.empty(4000, dtype=bmc.RESULT_DTYPE)
ex.run_model(bmc.UncertaintyModel(seed=4), 4000, out=out, sampler="device")
dd = torch.empty(4000, dtype=torch.float64, device="cuda")
hh = torch.empty(4000, dtype=torch.uint8, device="cuda")
stage = ex.stats_stage(4000, heads, [0.01], summarize=True)
stage.begin()
ex.run_model(bmc.UncertaintyModel(seed=4), 4000, device_out=(dd, None, hh), stats=stage, chunk=1500)
assert stage.finish(dd, hh)["n"] == 4000
stage.close()
g = ex.graph(2000)
g.run(samples[:2000])
g.run_model(bmc.UncertaintyModel(seed=6))
g.close()
ex.fp64_peak(reps=1)
ex.close()
print("sanitize probe OK")
