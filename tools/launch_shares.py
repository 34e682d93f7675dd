"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per
kernel count, total device time and share (cold-cache, serialised times)."""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
agg = collections.OrderedDict()
for r in csv.DictReader(lines[start:]):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("bmc::<unnamed>::", "")[:48]
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
             "msecond": 1.0, "s": 1e3, "second": 1e3}[r["Metric Unit"]]
    v = float(r["Metric Value"].replace(",", "")) * scale
    agg.setdefault(name, [0, 0.0])
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for k, v in agg.items() if "probe" not in k)
print(f"{'kernel':50s} {'launches':>8s} {'total ms':>11s} {'share':>7s}  (fp64 probe excluded from share)")
for k, (c, ms) in agg.items():
    share = "" if "probe" in k else f"{ms / tot:7.4f}"
    print(f"{k:50s} {c:8d} {ms:11.3f} {share:>7s}")
