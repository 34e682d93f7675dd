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

if len(sys.argv) > 2 and sys.argv[2] == "--list":
    # every launch in order, then the shares of the last step (predict .. select)
    seq = []
    for r in csv.DictReader(lines[start:]):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                 "msecond": 1.0, "s": 1e3, "second": 1e3}[r["Metric Unit"]]
        seq.append((float(r["Metric Value"].replace(",", "")) * scale, r["Kernel Name"][:110]))
    print()
    for ms, name in seq:
        print(f"  {ms:11.4f} ms  {name}")
    last = max(i for i, (_, nm) in enumerate(seq) if "predict_kernel" in nm)
    step = seq[last:]
    tot_step = sum(ms for ms, _ in step)
    print("\n# shares of the last step (predict .. select):")
    for ms, name in step:
        print(f"  {100 * ms / tot_step:7.3f}%  {ms:11.4f} ms  {name.split('(')[0]}")
    print(f"total {tot_step:.3f} ms")
