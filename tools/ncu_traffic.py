"""Summarise ncu --set full captures of the headline step into
profiles/round2_traffic.json: per kernel, DRAM bytes read / written per
launch and per sample, duration, and (rollout) the FP64 pipe utilisation.
bench.py reads this file for roofline.traffic and hbm_streams.

python tools/ncu_traffic.py gpurun_out/r2p_rollout.ncu-rep gpurun_out/r2p_hbm.ncu-rep \\
    --samples 1e8 --out profiles/round2_traffic.json
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "time_ms": ("gpu__time_duration.sum", {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3}),
    "dram_read": ("dram__bytes_read.sum", {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0,
                                          "Tbyte": 1e12}),
    "dram_write": ("dram__bytes_write.sum", {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0,
                                            "Tbyte": 1e12}),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", {"%": 1.0}),
    "registers": ("launch__registers_per_thread", {"register/thread": 1.0}),
}
SHORT = ["rollout_kernel", "predict_kernel", "bin_scan_kernel", "bin_scatter_kernel",
         "unpermute_kernel", "finalize1_kernel", "pass2_kernel", "targets_kernel",
         "compact_kernel", "select_kernel"]


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        yield head, units, r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--samples", type=float, default=1e8)
    ap.add_argument("--out", default="profiles/round2_traffic.json")
    a = ap.parse_args()
    n = a.samples
    res = {"samples": n, "source": "ncu --set full --clock-control none of "
                                   "tools/profile_headline.py --warm (the bench step at 1e8); "
                                   + ", ".join(a.reps), "kernels": {}}
    for rep in a.reps:
        for head, units, r in rows_of(rep):
            name = r[head.index("Kernel Name")]
            short = next((s for s in SHORT if s in name), name[:40])
            k = {}
            for key, (metric, scale) in KEYS.items():
                if metric in head:
                    i = head.index(metric)
                    try:
                        k[key] = float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
                    except ValueError:
                        pass
            if "dram_read" in k:
                k["bytes_per_sample"] = (k["dram_read"] + k.get("dram_write", 0.0)) / n
            res["kernels"][short] = k
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    for s, k in res["kernels"].items():
        print(f"{s:20s} {k.get('time_ms', 0):10.3f} ms  {k.get('bytes_per_sample', 0):8.2f} B/sample "
              f"fp64 {k.get('fp64_pipe_pct', 0):5.1f}%")


if __name__ == "__main__":
    main()
