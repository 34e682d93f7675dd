#!/bin/bash
# configs C1/C3/C4 + the default bench (1e8), one box.
mkdir -p gpurun_out
timeout 900 python tools/configs.py --out gpurun_out/round1_configs.json > gpurun_out/configs.log 2>&1
echo "rc=$?" >> gpurun_out/configs.log
timeout 900 python bench.py > gpurun_out/bench_1e8.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_1e8.log
