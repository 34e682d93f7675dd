#!/bin/bash
# Full default bench (1e8) + its ncu launch list + clocks.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_1e8.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_1e8.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_1e8.csv python bench.py --skip-cpu > gpurun_out/ncu_launch_1e8.log 2>&1
