#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -c 1 \
   -o gpurun_out/prof_rollout python tools/kernel_sweep.py --profile --samples 1e6 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
   --log-file gpurun_out/launches.csv python bench.py --samples 2e6 --steps 2 --warmup 1 \
   --skip-e2e --skip-latency --skip-cpu > gpurun_out/ncu_launch_bench.log 2>&1
