#!/bin/bash
# Profiles of the current default build: launch list of the bench command,
# ncu --set full of the rollout kernel (8e6 default samples).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_1e8.csv python bench.py --skip-cpu --skip-latency > gpurun_out/ncu_launch_1e8.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -c 1 \
   -o gpurun_out/prof_rollout python tools/kernel_sweep.py --profile --samples 8e6 > gpurun_out/ncu_full.log 2>&1
