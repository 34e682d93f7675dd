#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/kernel_sweep.py --samples 8e6 --quick > gpurun_out/sweep_default.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -c 1 \
   -o gpurun_out/prof_rollout python tools/kernel_sweep.py --profile --samples 8e6 > gpurun_out/ncu_full.log 2>&1
