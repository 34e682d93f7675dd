#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/kernel_sweep.py --samples 8e6 --quick --reps 2 2>&1 | grep "ilp=1" > gpurun_out/pred_sweep.log
timeout 300 python tools/kernel_sweep.py --samples 4e6 --model mixed --quick --reps 2 2>&1 | grep "shared bt=1024 ilp=1" >> gpurun_out/pred_sweep.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
