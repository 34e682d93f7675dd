#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/kernel_sweep.py --samples 8e6 --quick > gpurun_out/sweep_default.log 2>&1
timeout 300 python tools/kernel_sweep.py --samples 4e6 --model mixed --quick > gpurun_out/sweep_mixed.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
