#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --samples 2e7 --steps 3 --warmup 3 --latency-reps 200 --cpu-seconds 3 > gpurun_out/bench_2e7.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_2e7.log
