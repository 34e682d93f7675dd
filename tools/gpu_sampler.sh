#!/bin/bash
# Device-sampler round: its parity tests, smoke, a 2e7 bench with the new sections.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sampler.py -x -q > gpurun_out/pytest_sampler.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_sampler.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --samples 2e7 --steps 3 --warmup 3 --latency-reps 100 --cpu-seconds 5 > gpurun_out/bench_2e7.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_2e7.log
