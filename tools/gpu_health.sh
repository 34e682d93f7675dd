#!/bin/bash
# Health check of HEAD on a fresh box: smoke, device-sampler parity, all gpu tests, short bench.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu >> gpurun_out/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_sampler.py -x -q > gpurun_out/pytest_sampler.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_sampler.log
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --samples 2e7 --steps 3 --warmup 3 --latency-reps 100 --cpu-seconds 5 > gpurun_out/bench_2e7.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_2e7.log
