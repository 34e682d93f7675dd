#!/bin/bash
# First GPU pass: smoke, gpu tests, kernel sweep, short bench.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu >> gpurun_out/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python tools/kernel_sweep.py --samples 4e6 > gpurun_out/sweep_default.log 2>&1
timeout 300 python tools/kernel_sweep.py --samples 2e6 --model mixed > gpurun_out/sweep_mixed.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --samples 2e7 --steps 3 --warmup 3 --latency-reps 100 --cpu-seconds 5 > gpurun_out/bench_2e7.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_2e7.log
