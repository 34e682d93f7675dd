#!/bin/bash
# Round pass: gpu tests, full bench, launch list, ncu full capture of the rollout kernel.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_1e8.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_1e8.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_1e8.csv python bench.py --skip-cpu --skip-e2e > gpurun_out/ncu_launch_1e8.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -c 1 \
   -o gpurun_out/prof_rollout python tools/kernel_sweep.py --profile --samples 8e6 > gpurun_out/ncu_full.log 2>&1
