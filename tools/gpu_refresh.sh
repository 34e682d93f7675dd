#!/bin/bash
# Round refresh after the adaptive pipeline chunk: gpu tests, configs C1/C3/C4, full bench.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/configs.py --out gpurun_out/round1_configs.json > gpurun_out/configs.log 2>&1
echo "rc=$?" >> gpurun_out/configs.log
timeout 900 python bench.py > gpurun_out/bench_1e8.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_1e8.log
