#!/bin/bash
# Phased-rollout round: parity first (stop on failure), then timing.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
timeout 600 python tools/kernel_sweep.py --samples 8e6 --phased > gpurun_out/sweep_phased_default.log 2>&1
timeout 600 python tools/kernel_sweep.py --samples 4e6 --model mixed --phased > gpurun_out/sweep_phased_mixed.log 2>&1
