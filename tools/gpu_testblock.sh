#!/bin/bash
# Blocked termination test: parity of every loop variant, then timing (throughput + small batches).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
timeout 600 python tools/kernel_sweep.py --samples 8e6 --testblock > gpurun_out/sweep_tb_default.log 2>&1
timeout 600 python tools/kernel_sweep.py --samples 4e6 --model mixed --testblock > gpurun_out/sweep_tb_mixed.log 2>&1
timeout 600 python tools/kernel_sweep.py --samples 25000 --testblock --reps 20 > gpurun_out/sweep_tb_25k.log 2>&1
