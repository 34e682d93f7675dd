#!/bin/bash
# Loop-variant round: parity of every loop variant, then the timing sweep.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "loop_variants or criterion1 or mixed" > gpurun_out/pytest_variants.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_variants.log
timeout 600 python tools/kernel_sweep.py --samples 8e6 --unroll > gpurun_out/sweep_unroll_default.log 2>&1
timeout 600 python tools/kernel_sweep.py --samples 4e6 --model mixed --unroll > gpurun_out/sweep_unroll_mixed.log 2>&1
