#!/bin/bash
# parity of the loop variants, then one / two / four chains per thread vs batch size
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "loop_variants or criterion1 or mixed or ragged or known" > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
: > gpurun_out/ilpcmp.log
for n in 1e6 4e6 8e6; do
  timeout 300 python tools/kernel_sweep.py --samples $n --ilpcmp --reps 3 2>&1 | grep -v "probe peak" >> gpurun_out/ilpcmp.log
done
timeout 300 python tools/kernel_sweep.py --samples 4e6 --model mixed --ilpcmp --reps 3 2>&1 | grep -v "probe peak" >> gpurun_out/ilpcmp.log
