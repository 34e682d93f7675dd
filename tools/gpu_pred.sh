#!/bin/bash
mkdir -p gpurun_out
for h in 0.05 0.1 0.2 0.4; do
  echo "coarse step $h" >> gpurun_out/pred_sweep.log
  BMC_COARSE_STEP_S=$h timeout 300 python tools/kernel_sweep.py --samples 8e6 --quick --reps 2 2>&1 | grep "shared bt=1024 ilp=1" >> gpurun_out/pred_sweep.log
  BMC_COARSE_STEP_S=$h timeout 300 python tools/kernel_sweep.py --samples 4e6 --model mixed --quick --reps 2 2>&1 | grep "shared bt=1024 ilp=1" >> gpurun_out/pred_sweep.log
done
