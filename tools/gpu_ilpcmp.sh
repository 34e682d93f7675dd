#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ilpcmp.log
for n in 5e4 1e5 2.5e5 5e5 1e6 2e6 4e6; do
  timeout 300 python tools/kernel_sweep.py --samples $n --ilpcmp --reps 5 2>&1 | grep -v "probe peak" >> gpurun_out/ilpcmp.log
done
