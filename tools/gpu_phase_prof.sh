#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active --clock-control none --csv --log-file gpurun_out/phase_metrics.csv python tools/kernel_sweep.py --profile --samples 8e6 --table param > gpurun_out/phase_prof.log 2>&1
timeout 900 python tools/kernel_sweep.py --samples 5e7 --phased --reps 2 > gpurun_out/sweep_phased_5e7.log 2>&1
