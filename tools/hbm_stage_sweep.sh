#!/bin/bash
# A/B of the HBM-bound stages around the rollout at 1e8 (run under gpurun):
# scatter tile size, predictor coarse step, output path; bench step breakdown.
for cfg in "BMC_SCATTER_ITEMS=8" "BMC_SCATTER_ITEMS=16" "BMC_SCATTER_ITEMS=32" \
           "BMC_SCATTER_ITEMS=16 BMC_COARSE_STEP_S=0.4" "BMC_DIRECT_OUTPUTS=1"; do
  env $cfg timeout 600 python bench.py --steps 3 --warmup 3 --skip-e2e --skip-latency --skip-cpu \
      --skip-parity > gpurun_out/hbm_sweep.tmp 2>&1
  echo "$cfg $(grep -o '"step_breakdown_ms[^}]*}' gpurun_out/hbm_sweep.tmp | cut -c1-260)"
done
