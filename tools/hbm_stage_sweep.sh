#!/bin/bash
# A/B of the HBM-bound stages around the rollout at 1e8 (run under gpurun):
# bench step breakdown for the in-tree library and the A/B builds given as
# arguments (tools/ab_build.sh names), e.g.  tools/hbm_stage_sweep.sh nopreload
for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib="BMC_LIB_PATH=build/ab/$v/libbrakemc_b200.so"; fi
  env $lib timeout 600 python bench.py --steps 3 --warmup 3 --skip-e2e --skip-latency --skip-cpu \
      --skip-parity > gpurun_out/hbm_sweep.tmp 2>&1
  echo "$v $(grep -o '"step_breakdown_ms[^}]*}' gpurun_out/hbm_sweep.tmp | cut -c1-260)"
done
