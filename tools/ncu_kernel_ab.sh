#!/bin/bash
# usage: bash tools/_ab.sh "regex" variant...   (ncu kernel times, in-tree first)
mkdir -p gpurun_out
re=$1; shift
for v in default "$@"; do
  if [ $v = default ]; then unset BMC_LIB_PATH; else export BMC_LIB_PATH=build/ab/$v/libbrakemc_b200.so; fi
  echo "== $v"
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum --clock-control none -k regex:"$re" -c 4 python tools/profile_headline.py --warm 2>&1 | grep -E "^  [a-z]|duration|issue_active|inst_executed" | sed 's/(const .*//'
done
