#!/bin/bash
# Round-2 evidence refresh after the monotone-block rollout (run under gpurun):
# e2e pipeline probe with host-phase totals, the ncu launch list of the bench
# command, ncu --set full of the rollout and of the HBM stages at 1e8, the
# traffic summary the bench reads.  Outputs gpurun_out/r2c_*.
set -x
OUT=gpurun_out
mkdir -p $OUT
nproc > $OUT/r2c_host.txt; lscpu >> $OUT/r2c_host.txt 2>&1; free -g >> $OUT/r2c_host.txt
timeout 600 python tools/e2e_probe.py --n 1e8 > $OUT/r2c_e2e_probe.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/r2c_launches.csv \
    python bench.py --steps 2 --warmup 1 --skip-e2e --skip-latency --skip-cpu --skip-parity \
    > $OUT/r2c_launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 1 -c 1 \
    -o $OUT/r2c_rollout python tools/profile_headline.py --warm > $OUT/r2c_ncu_rollout.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'predict_kernel|bin_scatter_kernel|unpermute_kernel|pass2_kernel|compact_kernel|select_kernel|targets_kernel|finalize1_kernel|bin_scan_kernel' \
    -s 9 -c 9 -o $OUT/r2c_hbm python tools/profile_headline.py --warm > $OUT/r2c_ncu_hbm.log 2>&1
python tools/ncu_traffic.py $OUT/r2c_rollout.ncu-rep $OUT/r2c_hbm.ncu-rep --out profiles/round2_traffic.json \
    > $OUT/r2c_traffic.txt 2>&1 && cp profiles/round2_traffic.json $OUT/r2c_traffic.json
ls -la $OUT/r2c_*
