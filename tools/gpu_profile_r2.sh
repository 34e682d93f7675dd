#!/bin/bash
# Round-2 evidence on the B200 (run under gpurun): the bench line at the
# headline config, the ncu launch list of the same command (short form), and
# ncu --set full captures of the rollout kernel and the HBM-bound stages at
# 1e8 samples.  Outputs in gpurun_out/r2p_*.
set -x
OUT=gpurun_out
timeout 900 python bench.py > $OUT/r2p_bench.log 2> $OUT/r2p_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/r2p_launches.csv \
    python bench.py --steps 2 --warmup 1 --skip-e2e --skip-latency --skip-cpu --skip-parity \
    > $OUT/r2p_launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 1 -c 1 \
    -o $OUT/r2p_rollout python tools/profile_headline.py --warm > $OUT/r2p_ncu_rollout.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'predict_kernel|bin_scatter_kernel|unpermute_kernel|pass2_kernel|compact_kernel|select_kernel|targets_kernel|finalize1_kernel|bin_scan_kernel' \
    -s 9 -c 9 -o $OUT/r2p_hbm python tools/profile_headline.py --warm > $OUT/r2p_ncu_hbm.log 2>&1
ls -la $OUT/r2p_*
