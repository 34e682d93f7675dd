#!/bin/bash
# Round-2 evidence on the B200 (run under gpurun): the bench line at the
# headline config, the ncu launch list of the same command (short form), ncu
# --set full captures of the rollout kernel and the HBM-bound stages at 1e8
# samples, the C1/C3/C4 configs and the 1e9 stream.  Outputs gpurun_out/r2p_*.
set -x
OUT=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/r2p_launches.csv \
    python bench.py --steps 2 --warmup 1 --skip-e2e --skip-latency --skip-cpu --skip-parity \
    > $OUT/r2p_launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 1 -c 1 \
    -o $OUT/r2p_rollout python tools/profile_headline.py --warm > $OUT/r2p_ncu_rollout.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'predict_kernel|bin_scatter_kernel|unpermute_kernel|pass2_kernel|compact_kernel|select_kernel|targets_kernel|finalize1_kernel|bin_scan_kernel' \
    -s 9 -c 9 -o $OUT/r2p_hbm python tools/profile_headline.py --warm > $OUT/r2p_ncu_hbm.log 2>&1
[ "$1" = "all" ] && timeout 1200 python tools/configs.py > $OUT/r2p_configs.json 2> $OUT/r2p_configs.err
[ "$1" = "all" ] && timeout 900 python tools/run_1e9.py > $OUT/r2p_run_1e9.json 2> $OUT/r2p_run_1e9.err
python tools/ncu_traffic.py $OUT/r2p_rollout.ncu-rep $OUT/r2p_hbm.ncu-rep --out profiles/round2_traffic.json \
    > $OUT/r2p_traffic.txt 2>&1 && cp profiles/round2_traffic.json $OUT/r2p_traffic.json
timeout 900 python bench.py > $OUT/r2p_bench.log 2> $OUT/r2p_bench.err
timeout 600 python bench.py --impl reference > $OUT/r2p_bench_ref.log 2>&1
ls -la $OUT/r2p_*
