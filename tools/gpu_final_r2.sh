#!/bin/bash
# Round-2 closing evidence on one B200 (run under gpurun; outputs gpurun_out/r2g_*):
# GPU suite + smoke, ncu launch list and --set full captures (rollout, HBM stages)
# -> profiles/round2_traffic.json, then the bench line (reads that traffic), the
# reference arm, configs C1/C3/C4, the 1e9 stream and the sanitizers.
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu > $OUT/r2g_pytest.log 2>&1; echo "rc=$?" >> $OUT/r2g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r2g_smoke.log 2>&1; echo "rc=$?" >> $OUT/r2g_smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r2g_launches.csv \
    python bench.py --steps 2 --warmup 1 --skip-e2e --skip-latency --skip-cpu --skip-parity \
    > $OUT/r2g_launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 1 -c 1 \
    -o $OUT/r2g_rollout python tools/profile_headline.py --warm > $OUT/r2g_ncu_rollout.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'predict_kernel|bin_scatter_kernel|unpermute_kernel|pass2_kernel|compact_kernel|select_kernel|targets_kernel|finalize1_kernel|bin_scan_kernel' \
    -s 9 -c 9 -o $OUT/r2g_hbm python tools/profile_headline.py --warm > $OUT/r2g_ncu_hbm.log 2>&1
python tools/ncu_traffic.py $OUT/r2g_rollout.ncu-rep $OUT/r2g_hbm.ncu-rep --out profiles/round2_traffic.json \
    > $OUT/r2g_traffic.txt 2>&1 && cp profiles/round2_traffic.json $OUT/r2g_traffic.json
timeout 900 python bench.py > $OUT/r2g_bench.log 2> $OUT/r2g_bench.err
timeout 600 python bench.py --impl reference > $OUT/r2g_bench_ref.log 2>&1
timeout 1500 python tools/configs.py --out $OUT/r2g_configs.json > $OUT/r2g_configs.log 2>&1
timeout 900 python tools/run_1e9.py > $OUT/r2g_run_1e9.json 2> $OUT/r2g_run_1e9.err
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_probe.py \
    > $OUT/r2g_sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/r2g_sanitize_$tool.log
done
ls -la $OUT/r2g_*
