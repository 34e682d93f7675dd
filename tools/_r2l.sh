mkdir -p gpurun_out
bash tools/hbm_stage_sweep.sh nopreload > gpurun_out/r2l_sweep.log 2>&1
for v in default nopreload; do
  if [ $v = default ]; then unset BMC_LIB_PATH; else export BMC_LIB_PATH=build/ab/$v/libbrakemc_b200.so; fi
  echo "== $v"
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"bin_scatter|pass2_kernel|compact_kernel|predict_kernel" -c 4 python tools/profile_headline.py --warm 2>&1 | grep -E "^  [a-z]|duration|bytes"
done > gpurun_out/r2l_ncu.log 2>&1
unset BMC_LIB_PATH
timeout 900 python -m pytest tests/test_gpu_stats_stage.py tests/test_gpu_stats.py tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x > gpurun_out/r2l_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2l_pytest.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_probe.py > gpurun_out/r2l_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_probe.py > gpurun_out/r2l_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_racecheck.log
