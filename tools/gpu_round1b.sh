#!/bin/bash
# Round refresh: smoke, gpu tests, full 1e8 bench, its launch list, ncu full
# captures of the rollout kernel (8e6) and the on-device sampler.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_1e8.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_1e8.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_1e8.csv python bench.py --skip-cpu --skip-latency > gpurun_out/ncu_launch_1e8.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -c 1 \
   -o gpurun_out/prof_rollout python tools/kernel_sweep.py --profile --samples 8e6 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:draw_terms_kernel -s 1 -c 1 \
   -o gpurun_out/prof_draw python tools/draw_probe.py 1e7 > gpurun_out/ncu_draw.log 2>&1
timeout 300 python tools/draw_probe.py 1e8 > gpurun_out/draw_probe.log 2>&1
timeout 300 ./build/fp64_chain_probe > gpurun_out/fp64_chain_probe.log 2>&1
