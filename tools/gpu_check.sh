#!/bin/bash
# Health check of HEAD on a fresh box: smoke + gpu tests, host CPU facts.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu >> gpurun_out/nproc.txt; ldd --version >> gpurun_out/nproc.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
