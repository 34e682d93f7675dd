#!/bin/bash
# Build A/B variants of the product library with extra nvcc defines for
# bmc_kernels.cu (diagnostic; run with BMC_LIB_PATH=build/ab/<name>/libbrakemc_b200.so).
#   tools/ab_build.sh mono8 -DBMC_MONO_BLOCK=8
# SRC=<file> builds another bmc_kernels.cu (e.g. an older revision).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
make -s -C "$ROOT/paper_2604_27193_b200/csrc" >/dev/null
out="$ROOT/build/ab/$name"; mkdir -p "$out"
ARCH="-gencode arch=compute_100a,code=sm_100a"
/usr/local/cuda/bin/nvcc $ARCH -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
  -I"$ROOT/include" -I"$ROOT/paper_2604_27193_b200/csrc" --expt-relaxed-constexpr -Xptxas -v "$@" \
  -c "${SRC:-$ROOT/paper_2604_27193_b200/csrc/bmc_kernels.cu}" -o "$out/bmc_kernels.o" 2> "$out/ptxas.txt"
objs=$(ls "$ROOT"/build/obj/*.o | grep -v '/bmc_kernels.o$')
/usr/local/cuda/bin/nvcc $ARCH -shared -o "$out/libbrakemc_b200.so" "$out/bmc_kernels.o" $objs \
  -cudart static -Xlinker --exclude-libs,ALL -lpthread -ldl -lrt
echo "$out/libbrakemc_b200.so"
