#!/bin/bash
# Build A/B variants of the product library with extra nvcc defines for one
# kernel source (diagnostic; run with BMC_LIB_PATH=build/ab/<name>/libbrakemc_b200.so).
#   tools/ab_build.sh mono8 -DBMC_MONO_BLOCK=8                      (bmc_kernels.cu)
#   CU=bmc_fused_stats tools/ab_build.sh p2min2 -DBMC_P2_MINB=2
# SRC=<file> builds another revision of that source (e.g. an older one).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
cu=${CU:-bmc_kernels}
make -s -C "$ROOT/paper_2604_27193_b200/csrc" >/dev/null
out="$ROOT/build/ab/$name"; mkdir -p "$out"
ARCH="-gencode arch=compute_100a,code=sm_100a"
/usr/local/cuda/bin/nvcc $ARCH -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
  -I"$ROOT/include" -I"$ROOT/paper_2604_27193_b200/csrc" --expt-relaxed-constexpr -Xptxas -v "$@" \
  -c "${SRC:-$ROOT/paper_2604_27193_b200/csrc/$cu.cu}" -o "$out/$cu.o" 2> "$out/ptxas.txt"
objs=$(ls "$ROOT"/build/obj/*.o | grep -v "/$cu.o\$")
/usr/local/cuda/bin/nvcc $ARCH -shared -o "$out/libbrakemc_b200.so" "$out/$cu.o" $objs \
  -cudart static -Xlinker --exclude-libs,ALL -lpthread -ldl -lrt
echo "$out/libbrakemc_b200.so"
