#!/usr/bin/env bash
# Build libstreamkv_b200.so for sm_100a (cross-compiles without a GPU).
set -eo pipefail
cd "$(dirname "$0")"
OUT=paper_2409_09086_b200/libstreamkv_b200.so
SRC=paper_2409_09086_b200/csrc
mkdir -p build
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v"
objs=()
for f in decode decode_tc select compact prefill rope skv_abi; do
  nvcc $FLAGS -c $SRC/$f.cu -o build/$f.o 2> build/$f.ptxas.log || { cat build/$f.ptxas.log; exit 1; }
  objs+=(build/$f.o)
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT "${objs[@]}"
echo "built $OUT"
