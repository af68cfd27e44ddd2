#!/usr/bin/env bash
# Build libstreamkv_b200.so for sm_100a (cross-compiles without a GPU).
# SKV_INSTRUMENT=1 compiles the prefill instrumentation switches in (timing
# experiments only; the product build ignores SKV_PF_DBG / SKV_PF_TL / SKV_PF_LGT).
set -eo pipefail
cd "$(dirname "$0")"
OUT=paper_2409_09086_b200/libstreamkv_b200.so
SRC=paper_2409_09086_b200/csrc
mkdir -p build
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v"
if [ "${SKV_INSTRUMENT:-0}" = "1" ]; then FLAGS="$FLAGS -DSKV_INSTRUMENT=1"; fi
objs=()
pids=()
for f in decode decode_tc select compact prefill rope tensorops replay skv_abi; do
  nvcc $FLAGS -c $SRC/$f.cu -o build/$f.o 2> build/$f.ptxas.log &
  pids+=($!)
  objs+=(build/$f.o)
done
rc=0
for i in "${!pids[@]}"; do
  if ! wait "${pids[$i]}"; then cat "build/$(basename "${objs[$i]}" .o).ptxas.log"; rc=1; fi
done
[ $rc = 0 ] || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT "${objs[@]}"
echo "built $OUT"
