#!/bin/bash
# development: one ncu --set full capture of the dw sampling kernel per FFS_WARP_VARIANT
# usage: bash tools/gpu_ncu_variants.sh <kernel-regex> <tag> <variant>...
export PYTHONPATH=$PWD
mkdir -p gpurun_out
k=$1; tag=$2; shift 2
for v in "$@"; do
  FFS_WARP_VARIANT=$v FFS_QT_M=16384 python tools/quick_time.py dw > gpurun_out/plain_${tag}_$v.log 2>&1 && \
  FFS_WARP_VARIANT=$v FFS_QT_M=16384 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/${tag}_$v python tools/quick_time.py dw > gpurun_out/ncu_${tag}_$v.log 2>&1
  echo "$v ncu rc=$?"
done
