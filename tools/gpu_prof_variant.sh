#!/bin/bash
# development: phase-omission timings and one ncu --set full capture of a warp-kernel variant on dw
# usage: bash tools/gpu_prof_variant.sh <variant> <kernel-regex> <report-name>
export PYTHONPATH=$PWD
mkdir -p gpurun_out
v=$1; k=$2; o=$3
bash tools/skip_time.sh $v
FFS_WARP_VARIANT=$v FFS_QT_M=16384 python tools/quick_time.py dw > gpurun_out/plain_$o.log 2>&1 && \
FFS_WARP_VARIANT=$v FFS_QT_M=16384 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
  -o gpurun_out/$o python tools/quick_time.py dw > gpurun_out/ncu_$o.log 2>&1
echo "ncu rc=$?"
