#!/bin/bash
# ncu --set full of one batched GJ launch (C5, M = 1024, k0 = 512)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
FFS_QT_M=1024 timeout 600 python tools/quick_time.py dpp > gpurun_out/gjf_plain.log 2>&1; echo "plain rc=$?"
FFS_QT_M=1024 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ffs_dense_gj -s 64 -c 1 -o gpurun_out/gj_full \
  python tools/quick_time.py dpp > gpurun_out/gjf_ncu.log 2>&1; echo "ncu rc=$?"
