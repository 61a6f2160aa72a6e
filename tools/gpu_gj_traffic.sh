#!/bin/bash
# DRAM traffic of the batched Gauss-Jordan kernel (C5 full, M = 1024) at several block steps
export PYTHONPATH=$PWD
mkdir -p gpurun_out
FFS_QT_M=1024 timeout 600 python tools/quick_time.py dpp > gpurun_out/gj_plain.log 2>&1; echo "plain rc=$?"
for s in 16 64 96; do
FFS_QT_M=1024 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:ffs_dense_gj -s $s -c 1 --csv --log-file gpurun_out/gj_traffic_$s.csv \
  python tools/quick_time.py dpp > gpurun_out/gj_ncu_$s.log 2>&1; echo "ncu $s rc=$?"
done
