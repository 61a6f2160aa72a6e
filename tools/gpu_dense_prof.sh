#!/bin/bash
# launch list of the dense path on a config (default dpp, M = FFS_QT_M) + ncu --set full of one
# GEMM and one step launch (development / profiles)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
export FFS_QT_M=${FFS_QT_M:-256}
c=${CFG:-dpp}
python tools/quick_time.py $c > gpurun_out/dense_plain_$c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/dense_launches_$c.csv \
  python tools/quick_time.py $c > gpurun_out/dense_ncu1_$c.log 2>&1
echo "launch list rc=$?"
[ -n "$NO_FULL" ] && exit 0
ncu --set full --clock-control none --import-source on -k regex:ffs_dgemm -s 60 -c 1 -o gpurun_out/dense_gemm_$c \
  python tools/quick_time.py $c > gpurun_out/dense_ncu2_$c.log 2>&1
echo "gemm rc=$?"
ncu --set full --clock-control none --import-source on -k regex:ffs_cluster -s 60 -c 1 -o gpurun_out/dense_step_$c \
  python tools/quick_time.py $c > gpurun_out/dense_ncu3_$c.log 2>&1
echo "step rc=$?"
