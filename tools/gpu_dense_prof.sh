#!/bin/bash
# development: launch list of the dense path on dpp (M = FFS_QT_M) + ncu --set full of one GEMM and one step
export PYTHONPATH=$PWD
mkdir -p gpurun_out
export FFS_QT_M=${FFS_QT_M:-256}
python tools/quick_time.py dpp > gpurun_out/dense_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/dense_launches.csv \
  python tools/quick_time.py dpp > gpurun_out/dense_ncu1.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:ffs_dgemm -s 40 -c 1 -o gpurun_out/dense_gemm \
  python tools/quick_time.py dpp > gpurun_out/dense_ncu2.log 2>&1
echo "gemm rc=$?"
ncu --set full --clock-control none --import-source on -k regex:ffs_cluster -s 40 -c 1 -o gpurun_out/dense_step \
  python tools/quick_time.py dpp > gpurun_out/dense_ncu3.log 2>&1
echo "step rc=$?"
