#!/bin/bash
# bench lines for C4/C5 + launch list + ncu --set full of one Ozaki GEMM launch (C5)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_parity.py -q -k "dense_path" 2>&1 | tail -1
STEPS=3 bash tools/gpu_bench_configs.sh peierls dpp > gpurun_out/oz_bench.log 2>&1; cat gpurun_out/oz_bench.log | grep rc=
FFS_QT_M=1024 python tools/quick_time.py dpp > gpurun_out/ozp_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/oz_launches_dpp.csv \
  python tools/quick_time.py dpp > gpurun_out/ozp_ncu1.log 2>&1; echo "launches rc=$?"
FFS_QT_M=1024 ncu --set full --clock-control none --import-source on -k regex:ffs_ozaki_gemm -s 30 -c 1 -o gpurun_out/oz_gemm \
  python tools/quick_time.py dpp > gpurun_out/ozp_ncu2.log 2>&1; echo "ncu rc=$?"
