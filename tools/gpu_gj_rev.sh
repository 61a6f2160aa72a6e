#!/bin/bash
# reverse-order GJ step (3): parity of the dense paths, C4/C5 timing, GJ traffic at k0 = 512
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense or small_shapes or full_size" > gpurun_out/gjrev_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gjrev_tests.log
FFS_QT_M=1024 timeout 600 python tools/quick_time.py dpp > gpurun_out/gjrev_dpp.log 2>&1; cat gpurun_out/gjrev_dpp.log
timeout 600 python tools/quick_time.py peierls > gpurun_out/gjrev_peierls.log 2>&1; cat gpurun_out/gjrev_peierls.log
FFS_QT_M=1024 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:ffs_dense_gj -s 64 -c 1 --csv --log-file gpurun_out/gjrev_traffic_64.csv \
  python tools/quick_time.py dpp > gpurun_out/gjrev_ncu_64.log 2>&1; echo "ncu rc=$?"
