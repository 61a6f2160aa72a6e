#!/bin/bash
# GJ variant check: dense parity subset + C5/C4 timing
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dense or small_shapes" > gpurun_out/gjq_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gjq_tests.log
FFS_QT_M=1024 timeout 600 python tools/quick_time.py dpp peierls 2>&1 | tee gpurun_out/gjq_time.log
