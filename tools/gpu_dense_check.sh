#!/bin/bash
# development: dense-path parity (small shapes + full C4/C5) and timings vs the cluster path
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small and (2048 or 3000 or 2500 or 5000)" 2>&1 | tail -3
for c in ${CFGS:-peierls dpp}; do
  timeout 600 python tools/quick_time.py $c
  FFS_NO_DENSE=1 FFS_QT_M=${QT_M_OLD:-256} timeout 600 python tools/quick_time.py $c
done
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "full and (${FULLK:-dpp or peierls})" 2>&1 | tail -3
