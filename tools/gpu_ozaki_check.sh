#!/bin/bash
# development: dense path with the Ozaki GEMM: parity (small dense shapes, schedules, full C4/C5) and timings
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "(small and (2048 or 3000 or 2500)) or dense_path" 2>&1 | tail -3
for c in peierls dpp; do
  echo "ozaki $(timeout 600 python tools/quick_time.py $c | cut -c1-90)"
  echo "dmma  $(FFS_DENSE_GEMM=dmma timeout 600 python tools/quick_time.py $c | cut -c1-90)"
done
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "full and (dpp or peierls)" 2>&1 | tail -3
