#!/bin/bash
# development: persistent step kernel with panel prefetch vs one cluster per sample
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "(small and (2048 or 3000 or 2500)) or dense_path or large_L or degenerate" 2>&1 | tail -2
for c in peierls dpp; do
  echo "prefetch $(timeout 600 python tools/quick_time.py $c | cut -c1-80)"
  echo "plain    $(FFS_STEP_PREFETCH=0 timeout 600 python tools/quick_time.py $c | cut -c1-80)"
done
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "full and (dpp or peierls)" 2>&1 | tail -2
