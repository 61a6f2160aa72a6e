#!/bin/bash
# development: dense-path hybrid crossover (FFS_DENSE_THETA = fraction of N' contracted gathered)
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small and (2048 or 3000 or 2500)" 2>&1 | tail -2
for th in ${THETAS:-0 0.2 0.3 0.4 0.5}; do
  for c in ${CFGS:-peierls dpp}; do
    echo "theta=$th $(FFS_DENSE_THETA=$th timeout 600 python tools/quick_time.py $c | cut -c1-100)"
  done
done
