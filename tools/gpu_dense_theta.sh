#!/bin/bash
# development: dense-path hybrid crossover (FFS_DENSE_THETA = fraction of N' contracted gathered)
export PYTHONPATH=$PWD
for th in ${THETAS:-0 0.2 0.3 0.4 0.5}; do
  for c in ${CFGS:-peierls dpp}; do
    echo "theta=$th $(FFS_DENSE_THETA=$th timeout 600 python tools/quick_time.py $c | cut -c1-80)"
  done
done
