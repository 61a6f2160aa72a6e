#!/bin/bash
# development: dense-path schedule variants (streams / GEMM tile) on C4 and C5
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small and (2048 or 3000 or 2500)" 2>&1 | tail -2
for v in "1 32" "2 16" "2 32" "1 16"; do
  set -- $v
  for c in ${CFGS:-peierls dpp}; do
    echo "streams=$1 gemm=$2 $(FFS_DENSE_STREAMS=$1 FFS_DENSE_GEMM=$2 timeout 600 python tools/quick_time.py $c)"
  done
done
