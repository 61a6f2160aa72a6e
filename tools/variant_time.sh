#!/bin/bash
# time the dw config with each warp-kernel variant (FFS_WARP_VARIANT); quick parity check first
export PYTHONPATH=$PWD
for v in "$@"; do
  echo "variant $v"
  FFS_WARP_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "small and (256-32 or 200-60 or 50-17 or 16-4-4-False) or tiny or dw" 2>&1 | tail -1
  FFS_WARP_VARIANT=$v python tools/quick_time.py dw tiny
done
