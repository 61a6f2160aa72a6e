#!/bin/bash
# development: parity (small + dw) and dw timing for each FFS_WARP_VARIANT given
export PYTHONPATH=$PWD
for v in "$@"; do
  echo "== variant $v"
  FFS_WARP_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small or dw" 2>&1 | tail -2
  FFS_WARP_VARIANT=$v python tools/quick_time.py dw
done
