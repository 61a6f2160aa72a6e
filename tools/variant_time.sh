#!/bin/bash
# time the dw config with each warp-kernel variant
export PYTHONPATH=$PWD
for v in b4s1 b8 b8r200 s2; do
  echo "variant $v"; FFS_WARP_VARIANT=$v python tools/quick_time.py tiny dw
done
FFS_FORCE_GENERIC=1 python tools/quick_time.py dw
