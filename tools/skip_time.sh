#!/bin/bash
# development: time dw with phases skipped (FFS_DEBUG_SKIP bitmask; results are wrong)
export PYTHONPATH=$PWD
for v in "$@"; do
  for s in 0 1 2 4 3 5 6 7; do
    echo "variant $v skip $s $(FFS_WARP_VARIANT=$v FFS_DEBUG_SKIP=$s python tools/quick_time.py dw | python -c 'import json,sys; print(json.load(sys.stdin)["ms"])')"
  done
done
