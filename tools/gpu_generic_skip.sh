#!/bin/bash
# development: phase-omission timings of the generic CTA kernel (FFS_DEBUG_SKIP bit0 contraction, bit2 GJ)
export PYTHONPATH=$PWD
for c in ${CFGS:-anderson anderson:m}; do
  for sk in 0 1 4 5; do
    echo "$c skip=$sk $(FFS_DEBUG_SKIP=$sk python tools/quick_time.py $c | cut -c1-60)"
  done
done
