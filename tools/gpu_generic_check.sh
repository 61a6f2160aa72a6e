#!/bin/bash
# development: CTA-owner paths (one-launch kernel vs block-step + batched GJ) parity and timings
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small or anderson or edge" 2>&1 | tail -2
for v in 1 0; do
  for c in anderson anderson:m; do echo "step=$v $(FFS_STEP_GENERIC=$v python tools/quick_time.py $c | cut -c1-100)"; done
done
