#!/bin/bash
# development: cluster/dense parity (small L>=2048 shapes, full C4/C5 and the C5 marginal) + timings
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small and (2048 or 3000 or 2500 or 5000 or 9000 or 6000 or 2000)" 2>&1 | tail -2
for c in ${CFGS:-peierls dpp dpp:m}; do timeout 600 python tools/quick_time.py $c | cut -c1-120; done
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "full and (dpp or peierls)" 2>&1 | tail -2
