#!/bin/bash
# development: CTA-owner kernel parity (small shapes, full C3) and C3 timings
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small or anderson or edge" 2>&1 | tail -2
for c in anderson anderson:m; do python tools/quick_time.py $c | cut -c1-100; done
