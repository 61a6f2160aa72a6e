#!/bin/bash
# development: ncu --set full of the CTA-owner kernel on the C3 marginal workload
export PYTHONPATH=$PWD
python tools/quick_time.py anderson:m > gpurun_out/pg_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ffs_sample_kernel -s 2 -c 1 -o gpurun_out/prof_c3m \
  python tools/quick_time.py anderson:m > gpurun_out/pg_ncu.log 2>&1; echo "rc=$?"
