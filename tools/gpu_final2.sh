#!/bin/bash
export PYTHONPATH=$PWD
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/final2_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/final2_tests.log
STEPS=3 bash tools/gpu_bench_configs.sh peierls > gpurun_out/final2_bench.log 2>&1; tail -c 300 gpurun_out/bench_peierls.json
