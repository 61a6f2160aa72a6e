#!/bin/bash
# round 2: GPU parity suite + quick bench lines of C2 and C5 (8-slice Ozaki default)
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -s > gpurun_out/r2_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
timeout 300 python bench.py --config dw --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_bench_dw.log 2>&1
timeout 600 python bench.py --config dpp --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_bench_dpp.log 2>&1
timeout 600 python bench.py --config peierls --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_bench_peierls.log 2>&1
tail -3 gpurun_out/r2_pytest_gpu.log
