#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -s -k "dense or peierls or dpp" > gpurun_out/r2e_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2e_pytest.log
timeout 600 python bench.py --config peierls --no-sweep --no-cpu --steps 3 --warmup 3 > gpurun_out/r2e_bench_peierls.log 2>&1
timeout 600 python bench.py --config dpp --no-sweep --no-cpu --steps 3 --warmup 3 > gpurun_out/r2e_bench_dpp.log 2>&1
