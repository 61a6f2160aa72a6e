#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_lensemble.py -x -q -s > gpurun_out/r2b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
( time timeout 1200 python bench.py --steps 5 --warmup 3 ) > gpurun_out/r2b_bench.log 2> gpurun_out/r2b_bench.err
tail -3 gpurun_out/r2b_pytest.log
