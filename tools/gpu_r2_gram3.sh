#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s > gpurun_out/gram_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gram_pytest.log
tail -5 gpurun_out/gram_pytest.log
