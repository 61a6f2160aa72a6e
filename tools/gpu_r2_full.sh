#!/bin/bash
# full GPU suite (normal + checked build)
cd $GRAFT_REPO_ROOT
timeout 3000 python -m pytest tests -m gpu -x -q -s > gpurun_out/full_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/full_pytest.log
tail -4 gpurun_out/full_pytest.log
