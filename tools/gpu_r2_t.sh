#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dense_path and (opts8 or opts9 or opts10)" 2>&1 | tail -6
echo "rc=$?"
timeout 300 python tools/theta_scan.py dpp - gemm_2sm=4 2>&1 | tail -2
timeout 300 python tools/theta_scan.py peierls - gemm_2sm=4 2>&1 | tail -2
