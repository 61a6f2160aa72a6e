#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dense_path and (opts1 or opts3)" 2>&1 | tail -3
timeout 300 python tools/theta_scan.py dpp - 2>&1 | tail -1
timeout 300 python tools/theta_scan.py peierls - 2>&1 | tail -1
