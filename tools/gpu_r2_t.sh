#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dense_path or panel_paths or odd_marginal or small_batches or large_L" 2>&1 | tail -3
timeout 300 python tools/theta_scan.py dpp - 2>&1 | tail -1
