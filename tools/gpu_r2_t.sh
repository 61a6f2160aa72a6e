#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dense_path or gram_draw or small_batches or graph_replay or panel_paths or odd_marginal or large_L" 2>&1 | tail -6
timeout 600 python tools/theta_scan.py dpp - gj_pair=0 2>&1 | tail -2
timeout 600 python tools/theta_scan.py peierls - gj_pair=0 2>&1 | tail -2
