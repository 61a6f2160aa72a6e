#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dense_path or gram_draw or small_batches or graph_replay" 2>&1 | tail -6
timeout 900 python tools/theta_scan.py dpp 0.1 0.15 0.2 0.3 gram_draw=3 2>&1 | tail -5
timeout 900 python tools/theta_scan.py peierls 0.2 0.3 0.4 gram_draw=3 2>&1 | tail -4
