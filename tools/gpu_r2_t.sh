#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tile_gram_path or edge_cases or marginal" 2>&1 | tail -5
timeout 300 python tools/theta_scan.py anderson:marginal - 2>&1 | tail -1
timeout 300 python tools/theta_scan.py dpp:marginal - 2>&1 | tail -1
timeout 300 python tools/shape_time.py 65536 64 16 4096 2>&1 | grep "L="
