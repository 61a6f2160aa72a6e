#!/bin/bash
# large-L marginals outside the tile-Gram path (complex, N' > 64, or tile_gram = 0): block-step kernels
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "panel_paths or large_L_marginal or odd_marginal or degenerate" 2>&1 | tail -3
timeout 600 python tools/theta_scan.py dpp:marginal tile_gram=0 gram_draw=3 2>&1 | tail -2
timeout 300 python tools/shape_time.py 16384 1024 128 2048 --- gram_draw=3 2>&1 | grep "L="
