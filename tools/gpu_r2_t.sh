#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tile_gram or marginal or small_shapes or extreme" 2>&1 | tail -12
timeout 600 python tools/theta_scan.py anderson:marginal - tile_gram=4 2>&1 | tail -2
