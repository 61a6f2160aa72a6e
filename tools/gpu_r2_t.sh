#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_observe.py -m gpu -x -q -k "pair_correlations" 2>&1 | tail -12
