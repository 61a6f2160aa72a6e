#!/bin/bash
cd $GRAFT_REPO_ROOT
run() { for w in anderson:marginal dpp:marginal; do timeout 300 python tools/theta_scan.py $w - - 2>&1 | tail -2 | tr '\n' ' '; done; echo " <- $1"; }
run v4
cp paper_2109_07358_b200/libffs.so /tmp/libffs_new.so
cp paper_2109_07358_b200/libffs_base.so paper_2109_07358_b200/libffs.so
run base
cp /tmp/libffs_new.so paper_2109_07358_b200/libffs.so
run v4
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tile_gram_path and not complex" 2>&1 | tail -2
