#!/bin/bash
cd $GRAFT_REPO_ROOT
run() { for w in dpp peierls; do timeout 300 python tools/theta_scan.py $w - 2>&1 | tail -1 | tr '\n' ' '; done; timeout 300 python tools/shape_time.py 8192 128 128 512 tile_gram=0 2>&1 | tail -1 | tr '\n' ' '; FFS_COMPLEX=1 timeout 300 python tools/shape_time.py 4096 128 128 512 tile_gram=0 2>&1 | tail -1 | tr '\n' ' '; echo " <- $1"; }
run v4
cp paper_2109_07358_b200/libffs.so /tmp/libffs_new.so
cp paper_2109_07358_b200/libffs_base.so paper_2109_07358_b200/libffs.so
run base
cp /tmp/libffs_new.so paper_2109_07358_b200/libffs.so
run v4
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dense or block_step or cluster or panel_paths" 2>&1 | tail -2
