#!/bin/bash
cd $GRAFT_REPO_ROOT
run() { for w in anderson dw; do timeout 300 python tools/theta_scan.py $w - - 2>&1 | tail -2 | tr '\n' ' '; done; timeout 200 python tools/run_once.py lens 3 >/dev/null 2>&1; echo " <- $1"; }
run v4
cp paper_2109_07358_b200/libffs.so /tmp/libffs_new.so
cp paper_2109_07358_b200/libffs_base.so paper_2109_07358_b200/libffs.so
run base
cp /tmp/libffs_new.so paper_2109_07358_b200/libffs.so
run v4
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not full_size and not dense and not block_step and not tile_gram" 2>&1 | tail -2
