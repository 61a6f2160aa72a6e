#!/bin/bash
cd $GRAFT_REPO_ROOT
python tools/run_once.py peierls 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_peierls.csv python tools/run_once.py peierls 1 > /dev/null 2>&1
python tools/launch_share.py gpurun_out/ll_peierls.csv > gpurun_out/ll_peierls.txt; head -7 gpurun_out/ll_peierls.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dense_path or gram_draw or small_batches" 2>&1 | tail -3
