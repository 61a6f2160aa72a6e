#!/bin/bash
cd $GRAFT_REPO_ROOT
python tools/run_once.py peierls 1 > /dev/null 2>&1
FFS_OPTS=gj_pair=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_peierls_pair.csv python tools/run_once.py peierls 1 > /dev/null 2>&1
python tools/launch_share.py gpurun_out/ll_peierls_pair.csv > gpurun_out/ll_peierls_pair.txt; head -10 gpurun_out/ll_peierls_pair.txt
