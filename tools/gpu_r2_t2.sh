#!/bin/bash
cd $GRAFT_REPO_ROOT
python tools/run_once.py dpp 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_dpp.csv python tools/run_once.py dpp 1 > /dev/null 2>&1
python tools/launch_share.py gpurun_out/ll_dpp.csv | head -9
for i in 1 2 3; do timeout 300 python tools/theta_scan.py dpp - 2>&1 | tail -1; done
