#!/bin/bash
cd $GRAFT_REPO_ROOT
python tools/run_once.py dpp 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ffs_ozaki_gemm2w -c 40 --csv --log-file gpurun_out/ll_exp.csv python tools/run_once.py dpp 1 > /dev/null 2>&1
python tools/launch_share.py gpurun_out/ll_exp.csv | head -3
