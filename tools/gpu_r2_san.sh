#!/bin/bash
# compute-sanitizer over every path (tools/san_run.py); TOOL = memcheck | racecheck | synccheck | initcheck
cd $GRAFT_REPO_ROOT
TOOL=${1:-memcheck}
mkdir -p gpurun_out/san_r2
python tools/san_run.py > gpurun_out/san_r2/plain.log 2>&1
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL --print-limit 50 python tools/san_run.py \
  > gpurun_out/san_r2/$TOOL.log 2>&1
echo "rc=$?" >> gpurun_out/san_r2/$TOOL.log
SAN_GRAPH=0 timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL --print-limit 50 python tools/san_run.py \
  > gpurun_out/san_r2/${TOOL}_nograph.log 2>&1
echo "rc=$?" >> gpurun_out/san_r2/${TOOL}_nograph.log
tail -5 gpurun_out/san_r2/$TOOL.log
