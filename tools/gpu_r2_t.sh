#!/bin/bash
cd $GRAFT_REPO_ROOT
export FFS_COMPLEX=1
for s in "1024 64 16 8192" "1024 64 24 8192" "2048 256 32 4096" "4096 512 16 4096" "4096 512 32 4096" "8192 256 32 2048"; do
  timeout 300 python tools/shape_time.py $s --- tile_gram=0 2>&1 | grep "L="
done
