#!/bin/bash
cd $GRAFT_REPO_ROOT
for s in "1024 32 32 16384" "1024 48 48 16384" "1024 128 32 16384" "1024 128 48 16384" "2048 64 64 8192" "4096 64 64 8192" "4096 256 32 8192" "16384 64 64 2048" "512 24 24 16384" "512 64 8 16384"; do
  timeout 300 python tools/shape_time.py $s --- tile_gram=0 --- tile_gram=2 --- tile_gram=3 2>&1 | grep "L="
done
