#!/bin/bash
# tile-Gram path against the panel kernels over (L, N, N', M) -- the eligibility rule of kmarg_eligible
cd $GRAFT_REPO_ROOT
for s in "1024 32 32 16384" "1024 128 24 16384" "2048 64 64 8192" "2048 256 48 8192" "4096 64 64 8192" "4096 512 64 8192" "4096 512 96 4096" "8192 512 96 4096" "8192 512 128 4096" "16384 1024 64 8192" "16384 1024 96 2048" "16384 1024 128 2048"; do
  timeout 300 python tools/shape_time.py $s --- tile_gram=0 2>&1 | grep "L="
done
