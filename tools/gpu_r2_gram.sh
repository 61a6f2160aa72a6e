#!/bin/bash
# round 2: Gram-draw kernels -- dense-path parity tests, full-size C4/C5 parity, timings
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -k "dense_path or gram or graph_replay or small_batches" > gpurun_out/gram_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gram_pytest.log
tail -5 gpurun_out/gram_pytest.log
for w in dpp peierls; do
  timeout 600 python bench.py --config $w --steps 3 --warmup 3 --no-cpu --no-sweep > gpurun_out/gram_bench_$w.log 2>&1
  tail -c 1500 gpurun_out/gram_bench_$w.log
done
