#!/bin/bash
# round-end evidence: GPU tests, default bench line, launch list of the bench command, ncu full of the seg kernel
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/final_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/final_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"; cat gpurun_out/final_bench.json
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/final_b2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/final_ncu1.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:ffs_seg -s 3 -c 1 -o gpurun_out/final_seg \
  python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/final_ncu2.log 2>&1; echo "ncu full rc=$?"
