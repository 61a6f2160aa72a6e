#!/bin/bash
# bench lines for the non-default BASELINE.json configs (one JSON line each) -> gpurun_out/bench_<cfg>.json
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for c in "$@"; do
  case $c in
    *:m) name=${c%:m}; extra="--marginal";;
    *) name=$c; extra="";;
  esac
  timeout 900 python bench.py --config $name $extra --steps ${STEPS:-3} --warmup 3 --cpu-budget 10 > gpurun_out/bench_${c/:/_}.json 2> gpurun_out/bench_${c/:/_}.err
  echo "$c rc=$?"; tail -c 600 gpurun_out/bench_${c/:/_}.json
done
