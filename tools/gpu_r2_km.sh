#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -k "tile_gram or panel_paths or marginal or small_shapes or extreme or edge or gram" > gpurun_out/km_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/km_pytest.log
tail -5 gpurun_out/km_pytest.log
timeout 600 python tools/theta_scan.py anderson:marginal - > gpurun_out/km_anderson_m.log 2>&1
cat gpurun_out/km_anderson_m.log
timeout 600 python tools/theta_scan.py dpp:marginal - > gpurun_out/km_dpp_m.log 2>&1
cat gpurun_out/km_dpp_m.log
