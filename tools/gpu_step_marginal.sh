export PYTHONPATH=$PWD
FFS_STEP_MARGINAL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full and dpp and 64" 2>&1 | tail -2
for v in 0 1; do echo "step_marginal=$v $(FFS_STEP_MARGINAL=$v python tools/quick_time.py dpp:m | cut -c1-90)"; done
for s in 256 2048 8192; do echo "S=$s $(FFS_DENSE_S=$s FFS_STEP_MARGINAL=1 python tools/quick_time.py dpp:m | cut -c1-90)"; done
