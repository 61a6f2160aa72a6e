export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small and (2048 or 3000 or 5000)" 2>&1 | tail -3
timeout 600 python tools/quick_time.py dpp
FFS_NO_DENSE=1 FFS_QT_M=256 timeout 600 python tools/quick_time.py dpp
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full and dpp" 2>&1 | tail -3
