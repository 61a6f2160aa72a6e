export PYTHONPATH=$PWD
mkdir -p gpurun_out
for v in mma mma256; do
  echo "== variant $v"
  FFS_WARP_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small or dw" 2>&1 | tail -3
done
for v in default mma mma256; do
  echo "== time $v"
  FFS_WARP_VARIANT=$v python tools/quick_time.py dw
done
