export PYTHONPATH=$PWD
for v in default tiny4; do
  echo "== $v"; FFS_WARP_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny or 16-4-4-False or 7-3-3" 2>&1 | tail -1
  FFS_WARP_VARIANT=$v python tools/quick_time.py tiny | cut -c1-100
done
