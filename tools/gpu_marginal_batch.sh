export PYTHONPATH=$PWD
for S in 2048 4096 8192; do echo "S=$S $(FFS_DENSE_S=$S python tools/quick_time.py dpp:m | cut -c1-80)"; done
