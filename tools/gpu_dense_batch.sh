export PYTHONPATH=$PWD
for S in 512 1024 2048 4096; do echo "S=$S $(FFS_DENSE_S=$S python tools/quick_time.py peierls | cut -c1-70)"; done
for S in 512 1024; do echo "S=$S $(FFS_DENSE_S=$S python tools/quick_time.py dpp | cut -c1-70)"; done
