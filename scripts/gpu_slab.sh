# cfg 4 SAT decompositions: global, row slabs, row slabs x column bands (tiles)
export PYTHONPATH=.
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_batch.py -x -q > gpurun_out/tiles_tests.log 2>&1
tail -15 gpurun_out/tiles_tests.log
for v in "MODE=global" "MODE=tile SLAB_ROWS=1024" "MODE=tile SLAB_ROWS=512" "MODE=tile SLAB_ROWS=2048" \
         "MODE=tile SLAB_ROWS=1024 UWB_TILE_COLS=2048" "MODE=tile SLAB_ROWS=512 UWB_TILE_COLS=2048" \
         "MODE=tile SLAB_ROWS=2048 UWB_TILE_COLS=2048" "MODE=tile SLAB_ROWS=1024 UWB_TILE_COLS=512"; do
  echo "[$v] $(env $v timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
done
