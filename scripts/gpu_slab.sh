# cfg 4: tile-mode SAT, CFAR ring row chunks, multi-CTA merge sort
export PYTHONPATH=.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_batch.py tests/test_gpu_fullsize.py -x -q > gpurun_out/tiles_tests.log 2>&1
tail -3 gpurun_out/tiles_tests.log
for v in "MODE=tile SLAB_ROWS=512" "MODE=tile SLAB_ROWS=512 UWB_SORT_ONE_CTA=1" \
         "MODE=tile SLAB_ROWS=512 UWB_RING_ROWS=512" "MODE=tile SLAB_ROWS=512 UWB_RING_ROWS=1024" \
         "MODE=tile SLAB_ROWS=512 UWB_RING_ROWS=2048" "MODE=tile SLAB_ROWS=512 UWB_RING_ROWS=128"; do
  echo "[$v] $(env $v timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
done
