# cfg 4: band tables as separate pitched tables (band-major)
export PYTHONPATH=.
mkdir -p gpurun_out
timeout -s KILL 120 python scripts/cfg4_probe.py > gpurun_out/first.log 2>&1; echo "first rc=$?"; tail -1 gpurun_out/first.log
timeout -s KILL 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_batch.py tests/test_gpu_sat_cfar.py tests/test_gpu_refsuite.py tests/test_gpu_fullsize.py -x -q > gpurun_out/tiles_tests.log 2>&1
echo "tests: $(tail -1 gpurun_out/tiles_tests.log)"
UWB_CFAR_SIMPLE=1 timeout -s KILL 900 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/tiles_tests_simple.log 2>&1
echo "tests (simple CFAR kernel): $(tail -1 gpurun_out/tiles_tests_simple.log)"
for v in "SLAB_ROWS=512" "SLAB_ROWS=1024" "SLAB_ROWS=512 UWB_RING_DEBUG=1" "SLAB_ROWS=512 UWB_RING_GROUPS=1"; do
  echo "[$v] $(env MODE=tile $v timeout -s KILL 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
done
