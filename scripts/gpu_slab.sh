# detection sort: merge passes skip finished lists
export PYTHONPATH=.
timeout -s KILL 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_batch.py tests/test_gpu_fullsize.py tests/test_gpu_sat_cfar.py -x -q > gpurun_out/sort_tests.log 2>&1
echo "tests: $(tail -1 gpurun_out/sort_tests.log)"
for v in "SLAB_ROWS=512" "SLAB_ROWS=512 UWB_SORT_ONE_CTA=1"; do
  echo "[$v] $(env MODE=tile $v timeout -s KILL 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
done
echo "cfg5: $(timeout -s KILL 300 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | grep -o '"value": [0-9.]*, "unit": "Gcells/s", "steps"')"
