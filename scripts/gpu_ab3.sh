export PYTHONPATH=.
timeout -s KILL 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_tiles.py -x -q 2>&1 | tail -1
for i in 1 2; do timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | grep -o '"value": [0-9.]*, "unit": "Gcells/s", "n_gpus"\|"phases_ms": {[^}]*}'; done
