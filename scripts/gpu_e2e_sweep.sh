python -m pytest tests/test_gpu_batch.py -x -q 2>&1 | tail -2
for c in 32 64 128; do python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-chunk $c 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print($c, d['value'], d['e2e'])"; done
