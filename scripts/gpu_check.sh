# GPU round trip: parity tests, smoke, a short bench (no profiler).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -40
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} 2>&1 | tail -3
