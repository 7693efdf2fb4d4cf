# Round-2 GPU round trip: parity tests, smoke, bench (no profiler). Logs in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
tail -30 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; tail -3 gpurun_out/bench.log
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --exact --no-e2e --no-cpu-baseline > gpurun_out/bench_exact.log 2>&1; tail -3 gpurun_out/bench_exact.log
