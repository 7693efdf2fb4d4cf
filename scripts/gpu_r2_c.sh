mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_c.log 2>&1; tail -15 gpurun_out/pytest_c.log
CONFIGS="1 6" TAG=cfgsc bash scripts/gpu_configs.sh
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c.log 2>&1; tail -1 gpurun_out/bench_c.log | cut -c1-600
