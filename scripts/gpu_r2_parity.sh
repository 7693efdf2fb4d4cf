mkdir -p gpurun_out
timeout -s KILL 2400 python -m pytest tests/test_gpu_parity_full.py tests/test_gpu_frontend.py tests/test_gpu_batch.py -m gpu -q -x --durations=10 > gpurun_out/pytest_parity_full.log 2>&1; tail -30 gpurun_out/pytest_parity_full.log
