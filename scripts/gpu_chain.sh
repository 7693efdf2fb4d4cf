export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_fullsize.py tests/test_gpu_sat_cfar.py -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 900 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/cfg5_r01z6.log 2>&1; tail -1 gpurun_out/cfg5_r01z6.log | cut -c1-200
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/cfg3_r01z6.log 2>&1; tail -1 gpurun_out/cfg3_r01z6.log | cut -c1-200
