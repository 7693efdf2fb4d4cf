# cluster SAT: parity, then single-map timings (Table I shape, cfg 1), cfg 1 / cfg 6 lines
mkdir -p gpurun_out
TAG=${TAG:-r02p}
timeout -s KILL 600 python -m pytest tests/test_gpu_sat_cluster.py -x -q > gpurun_out/pytest_cluster_${TAG}.log 2>&1; tail -15 gpurun_out/pytest_cluster_${TAG}.log
timeout -s KILL 900 python -m pytest tests/test_gpu_sat_cfar.py tests/test_gpu_batch.py tests/test_gpu_frontend.py tests/test_gpu_refsuite.py -x -q > gpurun_out/pytest_some_${TAG}.log 2>&1; tail -5 gpurun_out/pytest_some_${TAG}.log
timeout -s KILL 300 python scripts/single_map.py > gpurun_out/single_map_${TAG}.log 2>&1; tail -20 gpurun_out/single_map_${TAG}.log
for c in 1 6; do timeout -s KILL 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${TAG}_cfg$c.log 2>&1; echo "cfg $c rc=$?"; tail -1 gpurun_out/${TAG}_cfg$c.log | cut -c1-1500; done
