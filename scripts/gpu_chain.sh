export PYTHONPATH=.
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
UWB_RING_FIXED_ROWS=1 timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_batch.py -m gpu -x -q 2>&1 | tail -1
timeout 300 python scripts/graph_probe.py 2>&1 | tail -1
echo "cfg3 $(timeout 120 python scripts/cfar_probe.py 2>&1 | tail -1)"
for c in 1 6 2; do timeout -s KILL 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/cfg${c}_r01z7.log 2>&1; done
