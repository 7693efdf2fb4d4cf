export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_sat_cfar.py tests/test_gpu_batch.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -2
echo "cfg3 $(timeout 120 python scripts/cfar_probe.py | tail -1)"
echo "cfg3 sentinel $(UWB_SAT_SENTINEL=1 timeout 120 python scripts/cfar_probe.py | tail -1)"
echo "16k $(timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
