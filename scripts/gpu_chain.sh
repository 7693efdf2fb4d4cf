export PYTHONPATH=.
for c in 128 256 512 1024 4096 16384; do
  echo "cols=$c $(COLS=$c timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
done
echo "cfg3 $(timeout 120 python scripts/cfar_probe.py | tail -1)"
timeout 900 python -m pytest tests -m gpu -x -q ${TESTS:-tests/test_gpu_sat_cfar.py tests/test_gpu_fused.py} 2>&1 | tail -2
