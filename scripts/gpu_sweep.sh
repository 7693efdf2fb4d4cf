# scratch sweep of the fused kernel (cfar phase = fused kernel)
export PYTHONPATH=. MAPS=1024
for t in $(python -m pytest tests/test_gpu_fused.py --collect-only -q 2>/dev/null | grep "::"); do
  timeout 60 python -m pytest "$t" -x -q 2>&1 | tail -1 | sed "s|^|$t: |"
done
echo -n "base: "; timeout 120 python scripts/cfar_probe.py 2>&1 | tail -1
