# A/B probe of the CFAR kernel variants (env knobs), then the CFAR parity tests.
export PYTHONPATH=. MAPS=${MAPS:-1024}
for v in "" "UWB_RING_OCC=3" "UWB_RING_DEBUG=2" "UWB_RING_DEBUG=2 UWB_RING_OCC=3" ${EXTRA_AB}; do
  echo "[$v] $(env $v timeout 120 python scripts/cfar_probe.py 2>&1 | tail -1)"
done
timeout 900 python -m pytest tests -m gpu -x -q ${TESTS:-tests/test_gpu_sat_cfar.py tests/test_gpu_refsuite.py} 2>&1 | tail -3
