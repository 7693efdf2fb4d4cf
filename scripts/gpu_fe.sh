export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_frontend.py tests/test_gpu_refsuite.py -x -q 2>&1 | tail -2
echo "fused   $(timeout 300 python scripts/cfg2_probe.py 2>&1 | tail -1)"
timeout 600 ncu -k regex:"frontend" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2n.csv python scripts/cfg2_probe.py > /dev/null 2>&1; echo ncu rc=$?
