export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_frontend.py -x -q 2>&1 | tail -15
echo "fused   $(timeout 300 python scripts/cfg2_probe.py 2>&1 | tail -1)"
echo "general $(UWB_FE_FUSED=0 timeout 300 python scripts/cfg2_probe.py 2>&1 | tail -1)"
timeout 600 ncu -k regex:"frontend|sat_|cfar|sort_" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2g.csv python scripts/cfg2_probe.py > /dev/null 2>&1; echo ncu rc=$?
