export PYTHONPATH=.
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
echo "fused   $(timeout 300 python scripts/cfg2_probe.py 2>&1 | tail -1)"
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 > gpurun_out/cfg2_r01z2.log 2>&1; tail -1 gpurun_out/cfg2_r01z2.log | cut -c1-600
timeout 600 ncu -k regex:"frontend|sat_|cfar|sort_" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2m.csv python scripts/cfg2_probe.py > /dev/null 2>&1; echo ncu rc=$?
