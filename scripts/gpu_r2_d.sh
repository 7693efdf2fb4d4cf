mkdir -p gpurun_out
./scripts/micro/lat
timeout -s KILL 300 python scripts/sanitize_run.py 2>&1 | tail -2
CMD="python bench.py --config 6 --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_cfg6.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg6.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sat_cta" -s 2 -c 1 -o gpurun_out/prof_cfg6 $CMD > gpurun_out/ncu_cfg6.log 2>&1
echo rc=$?
