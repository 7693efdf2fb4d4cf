mkdir -p gpurun_out
CONFIGS="1 4 5" TAG=cfgsb bash scripts/gpu_configs.sh
CMD="python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_cfg1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg1.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sat_systolic|cert_kernel" -s 4 -c 2 -o gpurun_out/prof_cfg1 $CMD > gpurun_out/ncu_cfg1.log 2>&1
echo rc=$?
