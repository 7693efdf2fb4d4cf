mkdir -p gpurun_out
CMD="python bench.py --config 6 --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_cfg6h.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sat_cta" -s 2 -c 1 -o gpurun_out/prof_cfg6h $CMD > gpurun_out/ncu_cfg6h.log 2>&1
echo rc=$?
