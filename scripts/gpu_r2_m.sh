mkdir -p gpurun_out
CMD="python bench.py --config 2 --steps 2 --warmup 2 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain_cfg2m.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"frontend_fft1024|frontend_stats" -s 2 -c 2 -o gpurun_out/prof_cfg2m $CMD > gpurun_out/ncu_cfg2m.log 2>&1
echo rc=$?
