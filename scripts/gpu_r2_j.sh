mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_sat_cfar.py -m gpu -q -x > gpurun_out/pytest_j.log 2>&1; tail -2 gpurun_out/pytest_j.log
CMD="python bench.py --config 6 --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_cfg6j.log 2>&1 && \
ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"sat_cta" -s 2 -c 1 -o gpurun_out/prof_cfg6j $CMD > gpurun_out/ncu_cfg6j.log 2>&1
echo rc=$?
