# final check of the session: all GPU tests, smoke, headline bench, cfg 4 bench + ncu of its kernels
export PYTHONPATH=.
mkdir -p gpurun_out
bash scripts/gpu_check.sh > gpurun_out/check_final.log 2>&1
grep -E "passed|failed|smoke" gpurun_out/check_final.log
timeout -s KILL 900 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/cfg4_final.log 2>&1
export MODE=tile SLAB_ROWS=512 REPS=1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"sat_systolic|cfar_ws" -s 2 -c 2 -o gpurun_out/prof_r01zzc4d python scripts/cfg4_probe.py > gpurun_out/ncu_c4d.log 2>&1; echo "ncu rc=$?"
UWB_RING_DEBUG=1 timeout -s KILL 600 ncu --set full --clock-control none -k regex:"cfar_ws" -s 1 -c 1 -o gpurun_out/prof_r01zzc4p python scripts/cfg4_probe.py > gpurun_out/ncu_c4p.log 2>&1; echo "ncu probe rc=$?"
