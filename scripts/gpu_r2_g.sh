mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_sat_cfar.py tests/test_gpu_batch.py tests/test_gpu_refsuite.py tests/test_gpu_frontend.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/pytest_g.log 2>&1; tail -4 gpurun_out/pytest_g.log
CONFIGS="1 6" TAG=cfgsg bash scripts/gpu_configs.sh 2>&1 | cut -c1-300
python - <<'PY'
import json
d=json.loads(open('gpurun_out/cfgsg_cfg6.log').read().strip().splitlines()[-1])
for r in d['table']: print(r['guard'], r['train'], round(r['gpu_naive_ms'],3), round(r['gpu_integral_ms'],3), round(r['gpu_speedup'],2), r['masks_equal'])
PY
CMD="python bench.py --config 6 --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_cfg6g.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg6g.csv $CMD > /dev/null 2>&1
echo rc=$?
