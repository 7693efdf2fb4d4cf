mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_frontend.py tests/test_gpu_parity_full.py -k "frontend or cfg2 or detect or fused_front or spectrum or stage" -m gpu -q -x > gpurun_out/pytest_l.log 2>&1; tail -3 gpurun_out/pytest_l.log
CONFIGS="2" TAG=cfgsl bash scripts/gpu_configs.sh 2>&1 | cut -c1-100
tail -1 gpurun_out/cfgsl_cfg2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps({k: d['roofline'][k] for k in ('achieved','frac','launch_ms')}))"
