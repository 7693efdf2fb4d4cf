for f in 1 0; do
  echo "== UWB_FUSED=$f"
  UWB_FUSED=$f python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', round(d['value'],1), round(d['ms_per_step'],2), d['phases_ms'])"
  UWB_FUSED=$f python bench.py --config 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
  UWB_FUSED=$f python bench.py --config 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
done
