mkdir -p gpurun_out
for f in "" "UWB_SAT_FLAGS=186" "UWB_SAT_FLAGS=58" "UWB_SAT_FLAGS=42" "UWB_SAT_FLAGS=26"; do
  echo "== $f"
  env $f timeout -s KILL 600 python bench.py --config 4 --steps 4 --warmup 2 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', round(d['value'],1), 'global', round(d['global_exact']['value'],2), {k: round(v,3) for k,v in d['global_exact']['phases_ms'].items()})"
  env $f timeout -s KILL 600 python bench.py --config 1 --steps 6 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1 ms', round(d['ms_per_step'],4))"
done
