MAPS=${MAPS:-1024}
run() {
  echo -n "$* : "
  env "$@" timeout -s KILL 300 python bench.py --maps $MAPS --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})" 2>&1 | tail -1
}
run UWB_X=0
timeout -s KILL 600 python bench.py --config 5 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg5', round(d['value'],2), round(d['ms_per_step'],3), d['phases_ms'])"
timeout -s KILL 600 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg4', round(d['value'],2), round(d['ms_per_step'],3), d['phases_ms'])"
