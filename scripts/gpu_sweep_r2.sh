# knob sweep (tuning build): cfg-3 bench per setting
mkdir -p gpurun_out
run() { echo "== $*"; env "$@" timeout -s KILL 300 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('value',round(d['value'],1),'ms',round(d['ms_per_step'],3),'phases',{k:round(v,3) for k,v in d['phases_ms'].items()})"; }
while read -r line; do [ -n "$line" ] && run $line; done <<< "${SWEEP}"
