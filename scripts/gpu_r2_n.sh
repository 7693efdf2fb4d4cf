mkdir -p gpurun_out
TAG=${TAG:-n}
timeout -s KILL 900 python -m pytest tests/test_gpu_sat_cfar.py tests/test_gpu_batch.py tests/test_gpu_cert.py -m gpu -q -x > gpurun_out/pytest_${TAG}.log 2>&1; tail -2 gpurun_out/pytest_${TAG}.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}.log 2>&1; tail -1 gpurun_out/bench_${TAG}.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('cfg3 value',round(d['value'],1),'phases',{k:round(v,3) for k,v in d['phases_ms'].items()})"
for c in 1 4 6; do timeout -s KILL 600 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_cfg$c.log 2>&1; done
tail -1 gpurun_out/${TAG}_cfg1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1 ms', d['ms_per_step'])"
tail -1 gpurun_out/${TAG}_cfg4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', round(d['value'],1), 'global', d['global_exact']['value'], d['global_exact']['phases_ms'])"
tail -1 gpurun_out/${TAG}_cfg6.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('tableI', [(r['guard'], r['train'], round(r['gpu_integral_ms'],3), round(r['gpu_speedup'],2)) for r in d['table']])"
