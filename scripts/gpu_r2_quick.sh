# quick loop: targeted tests + cfg-3 bench (no e2e / cpu baseline)
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout -s KILL 900 python -m pytest ${TESTS:-tests/test_gpu_cert.py tests/test_gpu_batch.py} -m gpu -q -x > gpurun_out/pytest_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_${TAG}.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_${TAG}.log 2>&1; tail -1 gpurun_out/bench_${TAG}.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('value',round(d['value'],1),'ms',round(d['ms_per_step'],3),'phases',{k:round(v,3) for k,v in d['phases_ms'].items()},'frac',round(d['roofline']['frac'],3), d['roofline']['kernel'], 'step_frac', round(d['step_hbm_frac'],3))"
