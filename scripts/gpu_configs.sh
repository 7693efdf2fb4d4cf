# every configuration line (no profiler)
mkdir -p gpurun_out
TAG=${TAG:-cfgs}
for c in ${CONFIGS:-1 2 4 5 6}; do
  echo "== config $c"
  timeout -s KILL 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS} > gpurun_out/${TAG}_cfg$c.log 2>&1; echo rc=$?
  tail -1 gpurun_out/${TAG}_cfg$c.log | cut -c1-1500
done
