export PYTHONPATH=.
mkdir -p gpurun_out
for c in 4 5; do
timeout -s KILL 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfg${c}_tiles.log 2>&1
tail -1 gpurun_out/cfg${c}_tiles.log | cut -c1-1500
done
UWB_SORT_ONE_CTA=1 timeout -s KILL 900 python bench.py --config 5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-600
