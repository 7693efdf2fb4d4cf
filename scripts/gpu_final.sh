# final check of the session: all GPU tests, smoke, headline bench, cfg 4 / 5
export PYTHONPATH=.
mkdir -p gpurun_out
bash scripts/gpu_check.sh > gpurun_out/check_final.log 2>&1
grep -E "passed|failed|smoke" gpurun_out/check_final.log
tail -1 gpurun_out/check_final.log | cut -c1-200
for c in 4 5; do timeout -s KILL 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfg${c}_final.log 2>&1; tail -1 gpurun_out/cfg${c}_final.log | grep -o '"value": [0-9.]*, "unit": "Gcells/s", "steps"\|"phases_ms": {[^}]*}' ; done
