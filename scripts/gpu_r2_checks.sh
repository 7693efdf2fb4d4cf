# the device-checks build (UWB_DEVICE_CHECKS=1, already in lib/): full GPU suite, the sanitizer workload, one cfg-3 step
mkdir -p gpurun_out
strings paper_2012_11077_b200/lib/libuwbvital_b200.so | grep -c "UWB_DCHECK failed" 
timeout -s KILL 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_checks.log 2>&1; tail -3 gpurun_out/pytest_checks.log
timeout -s KILL 600 python scripts/sanitize_run.py > gpurun_out/sanitize_checks.log 2>&1; echo "sanitize_run rc=$?"; tail -2 gpurun_out/sanitize_checks.log
timeout -s KILL 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_checks.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_checks.log | cut -c1-200
for c in 4 5; do timeout -s KILL 600 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/checks_cfg$c.log 2>&1; echo "cfg $c rc=$?"; done
grep -l "UWB_DCHECK failed" gpurun_out/*checks* 2>/dev/null | head
