export PYTHONPATH=.
mkdir -p gpurun_out
echo "16k sleep $(timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
echo "16k spin $(UWB_SAT_FLAGS=186 timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
echo "16k sleep-expl $(UWB_SAT_FLAGS=58 timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
UWB_SAT_FLAGS=186 UWB_SAT_TRACE=gpurun_out/trace_spin.txt REPS=1 timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1
