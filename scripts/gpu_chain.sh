export PYTHONPATH=.
mkdir -p gpurun_out
echo "16k $(timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
echo "16k no-touch $(UWB_SAT_FLAGS=122 timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
UWB_SAT_TRACE=gpurun_out/trace_touch.txt REPS=1 ROWS=2048 COLS=16384 timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1
