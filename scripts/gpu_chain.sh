export PYTHONPATH=.
mkdir -p gpurun_out
UWB_SAT_TRACE=gpurun_out/trace_sm.txt REPS=1 ROWS=2048 COLS=16384 timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1
UWB_SAT_TRACE=gpurun_out/trace_sm16.txt REPS=1 ROWS=16384 COLS=16384 timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1
