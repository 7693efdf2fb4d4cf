export PYTHONPATH=.
mkdir -p gpurun_out
UWB_SAT_TRACE=gpurun_out/trace_clk.txt REPS=1 ROWS=2048 COLS=16384 timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1
echo "16k $(timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
echo "16k auto-early $(UWB_SAT_FLAGS=26 timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
