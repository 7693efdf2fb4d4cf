export PYTHONPATH=.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
echo "16k $(timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
echo "cfg3 $(timeout 120 python scripts/cfar_probe.py | tail -1)"
for c in 4 1 6; do timeout -s KILL 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/cfg${c}_r01z3.log 2>&1; tail -1 gpurun_out/cfg${c}_r01z3.log | cut -c1-250; done
