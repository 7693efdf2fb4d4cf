# round-2 closing set: full GPU suite, smoke, both bench arms, every config, reports, single-map probes
mkdir -p gpurun_out
TAG=${TAG:-r02s}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_${TAG}.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; tail -1 gpurun_out/smoke_${TAG}.log
timeout -s KILL 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_${TAG}.log 2>&1; tail -1 gpurun_out/bench_ref_${TAG}.log | cut -c1-300
timeout -s KILL 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_${TAG}.log 2>&1; tail -1 gpurun_out/bench_${TAG}.log | cut -c1-300
for c in 1 2 4 5 6; do timeout -s KILL 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${TAG}_cfg$c.log 2>&1; echo "cfg $c rc=$?"; done
OUT=gpurun_out/reports_${TAG} bash scripts/refbench/run.sh > /dev/null 2>&1; ls gpurun_out/reports_${TAG} | wc -l
PYTHONPATH=. timeout -s KILL 300 python scripts/single_map.py > gpurun_out/single_map_${TAG}.log 2>&1
PYTHONPATH=. timeout -s KILL 300 python scripts/single_map_slope.py > gpurun_out/single_map_slope_${TAG}.log 2>&1
PYTHONPATH=. timeout -s KILL 300 python scripts/chain_probe.py > gpurun_out/chain_probe_${TAG}.log 2>&1
timeout 60 ./scripts/micro/_build/chain > gpurun_out/micro_chain_${TAG}.log 2>&1
timeout 60 ./scripts/micro/_build/dsmem_pingpong > gpurun_out/micro_dsmem_${TAG}.log 2>&1
