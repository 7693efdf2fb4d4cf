# ncu of the single-map path: launch list of bench.py --config 6 (Table I) and a full capture of the cluster SAT
# on the Table I shape and on config 4's global table (the chain)
mkdir -p gpurun_out
TAG=${TAG:-r02s}
python bench.py --config 6 --steps 3 --warmup 3 > gpurun_out/plain_cfg6_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg6_${TAG}.csv python bench.py --config 6 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_cfg6_${TAG}.log 2>&1
PYTHONPATH=. ncu --set full --clock-control none --import-source on -k regex:sat_cluster -s 3 -c 1 -o gpurun_out/prof_cluster_${TAG} -f python scripts/single_map_one.py 1024 600 f64 4 8 > gpurun_out/ncu_cluster_${TAG}.log 2>&1
PYTHONPATH=. ncu --set full --clock-control none --import-source on -k regex:sat_cluster -s 2 -c 1 -o gpurun_out/prof_chain_${TAG} -f python scripts/chain_one.py > gpurun_out/ncu_chain_${TAG}.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_chain_${TAG}.log
