# end-of-session measurement set: gpu_round.sh + config-4 (tile path) ncu captures
TAG=${TAG:-rX}
export PYTHONPATH=.
mkdir -p gpurun_out
TAG=$TAG bash scripts/gpu_round.sh > gpurun_out/round_${TAG}.txt 2>&1
# config 4 through the tile path (cfg4_probe = the bench's BatchCfar call)
P="python scripts/cfg4_probe.py"
export MODE=tile SLAB_ROWS=512 REPS=1
$P > gpurun_out/cfg4plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}c4.csv $P > /dev/null 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:"sat_systolic|cfar_ws|merge_pass|sort_runs" -s 4 -c 4 -o gpurun_out/prof_${TAG}c4 $P > gpurun_out/ncu_full_${TAG}c4.log 2>&1
echo "cfg4 ncu rc=$?"
