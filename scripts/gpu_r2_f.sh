# sanitizer (one tool per call: TOOL=memcheck|racecheck|synccheck) on scripts/sanitize_run.py, plus the multi-rank logs
mkdir -p gpurun_out
python scripts/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout -s KILL 1500 compute-sanitizer --tool ${TOOL:-memcheck} --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/sanitizer_${TOOL:-memcheck}.log 2>&1
echo "sanitizer rc=$?"; tail -5 gpurun_out/sanitizer_${TOOL:-memcheck}.log
if [ -n "$MULTI" ]; then
  UWB_DIST_BACKEND=gloo timeout -s KILL 900 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/multirank_cfg3_gloo2.log 2>&1; echo "cfg3 rc=$?"; tail -1 gpurun_out/multirank_cfg3_gloo2.log | cut -c1-400
  timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/multirank_cfg3_n1.log 2>&1; echo "cfg3 n1 rc=$?"
  UWB_DIST_BACKEND=gloo timeout -s KILL 900 python bench.py --config 4 --gpus 2 --steps 5 --warmup 3 > gpurun_out/multirank_cfg4_gloo2.log 2>&1; echo "cfg4 rc=$?"; tail -1 gpurun_out/multirank_cfg4_gloo2.log | cut -c1-400
  bash scripts/refbench/run.sh > /dev/null 2>&1; ls gpurun_out/reports
fi
