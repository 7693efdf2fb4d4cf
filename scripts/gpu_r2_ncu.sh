# Round 2: new GPU tests, then launch list + ncu --set full of the certified path's kernels.
mkdir -p gpurun_out
TAG=${TAG:-r02a}
MAPS=${MAPS:-1024}
timeout -s KILL 1200 python -m pytest ${TESTS:-tests/test_gpu_multirank.py tests/test_gpu_batch.py} -m gpu -q > gpurun_out/pytest_${TAG}.log 2>&1; tail -5 gpurun_out/pytest_${TAG}.log
CMD="python bench.py --maps $MAPS --steps 1 --warmup 3 --no-e2e --no-cpu-baseline ${CMDX}"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-cert_kernel|sat_systolic}" -s ${KSKIP:-2} -c ${KCOUNT:-2} -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/plain_${TAG}.log | cut -c1-400; tail -3 gpurun_out/ncu_full_${TAG}.log | cut -c1-300
