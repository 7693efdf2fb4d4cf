# ncu capture of the two hot kernels at the full config-3 batch (4096 maps),
# after the same command has exited 0 without the profiler.
TAG=${TAG:-r01}
MAPS=${MAPS:-4096}
CMD="python bench.py --maps $MAPS --steps 1 --warmup 1 --no-e2e --no-cpu-baseline ${CMDX}"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-cfar_fused|sat_systolic|cfar_ws}" -s ${KSKIP:-2} -c ${KCOUNT:-2} -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/plain_${TAG}.log | cut -c1-300; tail -5 gpurun_out/ncu_full_${TAG}.log | cut -c1-300
