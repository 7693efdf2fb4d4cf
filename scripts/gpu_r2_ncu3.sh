# ncu of the headline (config 3, 4096 maps) certified path: launch list + full capture of its kernels
mkdir -p gpurun_out
TAG=${TAG:-r02}
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"cert_kernel|sat_systolic|cert_resolve|cert_mark" -s 12 -c 4 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "rc=$?"; tail -1 gpurun_out/plain_${TAG}.log | cut -c1-300
