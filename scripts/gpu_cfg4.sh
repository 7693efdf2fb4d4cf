export PYTHONPATH=.
mkdir -p gpurun_out
for v in "" "UWB_SAT_CPL=2" "UWB_SAT_CPL=1" "UWB_SAT_FLAGS=0" ${EXTRA_AB}; do
  echo "[$v] $(env $v timeout 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
done
REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sat_systolic -s 1 -c 1 -o gpurun_out/prof_cfg4sat python scripts/cfg4_probe.py > gpurun_out/ncu_cfg4sat.log 2>&1; echo ncu rc=$?
