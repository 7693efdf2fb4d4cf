export PYTHONPATH=.
mkdir -p gpurun_out
RECS=256 timeout 600 ncu -k regex:"frontend" -c 2 --set full --import-source on --clock-control none -o gpurun_out/prof_fe3 python scripts/cfg2_probe.py > gpurun_out/ncu_fe3.log 2>&1; echo ncu rc=$?
