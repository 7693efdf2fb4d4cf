# Sweep the CFAR ring look-ahead / consumer-warp count (env knobs read by
# launch_cfar_ring) on a reduced batch; prints one bench line per setting.
MAPS=${MAPS:-1024}
for ncw in 4 2; do
  for ahead in 1 2 3 4; do
    echo "ncw=$ncw ahead=$ahead"
    UWB_RING_NCW=$ncw UWB_RING_AHEAD=$ahead timeout -s KILL 300 python bench.py --maps $MAPS --steps 5 --warmup 3 \
      --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('phases_ms'))" 2>&1 | tail -1
  done
done
