# cfg 4 CFAR at one CTA per SM: consumer wait mode
export PYTHONPATH=.
for v in "UWB_RING_DEBUG=0" "UWB_RING_DEBUG=2" "UWB_RING_DEBUG=2 UWB_RING_GROUPS=1" "UWB_RING_DEBUG=1" "UWB_RING_DEBUG=3"; do
  echo "[$v] $(env MODE=tile SLAB_ROWS=512 $v timeout -s KILL 120 python scripts/cfg4_probe.py 2>&1 | tail -1)"
done
for v in "UWB_RING_DEBUG=0" "UWB_RING_DEBUG=2"; do
echo "cfg3 [$v]: $(env $v timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | grep -o '"phases_ms": {[^}]*}')"
done
