# on the box: single-map timings with each probe library in lib/probe/
L=paper_2012_11077_b200/lib
cp $L/libuwbvital_b200.so /tmp/lib_release.so
for so in $L/probe/lib_*.so /tmp/lib_release.so; do
  cp $so $L/libuwbvital_b200.so 2>/dev/null
  echo "== $(basename $so)"
  python -m pytest tests/test_gpu_sat_cluster.py -q 2>&1 | tail -1
  PYTHONPATH=. python scripts/single_map.py 2>&1 | grep cluster
  PYTHONPATH=. python scripts/chain_probe.py 2>&1 | tail -2
done
cp /tmp/lib_release.so $L/libuwbvital_b200.so
