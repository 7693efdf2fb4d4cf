# on the box: time each probe variant (the release library is restored afterwards)
L=paper_2012_11077_b200/lib
cp $L/libuwbvital_b200.so /tmp/lib_release.so
for v in ${VARIANTS:-0 1 2 4 7}; do
  cp $L/probe/lib_$v.so $L/libuwbvital_b200.so
  echo "== probe $v"; PYTHONPATH=. python scripts/single_map_slope.py 2>&1 | grep -E "256x512|1024x512|1024x1024"
done
cp /tmp/lib_release.so $L/libuwbvital_b200.so
