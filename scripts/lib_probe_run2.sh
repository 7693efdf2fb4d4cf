# on the box: config 2 with each probe library in lib/probe/
L=paper_2012_11077_b200/lib
cp $L/libuwbvital_b200.so /tmp/lib_release.so
for so in $L/probe/lib_*.so; do
  cp $so $L/libuwbvital_b200.so
  echo "== $(basename $so)"
  python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('cfg2', d['value'], d['ms_per_step'], d['roofline']['launch_ms'])"
done
cp /tmp/lib_release.so $L/libuwbvital_b200.so
