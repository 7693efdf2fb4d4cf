# scratch sweep of the fused kernel (cfar phase = fused kernel)
export PYTHONPATH=. MAPS=1024
L=paper_2012_11077_b200/lib
cp $L/libuwbvital_b200.so /tmp/base.so
for v in x16; do
[ $v = base ] || cp $L/variants/lib_$v.so $L/libuwbvital_b200.so
echo "$v: $(timeout 120 python scripts/cfar_probe.py 2>&1 | tail -1) | idle $(UWB_FUSED_DEBUG=1 timeout 120 python scripts/cfar_probe.py 2>&1 | tail -1)"
done
cp /tmp/base.so $L/libuwbvital_b200.so
