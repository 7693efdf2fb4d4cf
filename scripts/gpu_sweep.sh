# scratch sweep of the fused kernel (cfar phase = fused kernel)
export PYTHONPATH=. MAPS=1024
echo -n "base: "; python scripts/cfar_probe.py 2>&1 | tail -1
echo -n "base consumers idle: "; UWB_FUSED_DEBUG=1 python scripts/cfar_probe.py 2>&1 | tail -1
echo -n "occ1 ring 160: "; UWB_FUSED_OCC=1 UWB_FUSED_RING=160 python scripts/cfar_probe.py 2>&1 | tail -1
echo -n "occ1 ring 160 consumers idle: "; UWB_FUSED_DEBUG=1 UWB_FUSED_OCC=1 UWB_FUSED_RING=160 python scripts/cfar_probe.py 2>&1 | tail -1
