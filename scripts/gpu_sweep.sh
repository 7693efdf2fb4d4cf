for o in 4 3; do for d in 0 1 2; do echo -n "occ $o debug $d: "; UWB_RING_OCC=$o UWB_RING_DEBUG=$d PYTHONPATH=. python scripts/cfar_probe.py 2>&1 | tail -1; done; done
