export PYTHONPATH=.
for ch in 2 4 8; do echo "$(CHUNKS=$ch timeout 300 python scripts/overlap2_probe.py 2>&1 | tail -1)"; done
for k in 1 2; do echo "satctas=$k $(UWB_SAT_CTAS_PER_SM=$k CHUNKS=4 timeout 300 python scripts/overlap2_probe.py 2>&1 | tail -1)"; done
echo "prio $(PRIO=1 CHUNKS=4 timeout 300 python scripts/overlap2_probe.py 2>&1 | tail -1)"
