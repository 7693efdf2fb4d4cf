for occ in 4 2 1; do echo "SAT ctas/sm $occ"; UWB_SAT_CTAS_PER_SM=$occ PYTHONPATH=. python scripts/overlap_probe.py 2>&1 | tail -6; done
