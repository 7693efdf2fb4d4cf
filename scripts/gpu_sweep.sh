export PYTHONPATH=. MAPS=1024
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
echo "occ4 $(timeout 120 python scripts/cfar_probe.py | tail -1)"
