export PYTHONPATH=.
echo "cfg5 default $(timeout 300 python scripts/cfg5_probe.py 2>&1 | tail -1)"
echo "cfg5 thru $(UWB_SAT_FLAGS=0 timeout 300 python scripts/cfg5_probe.py 2>&1 | tail -1)"
echo "cfg5 cpl2 $(UWB_SAT_CPL=2 timeout 300 python scripts/cfg5_probe.py 2>&1 | tail -1)"
echo "cfg5 cpl2 thru $(UWB_SAT_CPL=2 UWB_SAT_FLAGS=0 timeout 300 python scripts/cfg5_probe.py 2>&1 | tail -1)"
echo "cfg5 cpl1 $(UWB_SAT_CPL=1 timeout 300 python scripts/cfg5_probe.py 2>&1 | tail -1)"
