"""Stall-reason breakdown of one kernel from an ncu report's source page, by SASS region.

    python scripts/ncu_stalls.py REPORT KERNEL_REGEX [region_size]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
step = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ix = {h: hdr.index(h) for h in reasons}
ia = hdr.index("Instructions Executed")
tot = {h: sum(float(r[ix[h]] or 0) for r in data) for h in reasons}
T = sum(tot.values())
print("total samples", T, "instructions", sum(float(r[ia] or 0) for r in data))
for h, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {h:24s} {100 * v / T:5.1f}%")
# per-instruction top stalls
top = sorted(range(len(data)), key=lambda i: -sum(float(data[i][ix[h]] or 0) for h in reasons))[:25]
for i in sorted(top):
    r = data[i]
    s = sum(float(r[ix[h]] or 0) for h in reasons)
    main = max(reasons, key=lambda h: float(r[ix[h]] or 0))
    print(f"{i:5d} {100 * s / T:5.1f}% {main:22s} {r[1][:70]}")
