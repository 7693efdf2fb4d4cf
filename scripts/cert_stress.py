"""Repeat certified / certified-dense / exact on the same maps; count mismatching runs."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
maps = synth.cfg3_maps(n, seed=11, device="cuda")
p = uwb.CfarParams(2, 8, 1e-4)
e = BatchCfar(n, 1024, 1024, p, torch.float32, det_capacity=1024)
e(maps, exact=True); torch.cuda.synchronize()
ref = e.counts.clone(); refm = e.mask_bits.clone()
c = BatchCfar(n, 1024, 1024, p, torch.float32, det_capacity=1024)
bad = {"sparse": 0, "dense": 0}
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    for mode in ("sparse", "dense"):
        c(maps, dense_tables=(mode == "dense")); torch.cuda.synchronize()
        if not (torch.equal(c.counts, ref) and torch.equal(c.mask_bits, refm)):
            bad[mode] += 1
            d = (c.counts - ref)
            print(it, mode, "count diffs", d[d != 0].tolist()[:8], "maps", torch.nonzero(d).flatten().tolist()[:8])
print("mismatching runs:", bad)
