"""One single-map exact-path shape for ncu: rows cols dtype guard train."""
import sys
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar

rows, cols = int(sys.argv[1]), int(sys.argv[2])
dt = torch.float64 if sys.argv[3] == "f64" else torch.float32
g, b = int(sys.argv[4]), int(sys.argv[5])
m = synth.exponential_maps(1, rows, cols, seed=77, dtype=dt, device="cuda")
r = BatchCfar(1, rows, cols, uwb.CfarParams(g, b, 1e-4), dt, det_capacity=1 << 14)
for _ in range(6):
    r(m)
torch.cuda.synchronize()
