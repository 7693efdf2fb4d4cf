"""Config 4's global table once (16384 x 16384 fp32, exact path) for ncu."""
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar

m = synth.exponential_maps(1, 16384, 16384, seed=4, dtype=torch.float32, device="cuda")
r = BatchCfar(1, 16384, 16384, uwb.CfarParams(4, 32, 1e-5), torch.float32, det_capacity=1 << 16)
for _ in range(4):
    r(m)
torch.cuda.synchronize()
