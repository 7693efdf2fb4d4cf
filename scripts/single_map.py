"""One 1024 x 600 fp64 map (Table I shape) through the batch path, repeatedly."""
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar, phase_ms

m = synth.exponential_maps(1, 1024, 600, seed=77, dtype=torch.float64, device="cuda")
r = BatchCfar(1, 1024, 600, uwb.CfarParams(4, 8, 1e-3), torch.float64, det_capacity=1 << 14)
for _ in range(8):
    r(m, phase_events=True)
torch.cuda.synchronize()
print(phase_ms(1024)[2:8])
