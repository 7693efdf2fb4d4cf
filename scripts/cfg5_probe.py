"""SAT / CFAR phase times of config-5 maps (64 K-clutter maps 8192x2048, window (1,3,4,16))."""
import os
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar, phase_ms

n = int(os.environ.get("MAPS", "64"))
maps = torch.cat([synth.cfg5_maps(8, seed=5000 + b, device="cuda", rows=8192, cols=2048) for b in range(n // 8)])
p = uwb.CfarParams(1, 4, 1e-3, guard_cols=3, background_cols=16)
r = BatchCfar(n, 8192, 2048, p, torch.float32, det_capacity=1 << 15)
for _ in range(4):
    r(maps, phase_events=True)
torch.cuda.synchronize()
ph = phase_ms(1024)[1:4]
print("sat %.3f cfar %.3f sort %.3f ms" % tuple(ph[:, :3].mean(0).tolist()), flush=True)
