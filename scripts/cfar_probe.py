"""Time the CFAR phase alone under the ring kernel's debug probes (no checks)."""
import os
import sys
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar, phase_ms

dev = torch.device("cuda:0")
n = int(os.environ.get("MAPS", "1024"))
maps = torch.empty((n, 1024, 1024), dtype=torch.float32, device=dev)
for c in range(n // 64):
    synth.cfg3_maps(64, seed=c, device=dev, out=maps[c * 64:(c + 1) * 64])
r = BatchCfar(n, 1024, 1024, uwb.CfarParams(2, 8, 1e-4), torch.float32, det_capacity=512, device=dev)
for _ in range(3):
    r(maps, phase_events=True)
torch.cuda.synchronize()
phase_ms(1024)
for _ in range(5):
    r(maps, phase_events=True)
ph = phase_ms(1024)[:5]
print(os.environ.get("UWB_RING_DEBUG", "0"), "cfar ms", ph[:, 1].mean(), "sat ms", ph[:, 0].mean(), flush=True)
