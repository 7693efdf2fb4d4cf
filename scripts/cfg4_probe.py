"""Phase times of the config-4 map (one 16384^2 fp32 map, g=4, b=32) under env knobs.
SLAB_ROWS=n runs the map as slab-local tables of n owned rows (UWB_SAT_SLAB);
MODE=tile runs row slabs x column bands (UWB_SAT_TILE, UWB_TILE_COLS)."""
import os
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar, phase_ms

R = int(os.environ.get("ROWS", "16384"))
C = int(os.environ.get("COLS", "16384"))
slab = int(os.environ.get("SLAB_ROWS", "0"))
mode = os.environ.get("MODE", "slab" if slab else "global")
full = synth.cfg4_map(seed=4, device="cuda", rows=R, cols=C).unsqueeze(0)
r = BatchCfar(1, R, C, uwb.CfarParams(4, 32, 1e-5), torch.float32, det_capacity=1 << 16,
              sat_mode=mode, slab_rows=slab)
n = int(os.environ.get("REPS", "4"))
for _ in range(n + 1):
    r(full, phase_events=True)
torch.cuda.synchronize()
ph = phase_ms(1024)[1:n + 1]
print(mode + " " + os.environ.get("UWB_TILE_COLS", "") + " slab %d: sat %.3f cfar %.3f sort %.3f ms dets %d" % ((slab,) + tuple(ph[:, :3].mean(0).tolist())
                                                          + (int(r.counts.sum()),)), flush=True)
