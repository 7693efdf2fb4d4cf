import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar, phase_ms
for rows, cols in [(1024, 1024), (1024, 2048), (1024, 3072), (1024, 4096), (1024, 8192), (1024, 16384), (4096, 16384)]:
    m = synth.exponential_maps(1, rows, cols, seed=77, dtype=torch.float32, device="cuda")
    r = BatchCfar(1, rows, cols, uwb.CfarParams(2, 8, 1e-4), torch.float32, det_capacity=1 << 14)
    for _ in range(8):
        r(m, phase_events=True, exact=True)
    torch.cuda.synchronize()
    ph = phase_ms(1024)[3:].mean(axis=0)
    print(f"{rows}x{cols}: sat {ph[0]*1e3:.1f} us  strips {cols//128}", flush=True)
