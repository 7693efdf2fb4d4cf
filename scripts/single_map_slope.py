"""Per-step cost of the single-map SAT: SAT phase time against rows at fixed columns."""
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar, phase_ms

for cols, dt in [(8, torch.float64), (512, torch.float64), (1024, torch.float32)]:
    prev = None
    for rows in (256, 512, 1024, 2048, 4096):
        m = synth.exponential_maps(1, rows, cols, seed=77, dtype=dt, device="cuda")
        r = BatchCfar(1, rows, cols, uwb.CfarParams(2, 8, 1e-4), dt, det_capacity=1 << 14)
        for _ in range(12):
            r(m, phase_events=True)
        torch.cuda.synchronize()
        ph = phase_ms(1024)[4:].mean(axis=0)
        slope = "" if prev is None else f" slope {(ph[0] - prev[1]) * 1e6 / (rows - prev[0]):.1f} ns/row"
        print(f"{rows}x{cols} {dt}: sat {ph[0] * 1e3:.1f} us cfar {ph[1] * 1e3:.1f} sort {ph[2] * 1e3:.1f}{slope}", flush=True)
        prev = (rows, ph[0])
