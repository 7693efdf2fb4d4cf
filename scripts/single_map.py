"""Single-map latency (Table I shape 1024 x 600 fp64, cfg 1 shape 256 x 512 fp64, one
1024 x 1024 fp32 map): per-phase device times of the exact path, cluster SAT vs
one-CTA-per-table SAT, and the whole call as seen by CUDA events."""
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar, phase_ms

for (rows, cols, dt, g, b) in [(1024, 600, torch.float64, 4, 8), (256, 512, torch.float64, 2, 8),
                               (1024, 1024, torch.float32, 2, 8), (1024, 8, torch.float64, 4, 8)]:
    m = synth.exponential_maps(1, rows, cols, seed=77, dtype=dt, device="cuda")
    r = BatchCfar(1, rows, cols, uwb.CfarParams(g, b, 1e-4), dt, det_capacity=1 << 14)
    for cta in (False, True):
        for _ in range(8):
            r(m, phase_events=True, cta_tables=cta)
        torch.cuda.synchronize()
        ph = phase_ms(1024)[2:].mean(axis=0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            r(m, cta_tables=cta)
        e1.record()
        torch.cuda.synchronize()
        print(f"{rows}x{cols} {dt} {'cta' if cta else 'cluster'}: phases(ms) {[round(float(x), 4) for x in ph]} "
              f"call {e0.elapsed_time(e1) / 20 * 1e3:.1f} us", flush=True)
