"""The default scene's band map (1024 range bins x 7 band bins, fp64, g 4 b 8, full per-cell outputs):
phases of the integral and the naive backend, as the reference-schema pipeline report times them."""
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar, phase_ms

for cols in (7, 8):
    m = synth.exponential_maps(1, 1024, cols, seed=5, dtype=torch.float64, device="cuda")
    for full in (True, False):
        r = BatchCfar(1, 1024, cols, uwb.CfarParams(4, 8, 1e-3), torch.float64, det_capacity=1024 * cols,
                      want_mask_u8=full, want_thresholds=full)
        for naive in (False, True):
            for _ in range(10):
                r(m, phase_events=True, naive=naive)
            torch.cuda.synchronize()
            ph = phase_ms(1024)[3:].mean(axis=0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                r(m, naive=naive)
            e1.record()
            torch.cuda.synchronize()
            print(f"1024x{cols} full_outputs={full} {'naive' if naive else 'integral'}: sat {ph[0]*1e3:.1f} cfar {ph[1]*1e3:.1f} "
                  f"sort {ph[2]*1e3:.1f} us, call {e0.elapsed_time(e1) / 20 * 1e3:.1f} us", flush=True)
