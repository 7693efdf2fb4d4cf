"""Certified vs exact CFAR path on a config-3 batch: per-phase device times."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_11077_b200 as uwb  # noqa: E402
from paper_2012_11077_b200 import synth  # noqa: E402
from paper_2012_11077_b200.batch import BatchCfar, phase_ms4  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
maps = torch.empty((n, 1024, 1024), dtype=torch.float32, device="cuda")
for c in range(0, n, 64):
    synth.cfg3_maps(min(64, n - c), seed=3 * 1_000_003 + c // 64, device="cuda", out=maps[c:c + 64])
p = uwb.CfarParams(2, 8, 1e-4)
b = BatchCfar(n, 1024, 1024, p, torch.float32, det_capacity=512)
e = BatchCfar(n, 1024, 1024, p, torch.float32, det_capacity=512)
modes = ("exact", "cert", "exact", "cert") if len(sys.argv) < 3 else (sys.argv[2],)
for mode in modes:
    run = (lambda: e(maps, phase_events=True, exact=True)) if mode == "exact" else (lambda: b(maps, phase_events=True))
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    phase_ms4(1024)
    t0 = time.perf_counter()
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / 5
    ph = phase_ms4(1024)
    m = ph.mean(axis=0)
    print(f"{mode}: {t * 1e3:.2f} ms/step wall, phases certify {m[0]:.3f} sat {m[1]:.3f} cfar {m[2]:.3f} "
          f"sort {m[3]:.3f} -> {n * 2**20 / (m.sum() / 1e3) / 1e9:.1f} Gcell/s", flush=True)
ok = torch.equal(b.mask_bits, e.mask_bits) and torch.equal(b.counts, e.counts)
st = b.cert_status.cpu().numpy()
print("masks/counts equal:", ok, "status nonzero:", int((st != 0).sum()),
      "detections:", int(b.counts.sum()), "ties:", int(b.tie_counts.clamp(min=0).sum()))
