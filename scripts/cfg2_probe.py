"""Batched detect on config-2 records: per-kernel split (for profiling)."""
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import DetectBatch

import os
n = int(os.environ.get("RECS", "1024"))
recs = torch.stack([synth.cfg2_record(seed=2 + i, device="cuda") for i in range(n)]).contiguous()
cfg = uwb.PipelineConfig(mean_filter_window=5, fft_length=1024, cfar=uwb.CfarParams(1, 4, 1e-3))
db = DetectBatch(n, 512, 1024, cfg, prf=20.0, dtype=torch.float32, det_capacity=2048)
for _ in range(3):
    db(recs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    db(recs)
e1.record()
torch.cuda.synchronize()
print("ms per batch of", n, e0.elapsed_time(e1) / 5)
