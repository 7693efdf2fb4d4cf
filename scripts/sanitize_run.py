"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the library once, at sizes the tools finish
in minutes. Run as
    compute-sanitizer --tool <tool> --error-exitcode 9 python scripts/sanitize_run.py
and the exit code / summary line is the evidence (profiles/r02_sanitizer_*.log).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch
    import paper_2012_11077_b200 as uwb
    from paper_2012_11077_b200.batch import BatchCfar, DetectBatch

    g = torch.Generator(device="cuda").manual_seed(7)
    small = torch.empty((3, 96, 200), device="cuda", dtype=torch.float32).exponential_(1.0, generator=g)
    small[:, 40, 50] += 40.0
    p = uwb.CfarParams(2, 8, 1e-3)
    # one CTA per table (small batch, exact) + ring CFAR + sort
    b = BatchCfar(3, 96, 200, p, torch.float32, det_capacity=2048)
    b(small)
    # certified path (certify pass, tap marking, sparse systolic SAT, resolve)
    b(small, certify=True)
    # systolic SAT with the strip chain (more tables than SMs) + ring CFAR
    many = torch.empty((160, 64, 300), device="cuda", dtype=torch.float32).exponential_(1.0, generator=g)
    bm = BatchCfar(160, 64, 300, p, torch.float32, det_capacity=512)
    bm(many, exact=True)
    bm(many, certify=True)
    # per-cell outputs (general CFAR kernel), fused SAT+CFAR, naive backend
    bt = BatchCfar(3, 96, 200, p, torch.float32, det_capacity=2048, want_mask_u8=True, want_thresholds=True)
    bt(small)
    b(small, fused=True)
    b(small, naive=True)
    # tile mode with per-axis windows
    pa = uwb.CfarParams(guard_radius=1, background_radius=4, pfa=1e-3, guard_cols=3, background_cols=16)
    tall = torch.empty((1, 700, 2304), device="cuda", dtype=torch.float32).exponential_(1.0, generator=g)
    bb = BatchCfar(1, 700, 2304, pa, torch.float32, sat_mode="tile", slab_rows=256, det_capacity=4096)
    bb(tall)
    bb(tall, certify=True)
    # front end (fused two-kernel path and the general stage kernels) + CFAR
    recs = torch.randn((2, 64, 256), device="cuda", dtype=torch.float32, generator=g)
    cfg = uwb.PipelineConfig(mean_filter_window=5, fft_length=256, band_low_hz=0.3, band_high_hz=4.0,
                             cfar=uwb.CfarParams(1, 2, 1e-2))
    db = DetectBatch(2, 64, 256, cfg, prf=20.0, dtype=torch.float32, det_capacity=1024)
    db(recs)
    db(recs, general_kernels=True)
    torch.cuda.synchronize()
    print("sanitize_run: done", int(b.counts.sum()), int(bm.counts.sum()), int(bb.counts.sum()),
          int(db.counts.sum()), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
