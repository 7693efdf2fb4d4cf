"""Full-size parity on every BASELINE.json configuration (north_star: "detection
masks matching the CPU oracle on all five configs").

Every map at its stated size is compared with the CPU checker, map-parallel on
the host cores (each ctypes call releases the GIL):

* config 3: all 4096 maps of 1024 x 1024 against the reference's own
  cfar2d_integral (oracle/_ref = /root/reference/proj/src/cfar.cpp:218-227),
  masks, detection lists (row, col, value, threshold bit for bit) and counts;
* config 4: the whole 16384 x 16384 map on the reference-exact global path
  against cfar2d_integral(map, params, nproc); the tile path (UWB_SAT_TILE,
  the bench's config-4 line) against that result outside the tie band, with the
  tie-band cells it reports (|cut - T| <= 1e-6 T) covering every difference;
* config 5: all 64 maps of 8192 x 2048 for the four (window, Pfa) runs against
  the plain-C restatement with per-axis windows (the reference's CfarParams has
  one radius per kind, cfar.hpp:22-30; the restatement equals it when the axes
  agree, tests/test_oracle.py);
* config 2: a 1024-record batch through the batched device detect() against the
  reference detect() (pipeline.cpp:246-275) record by record;
* config 1: the single fp64 256 x 512 map (tests/test_gpu_sat_cfar.py also
  checks its table).
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from tests.helpers import assert_bitwise

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = max(1, len(os.sched_getaffinity(0)))


def _pack(mask_u8: np.ndarray) -> np.ndarray:
    """Reference u8 mask -> the device's little-endian u32 words per row."""
    rows, cols = mask_u8.shape
    words = (cols + 31) // 32
    padded = np.zeros((rows, words * 32), np.uint8)
    padded[:, :cols] = mask_u8
    return np.packbits(padded, axis=1, bitorder="little").view(np.uint32)


def _same_list(got, exp, what):
    assert len(got) == len(exp), f"{what}: {len(got)} detections vs {len(exp)}"
    for f in ("row", "col"):
        assert np.array_equal(got[f].astype(np.uint64), np.asarray(exp[f]).astype(np.uint64)), f"{what}: {f}"
    assert_bitwise(got["value"], np.asarray(exp["value"]), f"{what}: values")
    assert_bitwise(got["threshold"], np.asarray(exp["threshold"]), f"{what}: thresholds")


def test_cfg3_every_map_vs_reference(uwb, ref, cuda):
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    n, R, C = 4096, 1024, 1024
    maps = torch.empty((n, R, C), dtype=torch.float32, device=cuda)
    for c in range(n // 64):  # the bench's generator blocks
        synth.cfg3_maps(64, seed=3 * 1_000_003 + c, device=cuda, out=maps[c * 64:(c + 1) * 64])
    b = BatchCfar(n, R, C, uwb.CfarParams(2, 8, 1e-4), torch.float32, det_capacity=512, device=cuda)
    b(maps)
    torch.cuda.synchronize()
    b.check_inputs()
    assert (b.cert_status.cpu().numpy() == 0).all(), "config 3 maps all run the certified path"
    counts = b.detection_counts()
    bad = []
    with ThreadPoolExecutor(THREADS) as pool:
        for c0 in range(0, n, 256):
            host = maps[c0:c0 + 256].cpu().numpy()
            bits = b.mask_bits[c0:c0 + 256].cpu().numpy().view(np.uint32)

            def one(i, host=host, bits=bits, c0=c0):
                r = ref.cfar2d(host[i].astype(np.float64), 2, 8, 1e-4, "integral", det_cap=4096,
                               thresholds=False)
                ok = np.array_equal(_pack(r.mask), bits[i]) and len(r.detections) == counts[c0 + i]
                return c0 + i, ok, r.detections
            for k, ok, exp in pool.map(one, range(host.shape[0])):
                if not ok:
                    bad.append(k)
                    continue
                _same_list(b.detections(k), exp, f"map {k}")
    assert not bad, f"{len(bad)} of {n} maps differ from the reference: {bad[:10]}"


def _cfg4_map(cuda):
    from paper_2012_11077_b200 import synth
    return synth.cfg4_map(seed=4, device=cuda, rows=16384, cols=16384).unsqueeze(0).contiguous()


def test_cfg4_global_and_tile_paths_vs_reference(uwb, ref, cuda):
    from paper_2012_11077_b200.batch import BatchCfar
    R = C = 16384
    p = uwb.CfarParams(4, 32, 1e-5)
    m = _cfg4_map(cuda)
    g = BatchCfar(1, R, C, p, torch.float32, det_capacity=1 << 16, device=cuda)
    g(m)
    torch.cuda.synchronize()
    g.check_inputs()
    assert int(g.cert_status[0]) == 0
    host = m[0].cpu().numpy().astype(np.float64)
    r = ref.cfar2d(host, 4, 32, 1e-5, "integral", threads=THREADS, det_cap=1 << 16, thresholds=False)
    got_bits = g.mask_bits[0].cpu().numpy().view(np.uint32)
    assert np.array_equal(got_bits, _pack(r.mask)), "global path mask vs reference"
    _same_list(g.detections(0), r.detections, "config 4 global path")
    g_ties = g.tie_band(0)

    # tile path (the bench's config-4 line): 512-row slabs x 1024-column bands,
    # one table per tile; equal to the global result outside the tie band
    t = BatchCfar(1, R, C, p, torch.float32, sat_mode="tile", slab_rows=512, det_capacity=1 << 16,
                  tie_capacity=1 << 12, device=cuda)
    t(m)
    torch.cuda.synchronize()
    assert int(t.cert_status[0]) == 0
    t_bits = t.mask_bits[0].cpu().numpy().view(np.uint32)
    diff = np.argwhere(np.unpackbits((t_bits ^ got_bits).view(np.uint8), axis=1, bitorder="little")[:, :C])
    ties = t.tie_band(0)
    tie_cells = set(zip(ties["row"].tolist(), ties["col"].tolist())) | \
        set(zip(g_ties["row"].tolist(), g_ties["col"].tolist()))
    outside = [tuple(x) for x in diff.tolist() if tuple(x) not in tie_cells]
    assert not outside, f"tile path differs from the global table outside the tie band at {outside[:10]}"
    assert abs(int(t.counts[0]) - int(g.counts[0])) <= len(diff)


def test_cfg5_every_map_and_run_vs_restatement(uwb, oracle, cuda):
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    n, R, C = 64, 8192, 2048
    maps = torch.empty((n, R, C), dtype=torch.float32, device=cuda)
    for blk in range(n // 8):  # the bench's generator blocks
        synth.cfg5_maps(8, seed=5_000 + blk, device=cuda, rows=R, cols=C, out=maps[blk * 8:(blk + 1) * 8])
    runs = [((1, 3), (4, 16), 1e-3), ((1, 3), (4, 16), 1e-5), ((3, 1), (16, 4), 1e-3), ((3, 1), (16, 4), 1e-5)]
    host = maps.cpu().numpy()
    with ThreadPoolExecutor(THREADS) as pool:
        for (gr, gc), (br, bc), pfa in runs:
            p = uwb.CfarParams(guard_radius=gr, background_radius=br, pfa=pfa, guard_cols=gc, background_cols=bc)
            b = BatchCfar(n, R, C, p, torch.float32, det_capacity=1 << 15, device=cuda)
            b(maps)
            torch.cuda.synchronize()
            b.check_inputs()
            bits = b.mask_bits.cpu().numpy().view(np.uint32)

            def one(i, gr=gr, gc=gc, br=br, bc=bc, pfa=pfa, bits=bits):
                r = oracle.cfar(host[i].astype(np.float64), gr, gc, br, bc, pfa, det_cap=1 << 15)
                return i, np.array_equal(_pack(r.mask), bits[i]), r.detections
            for i, ok, exp in pool.map(one, range(n)):
                assert ok, f"run {(gr, gc, br, bc, pfa)} map {i}: mask"
                _same_list(b.detections(i), exp, f"run {(gr, gc, br, bc, pfa)} map {i}")


def test_cfg2_batch_of_1024_records_vs_reference(uwb, ref, cuda):
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import DetectBatch
    n_rec = 1024
    recs = torch.empty((n_rec, 512, 1024), dtype=torch.float32, device=cuda)
    for i in range(n_rec):
        recs[i] = synth.cfg2_record(seed=2 + i, device=cuda)  # the bench's records
    config = uwb.PipelineConfig(mean_filter_window=5, fft_length=1024, band_low_hz=0.3, band_high_hz=0.8,
                                cfar=uwb.CfarParams(1, 4, 1e-3))
    db = DetectBatch(n_rec, 512, 1024, config, prf=20.0, dtype=torch.float32, det_capacity=4096)
    db(recs)
    torch.cuda.synchronize()
    db.check_inputs()
    host = recs.cpu().numpy()
    band = db.band.cpu().numpy()

    def one(i):
        e = ref.detect(host[i].astype(np.float64), prf=20.0, mean_filter_window=5, fft_length=1024,
                       guard_radius=1, background_radius=4, pfa=1e-3)
        return i, e
    with ThreadPoolExecutor(THREADS) as pool:
        for i, e in pool.map(one, range(n_rec)):
            assert_bitwise(band[i], e["band_power"], f"record {i} band map")
            assert np.array_equal(db.mask(i), e["result"].mask), f"record {i} mask"
            _same_list(db.detections(i), e["result"].detections, f"record {i}")


def test_cfg1_single_fp64_map_vs_reference(uwb, ref, cuda):
    from paper_2012_11077_b200 import synth
    m = synth.cfg1_map(seed=1, device=cuda)
    host = m.cpu().numpy()
    got = uwb.cfar2d_integral(host, uwb.CfarParams(2, 8, 1e-4))
    exp = ref.cfar2d(host, 2, 8, 1e-4, "integral")
    assert np.array_equal(got.mask, exp.mask)
    assert_bitwise(got.threshold_map, exp.threshold_map, "config 1 thresholds")
    _same_list(got.detections, exp.detections, "config 1")
