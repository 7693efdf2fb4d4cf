"""Full BASELINE sizes (configs 3 and 4) through size-independent properties,
plus sampled bit-identity against the reference, and layout / window edge
cases that route to the fallback kernels.

Properties used at full size (the CPU oracle cannot run 4.3e9 cells in a test):
* the detection count of every map equals the popcount of its bit mask;
* every detection list is sorted (value desc, row asc, col asc; cfar.cpp:170-173);
* scale covariance: multiplying a map by 2^k multiplies every table entry,
  every window sum and every threshold by 2^k exactly, so masks are unchanged
  (test_cfar.cpp:241-276 states this for the reference);
* a seeded sample of maps is bit-identical to the reference (oracle/_ref).
"""
import numpy as np
import pytest
import torch

from tests.helpers import assert_bitwise

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _popcounts(bits: torch.Tensor) -> np.ndarray:
    """Set bits per map, on the device (256 maps at a time)."""
    lut = torch.tensor([bin(i).count("1") for i in range(256)], device=bits.device, dtype=torch.int64)
    out = [lut[c.contiguous().view(torch.uint8).long()].view(c.shape[0], -1).sum(1) for c in bits.split(256)]
    return torch.cat(out).cpu().numpy()


def _sorted_ok(d) -> bool:
    if len(d) < 2:
        return True
    key = np.lexsort((d["col"], d["row"], -d["value"]))
    return np.array_equal(key, np.arange(len(d)))


def test_cfg3_full_batch_properties_and_sample(uwb, ref, cuda):
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    n = 4096
    maps = torch.empty((n, 1024, 1024), dtype=torch.float32, device=cuda)
    for c in range(n // 64):
        synth.cfg3_maps(64, seed=3 * 1_000_003 + c, device=cuda, out=maps[c * 64:(c + 1) * 64])
    p = uwb.CfarParams(2, 8, 1e-4)
    b = BatchCfar(n, 1024, 1024, p, torch.float32, det_capacity=512, device=cuda)
    b(maps)
    torch.cuda.synchronize()
    b.check_inputs()
    counts = b.detection_counts()
    assert (counts <= 512).all() and counts.sum() > n * 32  # every map has its 32 targets plus false alarms
    assert np.array_equal(_popcounts(b.mask_bits), counts)
    for i in range(0, n, 509):
        assert _sorted_ok(b.detections(i)), f"map {i} list order"
    # scale covariance over the whole batch
    bits0 = b.mask_bits.clone()
    maps.mul_(8.0)
    b(maps)
    torch.cuda.synchronize()
    assert torch.equal(bits0, b.mask_bits)
    maps.mul_(0.125)
    # seeded sample, bit-identical to the reference
    for i in (0, 1777, 4095):
        host = maps[i].double().cpu().numpy()
        r = ref.cfar2d(host, 2, 8, 1e-4, "integral")
        bm = np.unpackbits(bits0[i].view(torch.uint8).cpu().numpy().reshape(1024, -1), axis=1,
                           bitorder="little")[:, :1024]
        assert np.array_equal(bm, r.mask), f"map {i} mask"


def test_cfg4_full_map_properties_and_rows(uwb, oracle, cuda):
    """One 16384 x 16384 map (g4 b32 Pfa 1e-5): mask/list consistency, scale
    covariance, and a band of rows bit-identical to the restatement (row range
    of the global table)."""
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    R = C = 16384
    m = synth.cfg4_map(seed=4, device=cuda, rows=R, cols=C).unsqueeze(0).contiguous()
    p = uwb.CfarParams(4, 32, 1e-5)
    b = BatchCfar(1, R, C, p, torch.float32, det_capacity=1 << 16, device=cuda)
    b(m)
    torch.cuda.synchronize()
    b.check_inputs()
    cnt = int(b.detection_counts()[0])
    assert cnt > 1000
    assert _popcounts(b.mask_bits)[0] == cnt
    assert _sorted_ok(b.detections(0))
    bits0 = b.mask_bits.clone()
    m.mul_(4.0)
    b(m)
    torch.cuda.synchronize()
    assert torch.equal(bits0, b.mask_bits)
    m.mul_(0.25)
    host = m[0].double().cpu().numpy()
    r0, r1 = 8000, 8064
    exp = oracle.cfar(host, 4, 4, 32, 32, 1e-5, row_begin=r0, row_end=r1)
    got = np.unpackbits(bits0[0, r0:r1].view(torch.uint8).cpu().numpy().reshape(r1 - r0, -1), axis=1,
                        bitorder="little")[:, :C]
    assert np.array_equal(got, exp.mask[r0:r1])


@pytest.mark.parametrize("g,b", [(2, 70), (30, 2)])
def test_windows_beyond_the_ring_box(uwb, ref, cuda, g, b):
    """hc > 62 runs the fallback CFAR kernel; a tall window (hr = 32) lowers the
    ring kernel's occupancy profile. Both bit-identical to the reference."""
    from paper_2012_11077_b200.batch import BatchCfar
    gen = torch.Generator(device="cuda").manual_seed(31)
    maps = torch.empty((2, 300, 420), device="cuda", dtype=torch.float32).exponential_(1.0, generator=gen)
    p = uwb.CfarParams(g, b, 1e-2)
    bt = BatchCfar(2, 300, 420, p, torch.float32, det_capacity=1 << 15, want_mask_u8=True, want_thresholds=True)
    bt(maps)
    torch.cuda.synchronize()
    host = maps.double().cpu().numpy()
    for i in range(2):
        r = ref.cfar2d(host[i], g, b, 1e-2, "integral")
        assert np.array_equal(bt.mask_u8[i].cpu().numpy(), r.mask)
        assert_bitwise(bt.thresholds[i].cpu().numpy(), r.threshold_map, f"map {i} thresholds")


def test_padded_and_unaligned_layouts(uwb, ref, cuda):
    """Row pitch larger than the width and odd widths (element staging in the SAT,
    fallback CFAR when rows are not 16-byte aligned) through uwb_dev_cfar2d."""
    import ctypes as C
    from paper_2012_11077_b200 import _native as N
    from paper_2012_11077_b200.errors import raise_for
    gen = torch.Generator(device="cuda").manual_seed(5)
    for rows, cols, ld in ((37, 129, 131), (64, 200, 256), (5, 3, 7)):
        buf = torch.empty((2, rows, ld), device="cuda", dtype=torch.float32).exponential_(1.0, generator=gen)
        p = uwb.CfarParams(1, 2, 0.05)
        cp = p.to_c()
        batch = N.uwb_map_batch(buf.data_ptr(), N.UWB_F32, 0, 2, rows, cols, ld, rows * ld)
        ws = N.lib.uwb_dev_cfar2d_workspace(C.byref(batch), C.byref(cp), N.UWB_SAT_GLOBAL, 0, 4096)
        work = torch.empty(int(ws), dtype=torch.uint8, device="cuda")
        alpha = torch.from_numpy(p.alpha_table()).to("cuda")
        words = (cols + 31) // 32
        bits = torch.zeros((2, rows, words), dtype=torch.int32, device="cuda")
        mask = torch.zeros((2, rows, cols), dtype=torch.uint8, device="cuda")
        thr = torch.zeros((2, rows, cols), dtype=torch.float64, device="cuda")
        dets = torch.zeros((2, 4096, 32), dtype=torch.uint8, device="cuda")
        cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
        fb = torch.zeros((2, 2), dtype=torch.int64, device="cuda")
        out = N.uwb_cfar_outputs(bits.data_ptr(), words, rows * words, mask.data_ptr(), thr.data_ptr(),
                                 dets.data_ptr(), 4096, cnt.data_ptr(), fb.data_ptr())
        raise_for(N.lib.uwb_dev_cfar2d(C.byref(batch), C.byref(cp), alpha.data_ptr(), N.UWB_SAT_GLOBAL, 0,
                                       C.byref(out), work.data_ptr(), C.c_uint64(work.numel()), 0,
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        torch.cuda.synchronize()
        host = buf[:, :, :cols].double().cpu().numpy()
        for i in range(2):
            r = ref.cfar2d(host[i], 1, 2, 0.05, "integral")
            assert np.array_equal(mask[i].cpu().numpy(), r.mask), f"{rows}x{cols} ld {ld} map {i}"
            assert_bitwise(thr[i].cpu().numpy(), r.threshold_map, f"{rows}x{cols} ld {ld} map {i}")
