"""GPU parity of the cluster SAT (csrc/sat_cluster.cu: one thread-block cluster
per table, strips handed over through distributed shared memory) against the
reference build_sat (sat.cpp:10-37, compiled into oracle/_ref): whole tables,
bit for bit, through the C ABI (uwb_dev_build_sat / uwb_dev_cfar2d). Shapes
cover one strip to the 24-strip limit, rows around the 8-row block and 32-lane
skew boundaries, both source types, batches of clusters and non-finite inputs;
the one-CTA-per-table kernel (flags bit 10) must give the same results."""
import ctypes as C

import numpy as np
import pytest
import torch

from tests.helpers import assert_bitwise

pytestmark = pytest.mark.gpu


def dev_tables(maps: torch.Tensor):
    """uwb_dev_build_sat over a (n, rows, cols) CUDA tensor -> (tables (n, rows+1, cols+1), first_nonfinite)."""
    from paper_2012_11077_b200 import _native as N
    from paper_2012_11077_b200.errors import raise_for
    n, rows, cols = maps.shape
    dt = N.UWB_F32 if maps.dtype == torch.float32 else N.UWB_F64
    b = N.uwb_map_batch(maps.data_ptr(), dt, 0, n, rows, cols, cols, rows * cols)
    ld = (cols + 32 + 31) // 32 * 32
    stride = (rows + 1) * ld
    tab = torch.full((n, rows + 1, ld), float("nan"), dtype=torch.float64, device=maps.device)
    bad = torch.zeros(n, dtype=torch.int64, device=maps.device)
    ws = torch.empty(int(N.lib.uwb_dev_build_sat_workspace(C.byref(b))), dtype=torch.uint8, device=maps.device)
    raise_for(N.lib.uwb_dev_build_sat(C.byref(b), tab.data_ptr(), C.c_uint64(ld), C.c_uint64(stride),
                                      bad.data_ptr(), ws.data_ptr(), C.c_uint64(ws.numel()),
                                      C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    return tab[:, :, 31:31 + cols + 1].cpu().numpy(), bad.cpu().numpy().astype(np.uint64)


@pytest.mark.parametrize("rows,cols", [(1, 2), (7, 64), (8, 66), (9, 128), (31, 130), (32, 512), (33, 600),
                                       (40, 1024), (100, 1536), (256, 512), (1024, 600), (263, 62), (2049, 190),
                                       (1024, 7), (33, 67), (100, 65), (5, 1), (300, 129)])
def test_cluster_sat_f64_bit_identical(ref, cuda, rows, cols):
    m = np.random.default_rng(rows * 7919 + cols).uniform(-1, 1, (rows, cols))
    got, bad = dev_tables(torch.from_numpy(m).to(cuda).unsqueeze(0).contiguous())
    assert_bitwise(got[0], ref.build_sat(m), f"cluster SAT f64 {rows}x{cols}")
    assert bad[0] == np.uint64(0xFFFFFFFFFFFFFFFF)


@pytest.mark.parametrize("rows,cols", [(1, 4), (5, 128), (8, 132), (39, 1024), (64, 3072), (512, 28), (1000, 1100),
                                       (1024, 1024), (50, 131), (7, 3), (200, 257), (64, 1001)])
def test_cluster_sat_f32_bit_identical(ref, cuda, rows, cols):
    m = np.random.default_rng(rows * 31 + cols).exponential(1.0, (rows, cols)).astype(np.float32)
    got, _ = dev_tables(torch.from_numpy(m).to(cuda).unsqueeze(0).contiguous())
    assert_bitwise(got[0], ref.build_sat(m.astype(np.float64)), f"cluster SAT f32 {rows}x{cols}")


@pytest.mark.parametrize("rows,cols,dt", [(300, 4000, np.float32), (33, 3200, np.float32), (1000, 8192, np.float32),
                                          (200, 2048, np.float64), (70, 1600, np.float64), (150, 4099, np.float32),
                                          (90, 2051, np.float64)])
def test_cluster_chain_bit_identical(ref, cuda, rows, cols, dt):
    """Tables wider than one cluster's 24 strips: a chain of 8-CTA clusters, the
    boundary columns handed over through global memory (relay warp)."""
    m = np.random.default_rng(rows + 13 * cols).exponential(1.0, (rows, cols)).astype(dt)
    got, bad = dev_tables(torch.from_numpy(m).to(cuda).unsqueeze(0).contiguous())
    assert_bitwise(got[0], ref.build_sat(m.astype(np.float64)), f"cluster chain {rows}x{cols}")
    assert bad[0] == np.uint64(0xFFFFFFFFFFFFFFFF)


def test_cluster_chain_two_maps(ref, cuda):
    """Two chained tables in one launch (2 x 4 clusters x 8 CTAs)."""
    m = np.random.default_rng(17).exponential(1.0, (2, 150, 4096)).astype(np.float32)
    got, _ = dev_tables(torch.from_numpy(m).to(cuda))
    for i in range(2):
        assert_bitwise(got[i], ref.build_sat(m[i].astype(np.float64)), f"cluster chain map {i}")


def test_cluster_sat_batch_of_clusters(ref, cuda):
    """18 tables x 8-CTA clusters = 144 CTAs resident at once; every table checked."""
    m = np.random.default_rng(5).exponential(1.0, (18, 300, 500))
    got, _ = dev_tables(torch.from_numpy(m).to(cuda))
    for i in range(18):
        assert_bitwise(got[i], ref.build_sat(m[i]), f"cluster SAT batch map {i}")


def test_cluster_sat_nonfinite_inputs(ref, cuda):
    """NaN / Inf inputs (incl. the all-ones and signalling NaN bit patterns) are
    reported as the first offending cell in row-major order and cannot stall
    the strip chain."""
    m = np.random.default_rng(6).uniform(0, 1, (4, 200, 256))
    m[0, 150, 63] = np.nan                                                       # last column of strip 0
    m[1, 10, 200] = np.inf
    m[1, 9, 255] = -np.inf
    m[2].view(np.uint64)[77, 127] = np.uint64(0xFFFFFFFFFFFFFFFF)                # all-ones NaN on a strip edge
    m[3].view(np.uint64)[3, 63] = np.uint64(0x7FF0000000000001)                  # signalling NaN on a strip edge
    got, bad = dev_tables(torch.from_numpy(m).to(cuda))
    assert bad.tolist() == [150 * 256 + 63, 9 * 256 + 255, 77 * 256 + 127, 3 * 256 + 63]
    # cells that do not depend on the bad cell are still the reference's
    clean = m[0].copy()
    clean[150, 63] = 0.0
    exp = ref.build_sat(clean)
    assert_bitwise(got[0][:151, :], exp[:151, :], "rows above the NaN")
    assert_bitwise(got[0][:, :64], exp[:, :64], "columns left of the NaN")


@pytest.mark.parametrize("dtype,shape,gb", [(torch.float64, (256, 512), (2, 8)), (torch.float64, (1024, 600), (4, 8)),
                                            (torch.float32, (700, 1400), (1, 3)), (torch.float32, (64, 28), (1, 2))])
def test_cluster_and_cta_tables_give_the_same_cfar(uwb, ref, cuda, dtype, shape, gb):
    """The whole single-map call (cluster SAT -> ring CFAR -> sort) against the
    reference, and against the one-CTA-per-table schedule (flags bit 10)."""
    from paper_2012_11077_b200.batch import BatchCfar
    g = torch.Generator(device="cuda").manual_seed(shape[0] + shape[1])
    maps = torch.empty((1,) + shape, device=cuda, dtype=dtype).exponential_(1.0, generator=g)
    p = uwb.CfarParams(gb[0], gb[1], 1e-3)
    outs = []
    for cta in (False, True):
        b = BatchCfar(1, shape[0], shape[1], p, dtype, det_capacity=1 << 14, want_thresholds=True)
        b(maps, cta_tables=cta)
        torch.cuda.synchronize()
        outs.append((b.thresholds[0].cpu().numpy(), b.mask(0), b.detections(0).tobytes()))
    exp = ref.cfar2d(maps[0].double().cpu().numpy(), gb[0], gb[1], 1e-3, "integral")
    assert_bitwise(outs[0][0], exp.threshold_map, "cluster tables: thresholds vs reference")
    assert np.array_equal(outs[0][1], exp.mask)
    assert_bitwise(outs[1][0], outs[0][0], "CTA tables vs cluster tables")
    assert np.array_equal(outs[1][1], outs[0][1]) and outs[1][2] == outs[0][2]


@pytest.mark.parametrize("rows,cols,certified", [(200, 2560, False), (300, 6016, True), (96, 4096, True)])
def test_cluster_chain_through_cfar(uwb, ref, cuda, rows, cols, certified):
    """Wide single maps end to end (BatchCfar -> uwb_dev_cfar2d): the exact path (a map
    whose strips fit one cluster only three per CTA runs as a chain of one-strip
    clusters) and the certified path (sparse-mode call answered by the dense chain),
    masks and detection lists against the reference."""
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    m = synth.exponential_maps(1, rows, cols, seed=rows + cols, dtype=torch.float32, device=cuda)
    m[0, rows // 2, cols // 3] += 400.0
    m[0, 5, cols - 7] += 300.0
    p = uwb.CfarParams(2, 8, 1e-4)
    b = BatchCfar(1, rows, cols, p, torch.float32, det_capacity=1 << 13)
    b(m)
    torch.cuda.synchronize()
    b.check_inputs()
    status = b.cert_status.cpu().numpy()  # -1: the exact path decided the map
    exp = ref.cfar2d(m[0].double().cpu().numpy(), 2, 8, 1e-4, "integral")
    assert np.array_equal(b.mask(0), exp.mask), "mask"
    d, r = b.detections(0), exp.detections
    assert len(d) == len(r) and len(d) >= 2
    assert np.array_equal(d["row"], r["row"]) and np.array_equal(d["col"], r["col"])
    assert_bitwise(d["value"], r["value"], "values")
    assert_bitwise(d["threshold"], r["threshold"], "thresholds")
    assert (int(status[0]) != -1) == certified, "path taken"


def test_cluster_sat_odd_width_nonfinite(ref, cuda):
    """Odd widths (helper-warp copies instead of TMA): a NaN in the straddling lane's only
    column and in an interior column are reported as the first row-major offender."""
    m = np.random.default_rng(3).exponential(1.0, (90, 7))
    m[40, 6] = np.nan
    m[70, 2] = np.inf
    _, bad = dev_tables(torch.from_numpy(m).to(cuda).unsqueeze(0).contiguous())
    assert bad[0] == np.uint64(40 * 7 + 6)
