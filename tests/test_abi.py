"""CPU: the drop-in boundary. The C-ABI library loads and exports every symbol
include/uwbvital_b200.h declares; the C++ drop-in library exports the
uwbvital:: entry points of the reference headers; host-only helpers behave like
the reference; without a GPU every compute call fails loudly (no CPU fallback);
the product never touches the oracle."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "uwbvital_b200.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(uwb_[a-z0-9_]+)\s*\(", src)))


def test_header_functions_exported_and_bound():
    from paper_2012_11077_b200 import _native as N
    declared = _declared_functions()
    assert len(declared) >= 25
    lib = ctypes.CDLL(N.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), f"{name} declared but not exported"
    assert sorted(N.SIGNATURES) == declared, "ctypes table and header disagree"


def test_dropin_library_exports_reference_api():
    from paper_2012_11077_b200 import _native as N
    out = subprocess.run(["nm", "-DC", "--defined-only", N.DROPIN_PATH], capture_output=True, text=True,
                         check=True).stdout
    for sym in ["uwbvital::build_sat(", "uwbvital::cfar2d_integral(", "uwbvital::cfar2d_naive(",
                "uwbvital::alpha_factor(", "uwbvital::training_window(", "uwbvital::remove_dc(",
                "uwbvital::detrend_linear(", "uwbvital::mean_filter_slow(", "uwbvital::subtract_slow_time_mean(",
                "uwbvital::normalize_slow(", "uwbvital::slow_time_spectrum(", "uwbvital::band_select(",
                "uwbvital::detect(", "uwbvital::SummedAreaTable::region_sum(", "uwbvital::CfarParams::validate(",
                "uwbvital::RadarFrame::validate(", "uwbvital::PipelineConfig::effective_fft_length("]:
        assert sym in out, f"{sym} missing from the drop-in"


def test_dropin_headers_compile_against_reference_call_sites(tmp_path):
    """A caller written against the reference headers compiles and links unchanged."""
    src = tmp_path / "caller.cpp"
    src.write_text("""
#include "uwbvital/cfar.hpp"
#include "uwbvital/pipeline.hpp"
#include "uwbvital/sat.hpp"
#include "uwbvital/errors.hpp"
using namespace uwbvital;
int main() {
    Matrix m(8, 8, 1.0);
    CfarParams p; p.guard_radius = 1; p.background_radius = 2; p.pfa = 1e-3;
    try { DetectionResult r = cfar2d_integral(m, p, 4); return (int)r.detections.size(); }
    catch (const Error& e) { return 3; }
    SummedAreaTable s = build_sat(m); (void)s.region_sum_unchecked(0, 1, 0, 1);
    RadarFrame f; PipelineConfig c; DetectOutput o = detect(f, c); (void)o;
}
""")
    from paper_2012_11077_b200 import _native as N
    lib = os.path.dirname(N.DROPIN_PATH)
    exe = tmp_path / "caller"
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), str(src), "-L", lib, "-luwbvital",
                    "-Wl,-rpath," + lib, "-o", str(exe)], check=True)
    assert exe.exists()


def test_host_helpers_match_reference(ref):
    import paper_2012_11077_b200 as uwb
    for n in (1, 5, 24, 112, 416, 544, 5248):
        for pfa in (1e-5, 1e-4, 1e-3, 0.5):
            assert uwb.alpha_factor(n, pfa) == ref.alpha_factor(n, pfa)
    for args in [(1, 1, 1e-3, 50, 50, 100, 100), (1, 1, 1e-3, 0, 0, 100, 100), (4, 8, 1e-3, 100, 100, 1024, 600),
                 (2, 8, 1e-4, 5, 1020, 1024, 1024)]:
        g, b, pfa, r, c, R, Cc = args
        w = uwb.training_window(uwb.CfarParams(g, b, pfa), r, c, R, Cc)
        e = ref.training_window(g, b, pfa, r, c, R, Cc)
        assert (w.outer.r0, w.outer.r1, w.outer.c0, w.outer.c1) == e["outer"]
        assert (w.guard.r0, w.guard.r1, w.guard.c0, w.guard.c1) == e["guard"]
        assert w.n_train == e["n_train"]
    from oracle.pyoracle import OracleError
    for bad in [(0, 0.5), (10, 0.0), (10, 1.0), (10, -0.1)]:
        with pytest.raises(uwb.ParameterError) as g:
            uwb.alpha_factor(*bad)
        with pytest.raises(OracleError) as r:
            ref.alpha_factor(*bad)
        assert str(g.value) == r.value.message
    for bad in [(10, 0, 8, 8), (8, 8, 4, 8), (5, 5, 2, 2)]:
        rows, cols, g_, b_ = bad
        for row, col in [(rows + 2, 0), (2, 2)]:
            try:
                ref.training_window(g_, b_, 1e-3, row, col, rows, cols)
                continue
            except OracleError as e:
                with pytest.raises(uwb.Error) as ge:
                    uwb.training_window(uwb.CfarParams(g_, b_, 1e-3), row, col, rows, cols)
                assert str(ge.value) == e.message and type(ge.value).__name__ == e.kind


def test_params_validation_messages(ref):
    import paper_2012_11077_b200 as uwb
    from oracle.pyoracle import OracleError
    for g, b, pfa in [(-1, 8, 1e-3), (1, 0, 1e-3), (1, 2, 1.5), (1, 2, 0.0)]:
        with pytest.raises(uwb.ParameterError) as ge:
            uwb.CfarParams(g, b, pfa).validate()
        with pytest.raises(OracleError) as re_:
            ref.cfar2d(np.ones((16, 16)), g, b, pfa, "naive")
        assert str(ge.value) == re_.value.message
    assert uwb.CfarParams(2, 8).interior_train_count() == 416
    assert uwb.CfarParams(1, 4, guard_cols=3, background_cols=16).interior_train_count() == 408
    a = uwb.CfarParams(2, 8, 1e-4).alpha_table()
    assert a[0] == 0 and a[416] == ref.alpha_factor(416, 1e-4) == 9.3130566043946388


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    import paper_2012_11077_b200 as uwb
    with pytest.raises(uwb.CudaError):
        uwb.build_sat(np.ones((4, 4)))
    with pytest.raises(uwb.CudaError):
        uwb.cfar2d_integral(np.ones((16, 16)), uwb.CfarParams(1, 2))
    with pytest.raises(uwb.CudaError):
        uwb.remove_dc(uwb.RadarFrame(np.ones((4, 4))))
    with pytest.raises(uwb.CudaError):
        uwb.detect(uwb.RadarFrame(np.ones((64, 64))), uwb.PipelineConfig())


def test_product_does_not_use_oracle():
    pkg = os.path.join(ROOT, "paper_2012_11077_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text and "pyoracle" not in text, f
                assert "libuwbref" not in text and "uwb_oracle" not in text, f
