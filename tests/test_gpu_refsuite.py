"""GPU: the reference's OWN unit tests (proj/tests/test_{sat,cfar,pipeline}.cpp,
60 doctest cases, compiled unchanged by tests/refsuite/Makefile against the B200
drop-in headers and libuwbvital.so) must give exactly the verdicts they give
against the reference library itself. The reference fails two of its own cases
(a 64-trace frame whose band is empty, and a scene whose echo falls outside a
64-sample window); the drop-in must fail those two the same way and pass the
other 58."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "refsuite", "_build", "ref_unit_tests")
REF_BIN = os.path.join(HERE, "refsuite", "_build", "ref_unit_tests_reference")
EXPECTED_REFERENCE_FAILURES = {"zero frame yields zero detections", "stage errors carry the stage name"}


def _run(path):
    p = subprocess.run([path], capture_output=True, text=True, timeout=900)
    verdicts = dict((name, v) for v, name in re.findall(r"^\[(pass|FAIL)\] (.+)$", p.stdout, re.M))
    return p, verdicts


def test_reference_unit_tests_against_dropin(cuda):
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} not built (build() compiles it where /root/reference is mounted)")
    p, got = _run(BIN)
    assert len(got) == 60, p.stdout[-2000:]
    failed = {n for n, v in got.items() if v == "FAIL"}
    assert failed == EXPECTED_REFERENCE_FAILURES, (failed, p.stderr[-3000:])
    if os.path.exists(REF_BIN):
        _, ref = _run(REF_BIN)
        assert ref == got, "drop-in verdicts differ from the reference's own"
