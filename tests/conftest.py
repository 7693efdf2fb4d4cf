import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running full-size parity case")


def _ensure_oracle():
    from oracle import pyoracle
    if not os.path.exists(pyoracle.ORACLE_SO) or (
            not os.path.exists(pyoracle.REF_SO) and os.path.isdir("/root/reference/proj/src")):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True,
                       stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def ref():
    """The reference C++ implementation (oracle/_ref/libuwbref.so)."""
    _ensure_oracle()
    from oracle.pyoracle import RefLib
    return RefLib()


@pytest.fixture(scope="session")
def oracle():
    """The plain-C restatement (oracle/_build/libuwboracle.so)."""
    _ensure_oracle()
    from oracle.pyoracle import OracleLib
    return OracleLib()


@pytest.fixture(scope="session")
def uwb():
    """The product package; GPU tests require a device and the built library."""
    import paper_2012_11077_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    return torch.device("cuda", 0)
