import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels through the C-ABI)")
    config.addinivalue_line("markers", "slow: long-running (full-size configurations)")


def _ensure_built():
    from paper_2312_05181_b200 import build as pkg_build
    from oracle import oracle

    pkg_build.build()
    if not os.path.exists(oracle.lib_path(False)):
        oracle.build(reference=False)
    if os.path.isdir("/root/reference/proj") and not os.path.exists(oracle.lib_path(True)):
        oracle.build(reference=True)


_ensure_built()


@pytest.fixture(scope="session")
def rs():
    import paper_2312_05181_b200 as m

    m.load()
    return m


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle

    return Oracle(reference=False)


@pytest.fixture(scope="session")
def ref():
    """The reference's own compiled tensor-core (built here from /root/reference; the
    prebuilt .so travels to the GPU box)."""
    from oracle.oracle import Oracle, lib_path

    if not os.path.exists(lib_path(True)):
        pytest.skip("reference tensor-core not built (no /root/reference and no prebuilt oracle/_ref)")
    return Oracle(reference=True)


@pytest.fixture(scope="session")
def ctx(rs):
    if rs.device_count() < 1:
        pytest.fail("GPU test requires a CUDA device")
    return rs.Context(1, [0], [0])
