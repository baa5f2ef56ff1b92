import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")


def _build_all():
    """Compile the oracle (gcc), the input generator and libsesgd (nvcc, sm_100a) in-tree
    if they are missing or stale, so a fresh checkout can run the suite."""
    import oracle
    import synth
    from paper_2007_00433_b200 import _build
    oracle.build()
    synth.build()
    _build.build(checked=os.environ.get("SESGD_LIB") == "checked")


_build_all()
