import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running parity case")
    # Build the engine and the oracle before collection: test modules import the
    # package, whose import fails loudly without the sm_100a library (nvcc
    # cross-compiles without a GPU, so a fresh clone collects cleanly).
    import __graft_entry__

    __graft_entry__.build()


def _engine_params():
    return ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)]


@pytest.fixture(params=_engine_params())
def engine(request):
    """The same reference-shaped API backed by the CPU oracle or the B200 engine."""
    import engines

    return engines.make(request.param)
