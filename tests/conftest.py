import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: large-size test")


def pytest_collection_modifyitems(config, items):
    """GPU tests get a (generous) per-test timeout: a hung device kernel must end the run with a
    failure rather than stall it.  The thread method is the one that works while the main thread
    is blocked inside a CUDA call (it dumps the stacks and exits the process)."""
    try:
        import pytest_timeout  # noqa: F401
    except ImportError:
        return
    import pytest
    for item in items:
        if item.get_closest_marker("gpu") and not item.get_closest_marker("timeout"):
            item.add_marker(pytest.mark.timeout(1200, method="thread"))
