import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through the C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as o
    o.lib()
    return o


def pytest_sessionfinish(session, exitstatus):
    """CPKIT_GUARD=1 runs (the pool has no compute-sanitizer): fail the session
    when any released device buffer had its red zones overwritten."""
    if os.environ.get("CPKIT_GUARD", "0") in ("", "0"):
        return
    try:
        from paper_1910_12331_b200 import cpkit
        if cpkit._lib is None:
            return
        import gc
        gc.collect()
        v = cpkit.guard_violations()
    except Exception:  # noqa: BLE001 - no library, nothing to report
        return
    print(f"\ncpkit guard: {v} red-zone violation(s)")
    if v:
        session.exitstatus = 1
