"""Guarded allocation mode (CPKIT_GUARD=1): the stand-in for compute-sanitizer
memcheck, which this GPU pool does not allow. Every device buffer sits between
64 KB red zones checked when it is released (common.h, runtime.cu)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, gc
sys.path.insert(0, {root!r})
from paper_1910_12331_b200 import cpkit
assert cpkit.guard_selftest(), "guard mode missed an out-of-bounds write"
base = cpkit.guard_violations()
sys.argv = ["sanitize_driver"]
sys.path.insert(0, {tools!r})
import sanitize_driver
sanitize_driver.main()
gc.collect()
print("VIOLATIONS", cpkit.guard_violations() - base)
"""


def test_guard_mode_detects_and_workload_is_clean():
    env = dict(os.environ, CPKIT_GUARD="1")
    code = SCRIPT.format(root=ROOT, tools=os.path.join(ROOT, "tools"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "VIOLATIONS 0" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_guard_selftest_needs_env():
    from paper_1910_12331_b200 import cpkit
    if os.environ.get("CPKIT_GUARD", "0") not in ("", "0"):
        pytest.skip("session already runs in guard mode")
    with pytest.raises(cpkit.CpkitError):
        cpkit.guard_selftest()
