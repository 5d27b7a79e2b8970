"""bench.py host logic (no GPU): the clock-based re-measure rule."""
import bench


def test_throttled_rule():
    ok = {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": []}
    assert not bench.throttled(ok)
    assert not bench.throttled(dict(ok, reasons=["sw_power_cap"]))  # kept and noted
    assert bench.throttled(dict(ok, reasons=["hw_slowdown"]))
    assert bench.throttled(dict(ok, reasons=["sw_thermal_slowdown"]))
    assert bench.throttled(dict(ok, sm_mhz=1200.0))  # stuck low with no reason
    assert not bench.throttled(dict(ok, sm_mhz=1200.0, reasons=["sw_power_cap"]))
    assert not bench.throttled(None) and not bench.throttled({"sm_mhz": None, "sm_max_mhz": None, "reasons": []})
