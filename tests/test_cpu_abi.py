"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every
symbol include/*.h declares, and maps host-side errors to cpkit_status codes."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ck():
    import __graft_entry__ as g
    from paper_1910_12331_b200 import cpkit
    if not os.path.exists(cpkit.LIB_PATH):
        g.build()
    cpkit.load()
    return cpkit


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    return set(re.findall(r"CPKIT_API\s+[\w\s\*]+?\b(cpkit_\w+)\s*\(", text))


def test_headers_list_matches_binding(ck):
    assert declared("cpkit.h") == set(ck.CPKIT_SYMBOLS)
    assert declared("cpkit_dev.h") == set(ck.CPKIT_DEV_SYMBOLS)


def test_library_exports_every_declared_symbol(ck):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", ck.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (cpkit_\w+)", out))
    missing = (declared("cpkit.h") | declared("cpkit_dev.h")) - exported
    assert not missing, missing
    # hidden visibility: no C++ internals leak
    assert not [s for s in re.findall(r" T (\S+)", out) if not s.startswith("cpkit_")]


def test_status_names_and_version(ck):
    assert ck.version() == "1.0.0"
    assert [ck.status_name(i) for i in range(8)] == list(ck.STATUS_NAMES)


def test_host_side_errors(ck, tmp_path):
    import numpy as np
    # null / invalid arguments never touch the device
    with pytest.raises(ck.CpkitError) as e:
        ck.Tensor.load_file(str(tmp_path / "missing.cpkt"))
    assert e.value.status == "io_error"
    bad = tmp_path / "bad.cpkt"
    bad.write_bytes(b"XXXXX")
    with pytest.raises(ck.CpkitError) as e:
        ck.Tensor.load_file(str(bad))
    assert e.value.status == "parse_error"
    t = ck.Tensor.create(np.arange(24.0).reshape(2, 3, 4))
    t.save(str(tmp_path / "t.cpkt"))
    back = ck.Tensor.load_file(str(tmp_path / "t.cpkt"))
    assert np.array_equal(back.numpy(), t.numpy())
    with pytest.raises(ck.CpkitError) as e:
        ck.Tensor.create(np.array([[1.0, np.nan]]))
    assert e.value.status == "invalid_argument"
    with pytest.raises(ck.CpkitError) as e:
        ck.decompose(t, "{not json" and {"optimizer": "als", "rank": 1, "als": {"decay_factor": 0.5}})
    assert e.value.status == "invalid_argument"
    with pytest.raises(ck.CpkitError) as e:
        ck.run_trace({"problem": {"family": "bogus", "dims": [2, 2]}})
    assert e.value.status == "parse_error"
    m = ck.matmul_tensor(2)
    assert m.numpy().sum() == 8.0 and m.shape == (4, 4, 4)  # test_capi.cpp:86-94


def test_cpkt1_format_matches_oracle_layout(ck, tmp_path):
    # CPKT1 (tensor.cpp:197-239): magic, u64 order, u64 dims, f64 LE data
    import numpy as np
    x = np.arange(6.0).reshape(2, 3)
    ck.Tensor.create(x).save(str(tmp_path / "a.cpkt"))
    raw = (tmp_path / "a.cpkt").read_bytes()
    assert raw[:5] == b"CPKT1"
    assert np.frombuffer(raw[5:29], dtype="<u8").tolist() == [2, 2, 3]
    assert np.array_equal(np.frombuffer(raw[29:], dtype="<f8"), x.ravel())


def test_runner_config_errors_before_any_device_work(ck):
    """Runner configs are validated on the host (harness.cpp:203-220, :295-308,
    selftest.cpp:201-203, :281-283) with the reference's status codes; no GPU needed."""
    cases = [
        (ck.run_likelihood, {"problem": {"family": "bogus", "dims": [2, 2]}}, 2),          # parse
        (ck.run_likelihood, {"problem": {"family": "uniform01", "dims": [2, 2], "ranks": [0]}}, 1),
        (ck.run_likelihood, {"problem": {"family": "uniform01", "dims": [2, 2]}, "optimizer": "nope"}, 2),
        (ck.run_likelihood, {"problem": {"family": "uniform01"}}, 2),                      # dims required
        (ck.run_matmul, {"n": 0}, 1),
        (ck.run_matmul, {"rank": 0}, 1),
        (ck.run_matmul, {"als": {"decay_every": 0}}, 1),
        (ck.run_matmul, {"gn": {"lambda": -1.0}}, 1),
        (ck.run_bench_matvec, {"order": 1}, 1),
        (ck.run_bench_matvec, {"reps": 0}, 1),
        (ck.run_selftest_oracle, {"instances": 0}, 1),
    ]
    for fn, cfg, code in cases:
        with pytest.raises(ck.CpkitError) as e:
            fn(cfg)
        assert e.value.code == code, (fn.__name__, cfg, e.value)
