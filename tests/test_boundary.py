"""Drop-in boundary tests the reference holds for its C ABI.

* A plain C99 consumer compiled and linked against include/*.h
  (proj/tests/capi_header.c, proj/tests/CMakeLists.txt:17-23) - CPU only.
* cpkit_report_ok reports a failing self-test as 0 (cpkit_c.cpp:379-385).
* A CUDA failure inside a runner instance surfaces as CPKIT_ERR_INTERNAL and
  is never recorded as a numerical failure (errors.hpp taxonomy).
* Independent solves run concurrently from host threads with results bitwise
  equal to the same solves run one at a time (test_harness.cpp:82-102: the
  harness pool's results do not depend on the thread count).
"""
import os
import shutil
import subprocess
import threading

import numpy as np
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


def test_c99_consumer_compiles_links_and_runs(ck, tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = tmp_path / "capi_consumer"
    libdir = os.path.dirname(ck.LIB_PATH)
    cmd = ["gcc", "-std=c99", "-pedantic", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "c", "capi_consumer.c"), "-L", libdir, "-lcpkit_b200",
           f"-Wl,-rpath,{libdir}", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "capi_consumer ok" in out.stdout


@pytest.mark.gpu
def test_report_ok_follows_selftest_outcome(ck, monkeypatch):
    rep = ck.run_selftest_oracle({"instances": 2, "seed": 3})
    assert rep.to_json()["all_pass"] is True and rep.ok()
    monkeypatch.setenv("CPKIT_SELFTEST_TOL_SCALE", "0")  # fault injection: every tolerance 0
    bad = ck.run_selftest_oracle({"instances": 2, "seed": 3})
    assert bad.to_json()["all_pass"] is False
    assert not bad.ok()
    # non-selftest reports are OK whenever they exist
    assert ck.run_trace({"problem": {"family": "uniform01", "dims": [5, 4, 3], "ranks": [2]},
                         "optimizer": "als", "als": {"max_sweeps": 3}}).ok()


@pytest.mark.gpu
def test_device_fault_in_runner_is_internal_error(ck, monkeypatch):
    cfg = {"problem": {"family": "uniform01", "dims": [6, 5, 4], "ranks": [2]}, "optimizer": "gn",
           "problems": 1, "inits": 2, "seed": 1, "gn": {"max_iters": 5}}
    monkeypatch.setenv("CPKIT_NO_TINY", "1")  # the DeviceProblem-per-tensor path
    monkeypatch.setenv("CPKIT_INJECT_DEVICE_FAULT", "1")
    with pytest.raises(ck.CpkitError) as e:
        ck.run_likelihood(cfg)
    assert e.value.status == "internal_error"


@pytest.mark.gpu
def test_run_trace_matmul_family(ck, orc):
    """run_trace builds the matmul tensor like build_problem_tensor (harness.cpp:422-431)."""
    cfg = {"problem": {"family": "matmul", "matmul_n": 2, "ranks": [7]}, "optimizer": "als", "seed": 4,
           "als": {"max_sweeps": 6, "residual_tol": 0.0, "step_tol": 0.0}}
    rep = ck.run_trace(cfg).to_json()
    recs = rep["trace"]["records"] if "trace" in rep else rep["records"]
    assert len(recs) == 6
    x = ck.matmul_tensor(2).numpy()
    init = orc.random_model([4, 4, 4], 7, orc.init_seed(4, 7, 0, 0), kind="gaussian")
    _, ref, _ = orc.als_optimize(x, init, orc.AlsConfig(max_sweeps=6, residual_tol=0.0, step_tol=0.0))
    for a, b in zip(recs, ref):
        assert abs(a["residual"] - b["residual"]) < 1e-9


CONCURRENT = [  # (dims, rank, optimizer)
    ([20, 18, 16], 4, "als"),
    ([12, 10, 9, 8], 3, "gn"),
    ([30, 30, 30], 5, "gn"),
    ([25, 20, 15], 6, "als"),
    ([40, 35, 30], 8, "gn"),
    ([14, 13, 12, 11], 4, "als"),
]


def _solve(ck, case, seed):
    dims, rank, opt = case
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(dims)
    cfg = {"optimizer": opt, "rank": rank, "seed": seed, "init": {"distribution": "uniform", "a": 0, "b": 1},
           "als": {"max_sweeps": 15}, "gn": {"max_iters": 8}}
    model, rep = ck.decompose(ck.Tensor.create(x), cfg)
    return [f.copy() for f in model.factors()], [r["residual"] for r in rep.to_json()["records"]]


@pytest.mark.gpu
def test_concurrent_decompose_is_bitwise_stable(ck):
    serial = [_solve(ck, c, 100 + i) for i, c in enumerate(CONCURRENT)]
    results = [None] * len(CONCURRENT)
    errors = []

    def work(i):
        try:
            for _ in range(2):  # twice per thread: overlapping different phases
                results[i] = _solve(ck, CONCURRENT[i], 100 + i)
        except Exception as exc:  # surfaced below
            errors.append((i, exc))

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(CONCURRENT))]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    for i, (got, ref) in enumerate(zip(results, serial)):
        assert got is not None, i
        assert got[1] == ref[1], (i, CONCURRENT[i])
        for a, b in zip(got[0], ref[0]):
            assert np.array_equal(a, b), (i, CONCURRENT[i])
