"""BASELINE.json configs on the device path.

Reduced-size versions of each config run against the oracle trace for trace
parity (same iteration count / CG counts, fitness within 1e-8); the FULL sizes
are checked through size-independent properties: MTTKRP rows recomputed
exactly on tensor slices with numpy, the fast-residual floor of an exact-rank
model, a vanishing gradient at the truth, monotone ALS, and tree == naive.
"""
import numpy as np
import pytest

from tests.helpers import rel_err, swamp_factors

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ck():
    from paper_1910_12331_b200 import cpkit
    cpkit.load()
    return cpkit


def _trace_parity(orc, ck, x, init, cfg_dev, cfg_orc, optimizer):
    dims, R = list(x.shape), init[0].shape[1]
    p = ck.DeviceProblem(dims, R)
    p.upload(x)
    got, rep = p.optimize(dict(cfg_dev, optimizer=optimizer), init)
    j = rep.to_json()
    if optimizer == "gn":
        _, recs, st = orc.gn_optimize(x, init, cfg_orc)
    else:
        _, recs, st = orc.als_optimize(x, init, cfg_orc)
    return j, recs, st


# ---------------------------------------------------------------- reduced configs vs oracle
def test_c3_swamp_reduced_trace_parity(orc, ck):
    # config 3 family (collinear c=0.9), reduced to s=30, R=5 so the oracle runs in seconds
    dims, R = [30, 30, 30], 5
    truth = swamp_factors(orc, dims, R, 11)
    x = orc.reconstruct(truth)
    init = orc.random_model(dims, R, orc.init_seed(0, R, 0, 0))
    j, recs, st = _trace_parity(orc, ck, x, init, {"gn": {"max_iters": 40, "residual_tol": 1e-10}},
                                orc.GnConfig(max_iters=40, residual_tol=1e-10), "gn")
    # The swamp trajectory is chaotic once an inner CG solve stops at its cap
    # (min(sum s R, 10 R) = 50): a capped Krylov iterate on an ill-conditioned
    # system amplifies last-bit summation-order differences (DESIGN.md §5,
    # SURVEY.md Appendix A.2). Records before the first (near-)capped solve
    # must agree exactly in CG counts and to 1e-8 in residual; the run must reach the same terminal status.
    cap = min(sum(dims) * R, 10 * R)
    assert j["status"] == st
    compared = 0
    for a, b in zip(j["records"], recs):
        if max(a["cg_iters"], b["cg_iters"]) >= 0.9 * cap:  # (near-)capped solve: drift starts here
            break
        assert a["cg_iters"] == b["cg_iters"], (a, b)
        assert abs(a["residual"] - b["residual"]) < 1e-8, (a, b)
        compared += 1
    assert compared >= 5
    j, recs, st = _trace_parity(orc, ck, x, init, {"als": {"max_sweeps": 60, "residual_tol": 1e-10}},
                                orc.AlsConfig(max_sweeps=60, residual_tol=1e-10), "als")
    assert j["status"] == st and len(j["records"]) == len(recs)
    assert abs(j["records"][-1]["fitness"] - recs[-1]["fitness"]) < 1e-8


def test_c4_order4_reduced_trace_parity(orc, ck):
    # config 4 family (order 4, uniform[0,1), exact rank), reduced to s=16, R=6
    dims, R = [16, 16, 16, 16], 6
    truth = orc.random_model(dims, R, orc.problem_seed(0, R, 0))
    x = orc.reconstruct(truth)
    init = orc.random_model(dims, R, orc.init_seed(0, R, 0, 0))
    j, recs, st = _trace_parity(orc, ck, x, init, {"gn": {"max_iters": 25}}, orc.GnConfig(max_iters=25), "gn")
    assert j["status"] == st and len(j["records"]) == len(recs)
    assert [a["cg_iters"] for a in j["records"]] == [b["cg_iters"] for b in recs]
    assert abs(j["records"][-1]["fitness"] - recs[-1]["fitness"]) < 1e-8
    j, recs, st = _trace_parity(orc, ck, x, init, {"als": {"max_sweeps": 40}}, orc.AlsConfig(max_sweeps=40), "als")
    assert j["status"] == st and len(j["records"]) == len(recs)
    assert abs(j["records"][-1]["fitness"] - recs[-1]["fitness"]) < 1e-8


def test_c2_family_noise_reduced_trace_parity(orc, ck):
    # config 2 family (exact rank + 1e-6 relative noise), reduced to s=40, R=10
    dims, R = [40, 40, 40], 10
    truth = orc.random_model(dims, R, orc.problem_seed(0, R, 0))
    x = orc.reconstruct(truth)
    e = np.array([orc.gaussian(1, 0x4E01, i) for i in range(x.size)]).reshape(dims)
    x = x + 1e-6 * np.linalg.norm(x) / np.linalg.norm(e) * e
    init = orc.random_model(dims, R, orc.init_seed(0, R, 0, 0))
    j, recs, st = _trace_parity(orc, ck, x, init, {"gn": {"max_iters": 15}}, orc.GnConfig(max_iters=15), "gn")
    assert j["status"] == st and len(j["records"]) == len(recs)
    assert [a["cg_iters"] for a in j["records"]] == [b["cg_iters"] for b in recs]
    assert abs(j["records"][-1]["fitness"] - recs[-1]["fitness"]) < 1e-8


# ---------------------------------------------------------------- full sizes: properties
FULL = [
    ("C2", [400, 400, 400], 100),
    ("C4", [100, 100, 100, 100], 50),
]


@pytest.mark.parametrize("name,dims,R", FULL)
def test_full_size_properties(ck, name, dims, R):
    truth = ck.random_factors(dims, R, ck.problem_seed(0, R, 0))
    p = ck.DeviceProblem(dims, R)
    p.generate(truth)
    xn2 = p.norm2()
    # exact-rank model: fast residual floor (test_generators.cpp:135-151), zero gradient
    p.set_factors(truth)
    p.mttkrp(len(dims) - 1, download=False)
    r, f = p.residual(xn2)
    assert r < 1e-7
    for n in range(len(dims) - 1):
        p.mttkrp(n, download=False)
    g = p.gradient()
    assert sum(np.linalg.norm(a) for a in g) <= 1e-10 * np.sqrt(xn2) * len(dims)
    # MTTKRP rows recomputed exactly from tensor slices (mode 0: X[i] contracted with the rest)
    init = ck.random_factors(dims, R, ck.init_seed(0, R, 0, 0))
    p.set_factors(init)
    m0 = p.mttkrp(0)
    x = p.download()
    for i in (0, dims[0] // 2, dims[0] - 1):
        sl = x[i]
        ref = sl.reshape(-1, dims[-1]) @ init[-1]                 # contract last mode
        for m in range(len(dims) - 2, 0, -1):                    # then the rest, descending
            ref = (ref.reshape(-1, dims[m], R) * init[m][None, :, :]).sum(axis=1)
        ref = ref.reshape(R)
        assert rel_err(m0[i], ref) < 1e-11
    # tree == naive for every mode; contraction budget (<= 2 per sweep)
    p.reset_contraction_counter()
    for n in range(len(dims)):
        t = p.mttkrp(n)
        assert rel_err(t, p.mttkrp_naive(n)) < 1e-12
    # ALS sweeps decrease the fast residual (als.cpp monotonicity, lambda = 0)
    p.set_factors(init)
    prev = 1.0
    counts = []
    for _ in range(3):
        step, cnt = p.als_sweep(0.0)
        counts.append(cnt)
        p.mttkrp(len(dims) - 1, download=False)
        r, _ = p.residual(xn2)
        assert r <= prev + 1e-12
        prev = r
    # order 3: multi-sweep dimension tree (3 roots per 2 sweeps); else the reference tree (2 per sweep)
    assert counts == ([2, 1, 2] if len(dims) == 3 else [2, 2, 2])


@pytest.mark.parametrize("dims,R", [([14, 12, 11], 5), ([9, 8, 7, 6], 4)])
def test_gn_reference_residual_semantics(orc, ck, dims, R):
    """gn.residual_after = "naive": residual_after from a third, uncached
    contraction of the stepped factors, as gauss_newton.cpp:442-444 does (the
    default reuses the next iteration's tree pass). Same trace as the oracle
    (which follows the reference), and exactly one extra front-root contraction
    per stepped iteration."""
    truth = orc.random_model(dims, R, orc.problem_seed(3, R, 0))
    x = orc.reconstruct(truth) + 1e-3 * orc.random_model([int(np.prod(dims))], 1, 77, kind="gaussian")[0].reshape(dims)
    init = orc.random_model(dims, R, orc.init_seed(3, R, 0, 0))
    _, recs, st = orc.gn_optimize(x, init, orc.GnConfig(max_iters=8))
    counts = {}
    for mode in ("tree", "naive"):
        p = ck.DeviceProblem(dims, R)
        p.upload(x)
        p.profile(True)
        _, rep = p.optimize({"optimizer": "gn", "gn": {"max_iters": 8, "residual_after": mode}}, init)
        _, cnt = p.profile_read()
        j = rep.to_json()
        assert j["status"] == st and len(j["records"]) == len(recs) == 8
        for a, b in zip(j["records"], recs):
            assert a["cg_iters"] == b["cg_iters"] and a["lambda"] == b["lambda"], (mode, a, b)
            assert abs(a["residual"] - b["residual"]) <= 1e-9, (mode, a, b)  # fitness, as the trace tests
        assert j["config"]["gn"].get("residual_after", "tree") == mode
        counts[mode] = cnt
    # profile counters [back roots, front/single-mode roots, CG solves]: a tree
    # pass is one of each; the naive mode adds one front root per stepped iteration
    assert counts["tree"][1] == counts["tree"][0], counts
    assert counts["naive"][1] - counts["naive"][0] == len(recs), counts
