"""GPU parity: every device kernel/driver of the hot path against the CPU oracle
on identical seeded inputs, called through the C ABI (libcpkit_b200.so).

Tolerances (north_star): per-kernel outputs within 1e-11 Frobenius-relative
(test_tensor_core.cpp:30-32 metric); same GN/ALS iteration counts; final
fitness within 1e-8.
"""
import os

import numpy as np
import pytest

from tests.helpers import gauss_factors, gauss_tensor, mttkrp_unfold, rel_err, vec_rel_err

pytestmark = pytest.mark.gpu

KTOL = 1e-11  # per-kernel Frobenius-relative tolerance


@pytest.fixture(scope="module")
def ck():
    from paper_1910_12331_b200 import cpkit
    cpkit.load()
    return cpkit


def make(ck, x, factors):
    p = ck.DeviceProblem(list(x.shape), factors[0].shape[1])
    p.upload(x)
    p.set_factors(factors)
    return p


# ---------------------------------------------------------------- MTTKRP
TREE_CASES = [
    ([5, 3], 3), ([3, 4, 2], 3), ([2, 3, 4, 5], 3), ([3, 2, 2, 3, 2], 2),  # odd dims, orders 2-5
    ([3, 3, 3], 4), ([3, 3, 3, 3], 4), ([3, 3, 3, 3, 3], 4),                # test_tensor_core.cpp:210-231
    ([50, 50, 50], 5),                                                      # C1 shape
    ([40, 31, 37], 20), ([17, 19, 23, 11], 7), ([33, 65, 129], 13),
    ([40, 30, 50], 100),                                                    # R=100 (NT=13 tiles)
    ([20, 24, 26], 200),                                                    # R=200 (two rank tiles)
    ([1, 1, 1], 1), ([1, 7, 1], 3),                                         # degenerate extents
]


@pytest.mark.parametrize("dims,rank", TREE_CASES)
def test_mttkrp_tree_matches_oracle(orc, ck, dims, rank):
    x = np.random.default_rng(sum(dims) + rank).standard_normal(dims)
    f = gauss_factors(orc, dims, rank, 11 + rank)
    ref, ref_cnt = orc.mttkrp_tree_all(x, f)
    p = make(ck, x, f)
    for n in range(len(dims)):
        got = p.mttkrp(n)
        assert rel_err(got, ref[n]) < KTOL, (n, rel_err(got, ref[n]))
    assert p.full_contractions == ref_cnt <= 2


# Back roots with more tiles than one wave and a partial last wave: the last
# wave's rows run as a separate split-K launch (fixed-order reduce). Results
# match the oracle, repeat bitwise, and agree with the single launch.
@pytest.mark.parametrize("dims,rank", [([160, 130, 30], 24), ([150, 200, 40], 100), ([40, 500, 36], 50)])
def test_root_tail_launch(orc, ck, dims, rank, monkeypatch):
    x = np.random.default_rng(rank).standard_normal(dims)
    f = gauss_factors(orc, dims, rank, 21)
    ref, _ = orc.mttkrp_tree_all(x, f)
    p = make(ck, x, f)
    a = p.mttkrp_naive(0)
    assert rel_err(a, ref[0]) < KTOL
    assert np.array_equal(a, p.mttkrp_naive(0))
    monkeypatch.setenv("CPKIT_NO_TAIL_LAUNCH", "1")
    assert rel_err(p.mttkrp_naive(0), a) < 1e-13


# Orders >= 4 run the front root on a transposed tensor copy (NN GEMM) when
# memory allows; the TN kernel on X itself stays covered with the copy off.
@pytest.mark.parametrize("copy", ["0", "1"])
@pytest.mark.parametrize("dims,rank", [([6, 5, 7, 9], 6), ([17, 19, 23, 11], 7), ([3, 2, 2, 3, 2], 2)])
def test_front_root_copy_and_tn(orc, ck, dims, rank, copy, monkeypatch):
    monkeypatch.setenv("CPKIT_FRONT_COPY", copy)
    x = np.random.default_rng(sum(dims)).standard_normal(dims)
    f = gauss_factors(orc, dims, rank, 31)
    ref, ref_cnt = orc.mttkrp_tree_all(x, f)
    p = make(ck, x, f)
    for n in range(len(dims)):
        assert rel_err(p.mttkrp(n), ref[n]) < KTOL, n
    assert p.full_contractions == ref_cnt


@pytest.mark.parametrize("dims,rank", [([3, 4, 2], 3), ([6, 5, 4, 3], 5), ([30, 20, 10], 9)])
def test_mttkrp_naive_and_unfolding(orc, ck, dims, rank):
    x = gauss_tensor(orc, dims, 5) if np.prod(dims) < 5000 else \
        np.random.default_rng(3).standard_normal(dims)
    f = gauss_factors(orc, dims, rank, 6)
    p = make(ck, x, f)
    for n in range(len(dims)):
        got = p.mttkrp_naive(n)
        assert rel_err(got, orc.mttkrp_naive(x, f, n)) < KTOL
        assert rel_err(got, mttkrp_unfold(x, f, n)) < KTOL
    assert p.full_contractions == 0  # uncached overload does not count


def test_mttkrp_kats(ck):
    # test_tensor_core.cpp:178-199
    p = make(ck, np.ones((2, 2, 2)), [np.ones((2, 2))] * 3)
    assert np.array_equal(p.mttkrp(0), 4 * np.ones((2, 2)))
    a = np.array([1.0, -2.0, 0.5]); b = np.array([2.0, 1.0, 1.0]); c = np.array([0.5, 3.0, -1.0])
    x = np.einsum("i,j,k->ijk", a, b, c)
    p = make(ck, x, [a[:, None], b[:, None], c[:, None]])
    assert rel_err(p.mttkrp(0), a[:, None] * (b @ b) * (c @ c)) < 1e-12


def test_workspace_invalidation(orc, ck):
    # test_tensor_core.cpp:233-244
    x = gauss_tensor(orc, [3, 4, 2], 29)
    f = gauss_factors(orc, [3, 4, 2], 2, 30)
    p = make(ck, x, f)
    p.mttkrp(0)
    f2 = [f[0], f[1], gauss_factors(orc, [2], 2, 31)[0]]
    p.set_factors(f2)
    p.note_factor_update(2)
    assert rel_err(p.mttkrp(0), orc.mttkrp_naive(x, f2, 0)) < KTOL


def test_mttkrp_mode_out_of_range(ck):
    p = make(ck, np.ones((2, 2, 2)), [np.ones((2, 2))] * 3)
    with pytest.raises(ck.CpkitError) as e:
        p.mttkrp(3)
    assert e.value.status == "invalid_argument"


# ---------------------------------------------------------------- Gamma / residual / gradient
@pytest.mark.parametrize("dims,rank", [([3, 2, 4, 2], 3), ([50, 50, 50], 5), ([40, 30, 20], 60)])
def test_gamma_set(orc, ck, dims, rank):
    f = gauss_factors(orc, dims, rank, 19)
    x = np.zeros(dims)
    p = make(ck, x, f)
    g, pr = p.gamma_set()
    rg, rp = orc.gamma_set(f)
    assert rel_err(g, rg) < KTOL and rel_err(pr, rp) < KTOL
    for n in range(len(dims)):
        for q in range(len(dims)):
            assert np.array_equal(pr[n, q], pr[q, n])  # bitwise symmetric (test_kruskal.cpp:140-149)


def test_gamma_kat(ck):
    a = np.array([[1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    p = make(ck, np.zeros((3, 3, 3)), [a, a, a])
    g, pr = p.gamma_set()
    assert np.array_equal(g[0], [[2.0, 1.0], [1.0, 2.0]])
    assert np.array_equal(pr[0, 0], [[4.0, 1.0], [1.0, 4.0]])


@pytest.mark.parametrize("seed", range(6))
def test_residual_matches_oracle(orc, ck, seed):
    rng = np.random.default_rng(seed)
    order = 3 + seed % 2
    dims = [int(rng.integers(2, 9)) for _ in range(order)]
    rank = int(rng.integers(1, 9))
    m = gauss_factors(orc, dims, rank, 100 + seed)
    t = gauss_factors(orc, dims, rank, 200 + seed)
    x = orc.reconstruct(t)
    xn2 = orc.norm2(x)
    p = make(ck, x, m)
    assert abs(p.norm2() - xn2) <= 1e-13 * xn2
    p.mttkrp(order - 1)
    r, f = p.residual(xn2)
    rr, ff = orc.residual(x, m, xn2)
    assert abs(r - rr) < 1e-10
    dense = np.linalg.norm(x - orc.reconstruct(m)) / np.linalg.norm(x)
    assert abs(r - dense) < 1e-10


def test_residual_exact_model_floor(orc, ck):
    f = gauss_factors(orc, [3, 3, 3], 2, 23)
    x = orc.reconstruct(f)
    p = make(ck, x, f)
    p.mttkrp(2)
    r, fit = p.residual(orc.norm2(x))
    assert r < 1e-7 and fit > 1 - 1e-7


def test_gradient(orc, ck):
    f = gauss_factors(orc, [6, 5, 4], 3, 7)
    x = gauss_tensor(orc, [6, 5, 4], 99)
    p = make(ck, x, f)
    mk = [orc.mttkrp_naive(x, f, n) for n in range(3)]
    rg, rp = orc.gamma_set(f)
    p.gamma_set()
    g = p.gradient(mk)
    assert vec_rel_err(g, orc.gradient(f, mk, rg, rp)) < KTOL


# ---------------------------------------------------------------- J^T J v
@pytest.mark.parametrize("dims,rank,lam,shape", [
    ([3, 3, 3], 2, 0.0, 0), ([3, 2, 4], 3, 0.37, 0), ([3, 3, 3], 2, 0.25, 1),
    ([5, 4], 3, 0.1, 0), ([3, 4, 2, 5], 2, 1e-3, 0), ([2, 3, 2, 2, 3], 2, 0.5, 1),
    ([50, 50, 50], 5, 1e-2, 0), ([60, 45, 70], 40, 1e-3, 0), ([100, 100, 100, 100], 50, 1e-4, 1),
])
def test_jtj_matvec(orc, ck, dims, rank, lam, shape):
    f = gauss_factors(orc, dims, rank, 17)
    w = gauss_factors(orc, dims, rank, 18)
    p = ck.DeviceProblem(dims, rank)
    p.set_factors(f)
    p.gamma_set()
    g, pr = orc.gamma_set(f)
    got = p.jtj_matvec(w, lam, shape)
    ref = orc.hessian_matvec(f, g, pr, w, lam, shape)
    assert vec_rel_err(got, ref) < KTOL


def test_jtj_vs_explicit_and_identity(orc, ck):
    # test_gauss_newton.cpp:146-195 and acceptance c1
    rng = np.random.default_rng(17)
    for trial in range(12):
        order = 2 + int(rng.integers(0, 3))
        dims = [2 + int(rng.integers(0, 3)) for _ in range(order)]
        rank = 1 + int(rng.integers(0, 3))
        f = gauss_factors(orc, dims, rank, 300 + trial)
        w = gauss_factors(orc, dims, rank, 600 + trial)
        p = ck.DeviceProblem(dims, rank)
        p.set_factors(f)
        p.gamma_set()
        u = p.jtj_matvec(w, 0.0)
        exp = orc.explicit_jtj(f) @ orc.vec_stack(w)
        assert np.linalg.norm(orc.vec_stack(u) - exp) <= 1e-12 * np.linalg.norm(exp)
    f = gauss_factors(orc, [3, 3, 3], 2, 11)
    p = ck.DeviceProblem([3, 3, 3], 2)
    p.set_factors(f)
    grams = np.stack([np.eye(2)] * 3)
    pair = np.zeros((3, 3, 2, 2))
    for n in range(3):
        pair[n, n] = np.eye(2)
    p.set_gamma_set(grams, pair)
    w = gauss_factors(orc, [3, 3, 3], 2, 12)
    assert vec_rel_err(p.jtj_matvec(w, 0.0), w) < 1e-14


# ---------------------------------------------------------------- SPD / preconditioner
def test_spd_solve_and_inverse(orc, ck):
    # 166 .. 233: the blocked factorisation on the packed lower triangle (the
    # square R x (R+1) layout no longer fits shared memory), incl. a ragged tail block
    for R in (2, 5, 33, 100, 165, 166, 180, 200, 233):
        a = gauss_factors(orc, [R + 7], R, R)[0]
        s = orc.gram(a)
        b = gauss_factors(orc, [37], R, R + 1)[0]
        p = ck.DeviceProblem([3, 3], R)
        assert rel_err(p.spd_solve(s, b, 1e-3), orc.spd_solve(s, b, 1e-3)) < 1e-10
        assert rel_err(p.spd_inverse(s, 1e-3), orc.spd_inverse(s, 1e-3)) < 1e-10
    p = ck.DeviceProblem([3, 3], 2)
    assert np.allclose(p.spd_solve(2 * np.eye(2), np.eye(2), 0.0), 0.5 * np.eye(2))
    y = p.spd_solve(np.ones((2, 2)), np.ones((1, 2)), 0.0)  # jitter retry (test_tensor_core.cpp:280-288)
    assert np.isfinite(y).all()
    with pytest.raises(ck.CpkitError) as e:
        p.spd_solve(np.zeros((2, 2)), np.eye(2), 0.0)
    assert e.value.status == "singular_system"
    for R in (100, 200):  # jitter retry and SingularSystem on the square and the packed blocked kernels
        p = ck.DeviceProblem([3, 3], R)
        y = p.spd_solve(np.ones((R, R)), np.ones((3, R)), 0.0)
        assert np.isfinite(y).all()
        with pytest.raises(ck.CpkitError) as e:
            p.spd_solve(np.zeros((R, R)), np.eye(R)[:4], 0.0)
        assert e.value.status == "singular_system"


@pytest.mark.parametrize("shape", [0, 1])
def test_preconditioner(orc, ck, shape):
    f = gauss_factors(orc, [4, 4, 4], 3, 41)
    p = make(ck, np.zeros((4, 4, 4)), f)
    p.gamma_set()
    g, pr = orc.gamma_set(f)
    assert rel_err(p.preconditioner(1e-3, shape), orc.preconditioner(g, pr, 1e-3, shape)) < 1e-10


# ---------------------------------------------------------------- CG
@pytest.mark.parametrize("dims,rank,lam,cfg", [
    ([3, 3, 3], 2, 1e-3, {"cg_tol": 1e-10, "cg_max_iters": 10000}),
    ([6, 5, 7], 3, 1e-2, {}),
    ([8, 9, 7, 6], 4, 1e-3, {"cg_beta": "stale_denominator", "cg_max_iters": 50}),
    ([30, 25, 20], 6, 1e-4, {"reg": {"shape": "diagonal"}}),
    ([50, 50, 50], 5, 1e-2, {"cg_max_iters": 20}),
])
def test_cp_cg_matches_oracle(orc, ck, dims, rank, lam, cfg):
    f = gauss_factors(orc, dims, rank, 59)
    x = np.random.default_rng(1).standard_normal(dims)
    mk = [orc.mttkrp_naive(x, f, n) for n in range(len(dims))]
    g, pr = orc.gamma_set(f)
    grad = orc.gradient(f, mk, g, pr)
    ocfg = orc.GnConfig(cg_tol=cfg.get("cg_tol", 1e-3), cg_max_iters=cfg.get("cg_max_iters", 0),
                        cg_beta=1 if cfg.get("cg_beta") == "stale_denominator" else 0,
                        reg_shape=1 if cfg.get("reg", {}).get("shape") == "diagonal" else 0)
    v_ref, it_ref, cap_ref, bd_ref = orc.cp_cg(f, g, pr, grad, lam, ocfg)
    p = make(ck, x, f)
    p.gamma_set()
    v, it, cap, bd = p.cp_cg(grad, lam, cfg)
    assert (it, cap, bd) == (it_ref, cap_ref, bd_ref)
    assert vec_rel_err(v, v_ref) < 1e-9  # iterate after `it` steps (error grows with conditioning)


def test_cg_isolated_identity_and_zero_gradient(orc, ck):
    # test_gauss_newton.cpp:323-346
    f = gauss_factors(orc, [3, 3, 3], 2, 47)
    p = make(ck, np.zeros((3, 3, 3)), f)
    grams = np.stack([np.eye(2)] * 3)
    pair = np.zeros((3, 3, 2, 2))
    for n in range(3):
        pair[n, n] = np.eye(2)
    p.set_gamma_set(grams, pair)
    g = gauss_factors(orc, [3, 3, 3], 2, 48)
    v, it, _, _ = p.cp_cg(g, 0.0, {"cg_tol": 1e-10})
    assert it == 1
    for n in range(3):
        assert np.linalg.norm(v[n] + g[n]) <= 1e-12 * np.linalg.norm(g[n])
    p.gamma_set()
    v, it, _, _ = p.cp_cg([np.zeros((3, 2))] * 3, 1e-3)
    assert it == 0 and all(np.linalg.norm(a) == 0 for a in v)


# ---------------------------------------------------------------- GN / ALS drivers
def test_gn_step_matches_oracle(orc, ck):
    dims, rank = [12, 10, 9], 4
    t = orc.random_model(dims, rank, 5)
    x = orc.reconstruct(t) + 1e-3 * np.random.default_rng(0).standard_normal(dims)
    init = orc.random_model(dims, rank, 6)
    xn2 = orc.norm2(x)
    for cfg, ocfg in [({}, orc.GnConfig()),
                      ({"armijo": True, "reg": {"mode": "constant", "lambda": 1e-3}},
                       orc.GnConfig(armijo=1, reg_mode=0, lambda_=1e-3))]:
        p = make(ck, x, init)
        d = p.gn_step(cfg, xn2)
        f_ref, d_ref = orc.gn_step(x, init, ocfg, xn2)
        for k in ("halt", "stepped", "cg_iters", "alpha", "armijo_exhausted", "cg_hit_cap"):
            assert d[k] == d_ref[k], (k, d, d_ref)
        for k in ("residual_before", "residual_after", "grad_norm", "step_norm"):
            assert abs(d[k] - d_ref[k]) <= 1e-9 * max(1.0, abs(d_ref[k])), (k, d[k], d_ref[k])
        assert vec_rel_err(p.get_factors(), f_ref) < 1e-9


def test_gn_step_kats(orc, ck):
    # exact-fit halt (test_gauss_newton.cpp:384-407)
    f = gauss_factors(orc, [3, 3, 3], 2, 67)
    x = orc.reconstruct(f)
    p = make(ck, x, f)
    d = p.gn_step({}, orc.norm2(x))
    assert d["halt"] == 1 and d["stepped"] == 0
    # Armijo on the one-entry tensor [8] (test_gauss_newton.cpp:426-467)
    x = np.array([8.0]).reshape(1, 1, 1)
    p = make(ck, x, [np.ones((1, 1))] * 3)
    d = p.gn_step({"residual_tol": 0.0, "reg": {"mode": "constant", "lambda": 1e-3}, "armijo": True},
                  64.0)
    assert d["stepped"] == 1 and d["alpha"] < 1.0 and d["armijo_exhausted"] == 0
    p = make(ck, x, [np.ones((1, 1))] * 3)
    d = p.gn_step({"residual_tol": 0.0, "reg": {"mode": "constant", "lambda": 1e-3},
                   "armijo": {"c1": 0.999999, "shrink": 0.5, "max_backtracks": 2}}, 64.0)
    assert d["armijo_exhausted"] == 1 and d["alpha"] == pytest.approx(0.25)


@pytest.mark.parametrize("dims,rank", [([3, 4, 2], 2), ([12, 10, 9], 4), ([8, 7, 6, 5], 3)])
def test_als_sweep_matches_oracle(orc, ck, dims, rank):
    t = orc.random_model(dims, rank, 1)
    x = orc.reconstruct(t)
    init = orc.random_model(dims, rank, 2)
    f_ref, step_ref, cnt_ref, _ = orc.als_sweep(x, init, 1e-3)
    p = make(ck, x, init)
    step, cnt = p.als_sweep(1e-3)
    assert cnt == cnt_ref == 2
    assert abs(step - step_ref) <= 1e-9 * step_ref
    assert vec_rel_err(p.get_factors(), f_ref) < 1e-10


# Order-3 ALS runs the multi-sweep dimension tree (each single-mode root serves
# two consecutive updates; roots rotate c = 2, 1, 0). Sweep by sweep it must
# track the oracle's reference tree at roundoff level, with 3 roots per 2 sweeps.
# Extents cover batched-root stages that run past s1 (s1 % 32 != 0, s1 % 16 != 0).
# copies=1: the single-mode roots run as NN GEMMs on mode-permuted tensor
# copies; copies=0: TN GEMMs on X itself (needs an even rank and last extent).
MSDT_CASES = [([24, 20, 18], 6), ([10, 37, 22], 8), ([33, 48, 16], 20), ([6, 5, 4], 2)]


@pytest.mark.parametrize("copies", ["1", "0"])
@pytest.mark.parametrize("dims,rank", MSDT_CASES + [([9, 11, 7], 5), ([13, 6, 3], 3)])
def test_als_msdt_tracks_oracle(orc, ck, dims, rank, copies, monkeypatch):
    if copies == "0" and (rank % 2 or dims[-1] % 2):
        pytest.skip("TN single-mode roots need an even rank and last extent")
    monkeypatch.setenv("CPKIT_MSDT_COPIES", copies)
    t = orc.random_model(dims, rank, 3)
    x = orc.reconstruct(t) + 1e-3 * np.random.default_rng(5).standard_normal(dims)
    f = orc.random_model(dims, rank, 4)
    p = make(ck, x, f)
    counts = []
    for sweep in range(6):
        f, step_ref, _, _ = orc.als_sweep(x, f, 1e-4)
        step, cnt = p.als_sweep(1e-4)
        counts.append(cnt)
        assert abs(step - step_ref) <= 1e-9 * step_ref, (sweep, step, step_ref)
        assert vec_rel_err(p.get_factors(), f) < 1e-10, sweep
    assert counts == [2, 1, 2, 1, 2, 1]
    # every M^(n) of the final factors still matches the tree after the rotation
    ref, _ = orc.mttkrp_tree_all(x, f)
    for n in range(3):
        assert rel_err(p.mttkrp(n), ref[n]) < KTOL


def test_als_msdt_single_roots_match_oracle(orc, ck):
    """The single-mode roots feed M^(n) exactly as the tree does: after a sweep
    pair every mode's MTTKRP of the current factors from each route agrees."""
    dims, rank = [40, 36, 30], 10
    x = np.random.default_rng(9).standard_normal(dims)
    f = gauss_factors(orc, dims, rank, 12)
    p = make(ck, x, f)
    for _ in range(2):
        p.als_sweep(0.0)
    cur = p.get_factors()
    ref, _ = orc.mttkrp_tree_all(x, cur)
    for n in range(3):
        assert rel_err(p.mttkrp(n), ref[n]) < KTOL


def _c1(orc):
    """BASELINE config 1: order 3, s=50, R=5, uniform[0,1) truth, exact rank."""
    dims, rank = [50, 50, 50], 5
    truth = orc.random_model(dims, rank, orc.problem_seed(0, rank, 0))
    x = orc.reconstruct(truth)
    init = orc.random_model(dims, rank, orc.init_seed(0, rank, 0, 0))
    return dims, rank, x, init


def test_c1_gn_trace_matches_oracle(orc, ck):
    dims, rank, x, init = _c1(orc)
    _, recs, st = orc.gn_optimize(x, init, orc.GnConfig(cg_max_iters=20))
    p = ck.DeviceProblem(dims, rank)
    p.upload(x)
    got, rep = p.optimize({"optimizer": "gn", "gn": {"cg_max_iters": 20}}, init)
    j = rep.to_json()
    assert j["status"] == st
    assert len(j["records"]) == len(recs)
    for a, b in zip(j["records"], recs):
        assert a["cg_iters"] == b["cg_iters"] and a["lambda"] == b["lambda"]
        assert abs(a["residual"] - b["residual"]) < 1e-8


def test_c1_als_trace_matches_oracle(orc, ck):
    dims, rank, x, init = _c1(orc)
    cfg = orc.AlsConfig(max_sweeps=300)
    _, recs, st = orc.als_optimize(x, init, cfg)
    p = ck.DeviceProblem(dims, rank)
    p.upload(x)
    got, rep = p.optimize({"optimizer": "als", "als": {"max_sweeps": 300}}, init)
    j = rep.to_json()
    assert j["status"] == st and len(j["records"]) == len(recs)
    assert abs(j["records"][-1]["fitness"] - recs[-1]["fitness"]) < 1e-8


@pytest.mark.parametrize("cfg", [{"max_sweeps": 300}, {"max_sweeps": 7}, {"max_sweeps": 300, "step_tol": 1e-3},
                                 {"max_sweeps": 40, "lambda0": 1e-2, "decay_every": 5}])
def test_als_pipelined_driver_equals_sequential(ck, orc, cfg, monkeypatch):
    """als_optimize queues sweep k+1 before reading sweep k (restoring the
    factors when k stops the run): records and factors are bitwise those of
    the sequential loop, for every stop rule (residual, cap, step norm)."""
    dims, rank, x, init = _c1(orc)
    runs = []
    for flag in ("1", None):
        if flag:
            monkeypatch.setenv("CPKIT_ALS_NO_PIPELINE", flag)
        else:
            monkeypatch.delenv("CPKIT_ALS_NO_PIPELINE", raising=False)
        p = ck.DeviceProblem(dims, rank)
        p.upload(x)
        got, rep = p.optimize({"optimizer": "als", "als": cfg}, init)
        j = rep.to_json()
        runs.append((got, j["status"], [(r["residual"], r["lambda"]) for r in j["records"]]))
    (f1, s1, r1), (f2, s2, r2) = runs
    assert s1 == s2 and r1 == r2
    for a, b in zip(f1, f2):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("dims,rank", [([300, 120, 200], 100), ([400, 70, 90], 37), ([130, 257, 64], 200)])
def test_gram_cluster_bitwise(ck, orc, dims, rank, monkeypatch):
    """The cluster Gram kernel sums the row-split partial tiles in split order
    through distributed shared memory: bitwise the split + finalize path."""
    f = gauss_factors(orc, dims, rank, 41)
    x = np.zeros(dims)
    p = make(ck, x, f)
    g1, pr1 = p.gamma_set()
    monkeypatch.setenv("CPKIT_GRAM_NO_CLUSTER", "1")
    q = make(ck, x, f)
    g2, pr2 = q.gamma_set()
    assert np.array_equal(g1, g2) and np.array_equal(pr1, pr2)
    for n, a in enumerate(f):  # and the reference definition S = A^T A, symmetrised
        s = a.T @ a
        assert rel_err(g1[n], 0.5 * (s + s.T)) < KTOL


@pytest.mark.parametrize("cfg", [{"cg_max_iters": 20}, {"max_iters": 4, "cg_max_iters": 20},
                                 {"residual_tol": 1e-3, "cg_max_iters": 20},
                                 {"step_tol": 1e-2, "cg_max_iters": 20},
                                 {"grad_tol": 1e9, "cg_max_iters": 20}])
def test_gn_pipelined_driver_equals_sequential(ck, orc, cfg, monkeypatch):
    """gn_optimize queues step k+1 before reading step k (undoing the queued
    step, or step k itself, on stop): records and factors are bitwise those of
    the sequential loop for every stop rule (cap, residual, step norm, gradient halt)."""
    dims, rank, x, init = _c1(orc)
    runs = []
    for flag in ("1", None):
        if flag:
            monkeypatch.setenv("CPKIT_GN_NO_PIPELINE", flag)
        else:
            monkeypatch.delenv("CPKIT_GN_NO_PIPELINE", raising=False)
        p = ck.DeviceProblem(dims, rank)
        p.upload(x)
        got, rep = p.optimize({"optimizer": "gn", "gn": cfg}, init)
        j = rep.to_json()
        runs.append((got, j["status"], [(r["residual"], r["lambda"], r["cg_iters"]) for r in j["records"]]))
    (f1, s1, r1), (f2, s2, r2) = runs
    assert s1 == s2 and r1 == r2
    for a, b in zip(f1, f2):
        assert np.array_equal(a, b)


# ---------------------------------------------------------------- C ABI end to end
def test_decompose_through_c_abi(orc, ck):
    # test_capi.cpp:96-126 shape: gaussian [4,4,4] rank 2, GN
    m, t = ck.generate_low_rank({"family": "gaussian", "dims": [4, 4, 4], "rank": 2, "seed": 3})
    truth = orc.random_model([4, 4, 4], 2, 3, kind="gaussian")
    assert np.array_equal(t.numpy(), orc.reconstruct(truth))  # bitwise generator parity
    model, rep = ck.decompose(t, {"optimizer": "gn", "rank": 2, "seed": 19,
                                  "gn": {"max_iters": 200, "residual_tol": 5e-5}})
    assert model.rank == 2
    js = rep.to_json_text()
    assert '"kind": "trace"' in js
    assert rep.config()["optimizer"] == "gn"
    # oracle run on the same start point (cpkit_c.cpp:256-272: gaussian init, init_seed)
    init = orc.random_model([4, 4, 4], 2, orc.init_seed(19, 2, 0, 0), kind="gaussian")
    _, recs, st = orc.gn_optimize(t.numpy(), init, orc.GnConfig(max_iters=200))
    j = rep.to_json()
    assert j["status"] == st and len(j["records"]) == len(recs)


def test_c_abi_errors(ck):
    t = ck.Tensor.create(np.zeros((2, 2, 2)))
    with pytest.raises(ck.CpkitError) as e:
        ck.decompose(t, {"optimizer": "als", "rank": 1})
    assert e.value.status == "invalid_argument"  # zero-norm tensor
    t = ck.Tensor.create(np.ones((2, 2, 2)))
    with pytest.raises(ck.CpkitError) as e:
        ck.decompose(t, {"optimizer": "bogus", "rank": 1})
    assert e.value.status == "parse_error"
    with pytest.raises(ck.CpkitError) as e:
        ck.decompose(t, {"optimizer": "gn"})
    assert e.value.status == "invalid_argument"  # rank required


def test_als_graph_replay_bitwise_and_lambda_decay(orc, monkeypatch):
    """The ALS sweep runs as a CUDA graph replay (captured per lambda and cache state):
    bitwise equal to the eager launch sequence, re-captured when the decay schedule
    changes lambda, and the trace matches the oracle."""
    from paper_1910_12331_b200 import cpkit
    dims, R = [30, 26, 22], 6
    truth = orc.random_model(dims, R, orc.problem_seed(0, R, 0))
    x = orc.reconstruct(truth)
    init = orc.random_model(dims, R, orc.init_seed(0, R, 0, 0))
    cfg = {"optimizer": "als", "als": {"max_sweeps": 12, "residual_tol": 0.0, "step_tol": 0.0,
                                       "lambda0": 1e-2, "decay_factor": 2.0, "decay_every": 3}}
    p = cpkit.DeviceProblem(dims, R)
    p.upload(x)
    fa, ra = p.optimize(cfg, init)
    monkeypatch.setenv("CPKIT_NO_GRAPH", "1")
    q = cpkit.DeviceProblem(dims, R)
    q.upload(x)
    fb, rb = q.optimize(cfg, init)
    for a, b in zip(fa, fb):
        assert np.array_equal(a, b)
    ja, jb = ra.to_json(), rb.to_json()
    assert [r["residual"] for r in ja["records"]] == [r["residual"] for r in jb["records"]]
    _, recs, st = orc.als_optimize(x, init, orc.AlsConfig(max_sweeps=12, residual_tol=0.0, step_tol=0.0,
                                                          lambda0=1e-2, decay_factor=2.0, decay_every=3))
    assert ja["status"] == st and len(ja["records"]) == len(recs)
    for a, b in zip(ja["records"], recs):
        assert a["lambda"] == b["lambda"]
        assert abs(a["residual"] - b["residual"]) < 1e-10


def _pair_with_offdiag(N, R, c):
    grams = np.stack([np.eye(R)] * N)
    pair = np.zeros((N, N, R, R))
    for n in range(N):
        for q in range(N):
            pair[n, q] = np.eye(R) if n == q else c * np.ones((R, R))
    return grams, pair


@pytest.mark.parametrize("c", [1.0, 5.0])
def test_cg_breakdown_matches_oracle(orc, ck, c):
    """gauss_newton.cpp:318-324: <W, Q> <= 0 stops the solve with the current
    iterate (breakdown). An SPD preconditioner (Gamma(n,n) = I) with strongly
    negative off-diagonal Gamma blocks makes J^T J indefinite."""
    dims, R = [5, 4, 6], 3
    f = orc.random_model(dims, R, 3)
    g = orc.random_model(dims, R, 4, kind="gaussian")
    grams, pair = _pair_with_offdiag(3, R, -c)
    v_ref, it_ref, cap_ref, bd_ref = orc.cp_cg(f, grams, pair, g, 0.0, orc.GnConfig(cg_max_iters=50))
    assert bd_ref
    p = make(ck, np.zeros(dims), f)
    p.set_gamma_set(grams, pair)
    v, it, cap, bd = p.cp_cg(g, 0.0, {"cg_max_iters": 50})
    assert (it, cap, bd) == (it_ref, cap_ref, bd_ref)
    assert vec_rel_err(v, v_ref) < 1e-12


@pytest.mark.parametrize("c", [1e307, 1.7e308])
def test_cg_nonfinite_iterate_is_numerical_failure(orc, ck, c):
    """gauss_newton.cpp:341-343: a non-finite V or R after an iteration throws
    NumericalFailure, which the C ABI maps to CPKIT_ERR_NUMERICAL (5)."""
    dims, R = [5, 4, 6], 3
    f = orc.random_model(dims, R, 3)
    g = [np.abs(x) for x in orc.random_model(dims, R, 4, kind="gaussian")]
    grams, pair = _pair_with_offdiag(3, R, c)
    with pytest.raises(Exception, match="non-finite"):
        orc.cp_cg(f, grams, pair, g, 0.0, orc.GnConfig(cg_max_iters=50))
    p = make(ck, np.zeros(dims), f)
    p.set_gamma_set(grams, pair)
    with pytest.raises(ck.CpkitError) as ei:
        p.cp_cg(g, 0.0, {"cg_max_iters": 50})
    assert ei.value.code == 5 and "non-finite" in str(ei.value)


@pytest.mark.parametrize("dims", [[24, 22, 20, 18], [150, 150, 20, 10]])
@pytest.mark.parametrize("optimizer", ["als", "gn"])
def test_decompose_overlapped_first_root(ck, dims, optimizer):
    """cpkit_decompose on an order-4 tensor runs the start factors' back root
    slab by slab while the tensor crosses PCIe (solver.cu upload_tensor with
    start); the trace must equal the device path that uploads first and
    contracts after (cpkit_dev_optimize): bitwise with one slab, within
    roundoff with several (each slab's rows get their own tile plan)."""
    R = 6
    truth = ck.random_factors(dims, R, ck.problem_seed(2, R, 0))
    p0 = ck.DeviceProblem(dims, R)
    p0.generate(truth, noise_seed=3, noise_rel=1e-3)
    x = p0.download()
    p0.close()
    cfg = {"optimizer": optimizer, "rank": R, "seed": 4, "init": {"distribution": "uniform", "a": 0.0, "b": 1.0},
           "als": {"max_sweeps": 6, "residual_tol": 0.0, "step_tol": 0.0}, "gn": {"max_iters": 4}}
    m, rep = ck.decompose(ck.Tensor.create(x), cfg)
    j = rep.to_json()
    init = ck.random_factors(dims, R, ck.init_seed(4, R, 0, 0))
    p = ck.DeviceProblem(dims, R)
    p.upload(x)
    f, rep2 = p.optimize(cfg, init)
    j2 = rep2.to_json()
    assert len(j["records"]) == len(j2["records"]) > 0
    one_slab = dims[0] * dims[1] < 20000
    for a, b in zip(j["records"], j2["records"]):
        assert a["cg_iters"] == b["cg_iters"] and a["lambda"] == b["lambda"]
        if one_slab:
            assert a["residual"] == b["residual"], (a, b)
        else:
            assert abs(a["residual"] - b["residual"]) < 1e-10, (a, b)
    assert vec_rel_err(m.factors(), f) < (1e-15 if one_slab else 1e-9)


def test_second_level_timing_seam_leaves_results_intact(orc, ck):
    """cpkit_dev_time_second_level (bench.py's HBM line item) repeats the second tree level on
    the cached back-root partial; the MTTKRPs afterwards still match the oracle."""
    dims, rank = [24, 18, 20, 16], 12
    x = np.random.default_rng(7).standard_normal(dims)
    f = gauss_factors(orc, dims, rank, 41)
    ref, _ = orc.mttkrp_tree_all(x, f)
    p = make(ck, x, f)
    ms, nbytes = p.time_second_level(3)
    assert ms > 0.0 and nbytes == 8.0 * dims[0] * dims[1] * rank
    for n in range(len(dims)):
        assert rel_err(p.mttkrp(n), ref[n]) < KTOL, n


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# Back roots with fewer row tiles than SMs and a long contraction run as one
# stream-K launch (every CTA an equal run of k blocks; tiles shared by several
# CTAs summed in fixed k order by the fix-up kernel) instead of a k split into
# full-size slabs. Against the oracle, bitwise repeatable, and against the
# classic split-K path (CPKIT_NO_STREAMK=1; env read once per process).
@pytest.mark.parametrize("dims,rank", [([30, 40, 70, 64], 24), ([1000, 5000], 50), ([30, 31, 4500], 77)])
def test_root_stream_k(orc, ck, dims, rank, tmp_path):
    import subprocess
    import sys
    x = np.random.default_rng(rank + 1).standard_normal(dims)
    f = gauss_factors(orc, dims, rank, 23)
    ref, _ = orc.mttkrp_tree_all(x, f)
    np.save(tmp_path / "x.npy", x)
    np.save(tmp_path / "f.npy", np.concatenate([a.ravel() for a in f]))
    code = f"""
import sys, numpy as np
sys.path.insert(0, {repr(str(ROOT))})
from paper_1910_12331_b200 import cpkit
x = np.load({repr(str(tmp_path / 'x.npy'))}); flat = np.load({repr(str(tmp_path / 'f.npy'))})
dims, R = {dims!r}, {rank}
f, at = [], 0
for d in dims:
    f.append(flat[at:at + d * R].reshape(d, R)); at += d * R
p = cpkit.DeviceProblem(dims, R); p.upload(x); p.set_factors(f)
a = p.mttkrp_naive(0)
assert np.array_equal(a, p.mttkrp_naive(0))
np.save(sys.argv[1], a)
"""
    outs = {}
    for tag, env_add in (("sk", {"CPKIT_PLAN_DEBUG": "1"}), ("classic", {"CPKIT_PLAN_DEBUG": "1", "CPKIT_NO_STREAMK": "1"})):
        r = subprocess.run([sys.executable, "-c", code, str(tmp_path / f"{tag}.npy")], env=dict(os.environ, **env_add),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        assert ("plan stream-K" in r.stderr) == (tag == "sk"), r.stderr[-2000:]
        outs[tag] = np.load(tmp_path / f"{tag}.npy")
    assert rel_err(outs["sk"], ref[0]) < KTOL
    assert rel_err(outs["sk"], outs["classic"]) < 1e-13


M8_CASES = [([30, 28, 26, 24], 200), ([40, 36, 34], 120), ([400, 50, 40], 200)]


@pytest.mark.parametrize("dims,R", M8_CASES)
def test_odd_cell_root_kernels(orc, ck, dims, R, tmp_path):
    """Ranks with an odd number of n8 cells (R = 200: 25) run the NN roots
    without rank padding: by default the m16n8k16 kernel with the row-split
    dealing (RS: 13 + 12 cells per m16 row), with CPKIT_NN_RS=0 the m8n8k4
    strip kernel, with CPKIT_NN_M8=0 as well the padded m16 plan. Every mode's
    MTTKRP against the oracle, and the three variants against each other (the
    env switches are read once per process: subprocesses)."""
    import subprocess
    import sys
    f = gauss_factors(orc, dims, R, 61)
    x = np.random.default_rng(5).standard_normal(dims)
    p = make(ck, x, f)
    got = np.concatenate([p.mttkrp(n).ravel() for n in range(len(dims))])
    ref, _ = orc.mttkrp_tree_all(x, f)
    for n in range(len(dims)):
        assert rel_err(p.mttkrp(n), ref[n]) < 1e-11, n
    np.save(tmp_path / "x.npy", x)
    np.save(tmp_path / "f.npy", np.concatenate([a.ravel() for a in f]))
    for tag, env_add in (("m8", {"CPKIT_NN_RS": "0"}), ("pad", {"CPKIT_NN_RS": "0", "CPKIT_NN_M8": "0"})):
        code = f"""
import sys, numpy as np
sys.path.insert(0, {repr(str(ROOT))})
from paper_1910_12331_b200 import cpkit
x = np.load({repr(str(tmp_path / 'x.npy'))}); flat = np.load({repr(str(tmp_path / 'f.npy'))})
dims, R = {dims!r}, {R}
f, at = [], 0
for d in dims:
    f.append(flat[at:at + d * R].reshape(d, R)); at += d * R
p = cpkit.DeviceProblem(dims, R); p.upload(x); p.set_factors(f)
np.save({repr(str(tmp_path / 'v.npy'))}, np.concatenate([p.mttkrp(n).ravel() for n in range(len(dims))]))
"""
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env_add), capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        assert rel_err(got, np.load(tmp_path / "v.npy")) < 1e-13, tag
