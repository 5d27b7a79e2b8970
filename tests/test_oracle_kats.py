"""Pins the CPU oracle to every known-answer and property test the reference
suites hold for the hot path. CPU only.

Each test cites the reference test it restates. Random inputs come from the
reference's keyed RNG instead of std::mt19937 (same distribution family).
"""
import math

import numpy as np
import pytest

from tests.helpers import (gauss_factors, gauss_matrix, gauss_tensor, khatri_rao, matricize,
                           mttkrp_unfold, rel_err, vec_rel_err)


# ---------------------------------------------------------------- rng / generators
def test_rng_bitwise_determinism(orc):
    # test_generators.cpp:20-35
    a = orc.random_model([3, 4, 2], 2, 321, kind="gaussian")
    b = orc.random_model([3, 4, 2], 2, 321, kind="gaussian")
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    c = orc.random_model([3, 4, 2], 2, 322, kind="gaussian")
    assert not np.array_equal(a[0], c[0])


def test_uniform_interval_and_gaussian_mean(orc):
    # test_generators.cpp:37-55
    m = orc.random_model([20, 20], 5, 7, kind="uniform", a=-1.0, b=1.0)
    for f in m:
        assert f.min() >= -1.0 and f.max() < 1.0
    g = orc.random_model([50, 50, 50], 10, 99, kind="gaussian")
    allv = np.concatenate([f.ravel() for f in g])
    assert abs(allv.mean()) <= 4.0 / math.sqrt(allv.size)


def test_positive_uniform_factors_positive_tensor(orc):
    # test_generators.cpp:12-18
    f = orc.random_model([4, 4, 4], 3, orc.problem_seed(11, 3, 0))
    assert (orc.reconstruct(f) > 0).all()


def test_mix64_reference_values(orc):
    # SplitMix64 finalizer constants (rng.hpp:11-16): mix64(0) is the first
    # SplitMix64 output for state 0, a published value.
    assert orc.mix64(0) == 0xE220A8397B1DCDAF


def test_ground_truth_residual_floor(orc):
    # test_generators.cpp:135-151
    for seed in range(5):
        f = orc.random_model([4, 4, 4], 6, seed, kind="uniform", a=-1.0, b=1.0)
        x = orc.reconstruct(f)
        r, _ = orc.residual(x, f, orc.norm2(x))
        assert r <= 1e-7


# ---------------------------------------------------------------- matrix ops
def test_gram_examples(orc):
    # test_tensor_core.cpp:155-163
    assert np.allclose(orc.gram(np.eye(3)), np.eye(3))
    assert np.allclose(orc.gram(np.ones((3, 2))), 3 * np.ones((2, 2)))
    assert np.array_equal(orc.gram(np.array([[1.0, 2.0], [3.0, 4.0]])),
                          np.array([[10.0, 14.0], [14.0, 20.0]]))


def test_spd_solve_examples(orc):
    # test_tensor_core.cpp:254-288
    assert np.allclose(orc.spd_solve(2 * np.eye(2), np.eye(2), 0.0), 0.5 * np.eye(2))
    b = gauss_matrix(orc, 3, 2, 31)
    assert np.allclose(orc.spd_solve(np.eye(2), b, 1.0), 0.5 * b)
    s = orc.gram(gauss_matrix(orc, 4, 4, 37))
    b = gauss_matrix(orc, 4, 4, 38)
    y = orc.spd_solve(s, b, 1e-3)
    assert np.linalg.norm(y @ (s + 1e-3 * np.eye(4)) - b) <= 1e-10 * np.linalg.norm(b)
    with pytest.raises(orc.OracleError) as e:
        orc.spd_solve(np.zeros((2, 2)), np.eye(2), 0.0)
    assert e.value.code == 4  # CPKIT_ERR_SINGULAR
    y = orc.spd_solve(np.ones((2, 2)), np.ones((1, 2)), 0.0)  # jitter retry
    assert np.isfinite(y).all()


def test_spd_inverse_examples(orc):
    # test_tensor_core.cpp:290-301
    assert np.allclose(orc.spd_inverse(np.eye(2), 0.0), np.eye(2))
    assert np.allclose(orc.spd_inverse(np.diag([1.0, 3.0]), 1.0), np.diag([0.5, 0.25]))
    sp = orc.gram(gauss_matrix(orc, 5, 4, 41))
    inv = orc.spd_inverse(sp, 1e-3)
    assert np.linalg.norm(inv @ (sp + 1e-3 * np.eye(4)) - np.eye(4)) < 1e-10


# ---------------------------------------------------------------- MTTKRP
def test_mttkrp_all_ones(orc):
    # test_tensor_core.cpp:178-182
    x = np.ones((2, 2, 2))
    f = [np.ones((2, 2))] * 3
    assert np.array_equal(orc.mttkrp_naive(x, f, 0), 4 * np.ones((2, 2)))


def test_mttkrp_rank1(orc):
    # test_tensor_core.cpp:184-199
    a = np.array([1.0, -2.0, 0.5]); b = np.array([2.0, 1.0, 1.0]); c = np.array([0.5, 3.0, -1.0])
    x = np.einsum("i,j,k->ijk", a, b, c)
    m = orc.mttkrp_naive(x, [a[:, None], b[:, None], c[:, None]], 0)
    assert rel_err(m, a[:, None] * (b @ b) * (c @ c)) < 1e-12


def test_mttkrp_matches_unfolding(orc):
    # test_tensor_core.cpp:201-208
    x = gauss_tensor(orc, [3, 3, 3], 17)
    f = gauss_factors(orc, [3, 3, 3], 2, 18)
    naive = matricize(x, 0) @ khatri_rao(f[1], f[2])
    assert rel_err(orc.mttkrp_naive(x, f, 0), naive) < 1e-12


@pytest.mark.parametrize("order", [3, 4, 5])
def test_workspace_tree_matches_unfolding_within_budget(orc, order):
    # test_tensor_core.cpp:210-231
    dims = [3] * order
    x = gauss_tensor(orc, dims, 23 + order)
    f = gauss_factors(orc, dims, 4, 100 + order)
    ms, cnt = orc.mttkrp_tree_all(x, f)
    for n in range(order):
        assert rel_err(ms[n], mttkrp_unfold(x, f, n)) < 1e-12
    assert cnt <= 2


def test_mttkrp_odd_dims_orders_2_to_5(orc):
    for order, dims in [(2, [5, 3]), (3, [3, 4, 2]), (4, [2, 3, 4, 5]), (5, [3, 2, 2, 3, 2])]:
        x = gauss_tensor(orc, dims, 7)
        f = gauss_factors(orc, dims, 3, 8)
        ms, cnt = orc.mttkrp_tree_all(x, f)
        for n in range(order):
            ref = mttkrp_unfold(x, f, n)
            assert rel_err(ms[n], ref) < 1e-12
            assert rel_err(orc.mttkrp_naive(x, f, n), ref) < 1e-12
        assert cnt <= 2


def test_mttkrp_input_validation(orc):
    # test_tensor_core.cpp:246-252
    x = np.zeros((2, 2, 2))
    with pytest.raises(orc.OracleError):
        orc.mttkrp_naive(x, [np.ones((2, 2))] * 3, 3)


# ---------------------------------------------------------------- Gamma / residual
def test_gamma_identity(orc):
    # test_kruskal.cpp:99-111
    grams, pair = orc.gamma_set([np.eye(2)] * 3)
    for n in range(3):
        for p in range(3):
            assert np.allclose(pair[n, p], np.eye(2))


def test_gamma_hadamard_kat(orc):
    # test_kruskal.cpp:113-130
    a = np.array([[1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    grams, pair = orc.gamma_set([a, a, a])
    s = np.array([[2.0, 1.0], [1.0, 2.0]])
    assert np.array_equal(grams[0], s)
    assert np.array_equal(pair[0, 1], s)
    assert np.array_equal(pair[0, 0], np.array([[4.0, 1.0], [1.0, 4.0]]))


def test_gamma_order2_empty_product(orc):
    # test_kruskal.cpp:132-138
    f = gauss_factors(orc, [3, 4], 2, 17)
    grams, pair = orc.gamma_set(f)
    assert np.array_equal(pair[0, 1], np.ones((2, 2)))
    assert np.allclose(pair[0, 0], grams[1])


def test_gamma_bitwise_symmetric(orc):
    # test_kruskal.cpp:140-149
    f = gauss_factors(orc, [3, 2, 4, 2], 3, 19)
    _, pair = orc.gamma_set(f)
    for n in range(4):
        for p in range(4):
            assert np.array_equal(pair[n, p], pair[p, n])


def test_residual_exact_and_zero_models(orc):
    # test_kruskal.cpp:151-168
    f = gauss_factors(orc, [3, 3, 3], 2, 23)
    x = orc.reconstruct(f)
    r, fit = orc.residual(x, f, orc.norm2(x))
    assert r < 1e-7 and fit > 1 - 1e-7
    z = [np.zeros((3, 2))] * 3
    r, fit = orc.residual(x, z, orc.norm2(x))
    assert r == pytest.approx(1.0) and fit == pytest.approx(0.0)


def test_fast_residual_matches_dense(orc):
    # test_kruskal.cpp:170-192 (30 trials, N in {3,4}, s in [2,6], R in [1,8])
    rng = np.random.default_rng(31)
    for trial in range(30):
        order = 3 + int(rng.integers(0, 2))
        dims = [2 + int(rng.integers(0, 5)) for _ in range(order)]
        rank = 1 + int(rng.integers(0, 8))
        m = gauss_factors(orc, dims, rank, 1000 + trial)
        t = gauss_factors(orc, dims, rank, 2000 + trial)
        x = orc.reconstruct(t)
        r, fit = orc.residual(x, m, orc.norm2(x))
        dense = np.linalg.norm(x - orc.reconstruct(m)) / np.linalg.norm(x)
        assert abs(r - dense) < 1e-10
        assert fit == pytest.approx(1 - r)


def test_residual_rejects_zero_norm(orc):
    # test_kruskal.cpp:194-198
    with pytest.raises(orc.OracleError) as e:
        orc.residual(np.zeros((2, 2)), [np.zeros((2, 1))] * 2, 0.0)
    assert e.value.code == 1


# ---------------------------------------------------------------- GN pieces
def test_schedule_kat(orc):
    # test_gauss_newton.cpp:69-76
    lam, d = 1e-2, 0
    for v in [5e-3, 2.5e-3, 1.25e-3, 6.25e-4, 1.25e-3, 2.5e-3]:
        lam, d = orc.schedule_next(1, lam, 2.0, 1e-3, 1e-2, d)
        assert lam == pytest.approx(v)


def test_schedule_band_and_constant(orc):
    # test_gauss_newton.cpp:78-103
    lam, d = 1e-2, 0
    for _ in range(200):
        lam, d = orc.schedule_next(1, lam, 3.0, 1e-6, 1e-2, d)
        assert 1e-6 / 3 <= lam <= 1e-2 * 3
    lam, d = 1e-3, 0
    for _ in range(10):
        lam, d = orc.schedule_next(0, lam, 2.0, 1e-6, 1e-2, d)
        assert lam == 1e-3


def test_gradient_exact_fit_and_zero_tensor(orc):
    # test_gauss_newton.cpp:111-132
    f = gauss_factors(orc, [4, 4, 4], 3, 3)
    x = orc.reconstruct(f)
    mk = [orc.mttkrp_naive(x, f, n) for n in range(3)]
    grams, pair = orc.gamma_set(f)
    for g in orc.gradient(f, mk, grams, pair):
        assert np.linalg.norm(g) <= 1e-10 * np.linalg.norm(x)
    f = gauss_factors(orc, [3, 3, 3], 2, 5)
    grams, pair = orc.gamma_set(f)
    g = orc.gradient(f, [np.zeros((3, 2))] * 3, grams, pair)
    for n in range(3):
        assert np.allclose(g[n], f[n] @ pair[n, n])


def _dense_objective(x, f):
    return 0.5 * float(np.sum((x - np.einsum("ir,jr,kr->ijk", *f)) ** 2))


def test_gradient_matches_finite_differences(orc):
    # test_gauss_newton.cpp:134-144 (h = 1e-5, tolerance 1e-6)
    f = gauss_factors(orc, [4, 4, 4], 3, 7)
    x = gauss_tensor(orc, [4, 4, 4], 99)
    mk = [orc.mttkrp_naive(x, f, n) for n in range(3)]
    grams, pair = orc.gamma_set(f)
    g = orc.gradient(f, mk, grams, pair)
    fd = []
    h = 1e-5
    for n in range(3):
        gn = np.zeros_like(f[n])
        for i in range(f[n].shape[0]):
            for r in range(f[n].shape[1]):
                p = [a.copy() for a in f]
                p[n][i, r] += h
                fp = _dense_objective(x, p)
                p[n][i, r] -= 2 * h
                fm = _dense_objective(x, p)
                gn[i, r] = (fp - fm) / (2 * h)
        fd.append(gn)
    assert vec_rel_err(g, fd) < 1e-6


def _isolated_identity(order, rank):
    # test_gauss_newton.cpp:44-55
    grams = np.stack([np.eye(rank)] * order)
    pair = np.zeros((order, order, rank, rank))
    for n in range(order):
        pair[n, n] = np.eye(rank)
    return grams, pair


def test_matvec_isolated_identity_and_zero(orc):
    # test_gauss_newton.cpp:146-167
    f = gauss_factors(orc, [3, 3, 3], 2, 11)
    grams, pair = _isolated_identity(3, 2)
    w = gauss_factors(orc, [3, 3, 3], 2, 12)
    u = orc.hessian_matvec(f, grams, pair, w, 0.0)
    assert vec_rel_err(u, w) < 1e-14
    f = gauss_factors(orc, [3, 2, 4], 3, 13)
    grams, pair = orc.gamma_set(f)
    u = orc.hessian_matvec(f, grams, pair, [np.zeros((d, 3)) for d in (3, 2, 4)], 3.5)
    assert all(np.linalg.norm(x) == 0.0 for x in u)


def test_matvec_vs_explicit_jtj(orc):
    # test_gauss_newton.cpp:169-195 (40 trials) and acceptance c1
    rng = np.random.default_rng(17)
    for trial in range(40):
        order = 2 + int(rng.integers(0, 3))
        dims = [2 + int(rng.integers(0, 3)) for _ in range(order)]
        rank = 1 + int(rng.integers(0, 3))
        f = gauss_factors(orc, dims, rank, 300 + trial)
        grams, pair = orc.gamma_set(f)
        w = gauss_factors(orc, dims, rank, 600 + trial)
        u = orc.hessian_matvec(f, grams, pair, w, 0.0)
        exp = orc.explicit_jtj(f) @ orc.vec_stack(w)
        assert np.linalg.norm(orc.vec_stack(u) - exp) <= 1e-12 * np.linalg.norm(exp)
        ud = orc.hessian_matvec(f, grams, pair, w, 0.37)
        for n in range(order):
            diff = ud[n] - u[n] - 0.37 * w[n]
            assert np.abs(diff).max() <= 1e-13 * np.abs(w[n]).max()


def test_matvec_diagonal_shape_and_linearity(orc):
    # test_gauss_newton.cpp:197-232
    f = gauss_factors(orc, [3, 3, 3], 2, 19)
    grams, pair = orc.gamma_set(f)
    w = gauss_factors(orc, [3, 3, 3], 2, 20)
    u0 = orc.hessian_matvec(f, grams, pair, w, 0.0, shape=1)
    u = orc.hessian_matvec(f, grams, pair, w, 0.25, shape=1)
    for n in range(3):
        exp = u0[n] + 0.25 * w[n] * np.diag(pair[n, n])[None, :]
        assert np.allclose(u[n], exp, rtol=1e-12, atol=0)
    f = gauss_factors(orc, [3, 4, 2], 3, 23)
    grams, pair = orc.gamma_set(f)
    w1 = gauss_factors(orc, [3, 4, 2], 3, 24)
    w2 = gauss_factors(orc, [3, 4, 2], 3, 25)
    combo = [1.7 * a - 0.4 * b for a, b in zip(w1, w2)]
    u1 = orc.hessian_matvec(f, grams, pair, w1, 0.1)
    u2 = orc.hessian_matvec(f, grams, pair, w2, 0.1)
    uc = orc.hessian_matvec(f, grams, pair, combo, 0.1)
    assert vec_rel_err(uc, [1.7 * a - 0.4 * b for a, b in zip(u1, u2)]) < 1e-12


def test_explicit_jtj_kats(orc):
    # test_gauss_newton.cpp:234-278
    h = orc.explicit_jtj([np.ones((1, 1)), np.ones((1, 1))])
    assert np.allclose(h, np.ones((2, 2)))
    f = gauss_factors(orc, [3, 3, 3], 2, 29)
    h = orc.explicit_jtj(f)
    assert np.abs(h - h.T).max() == 0.0
    ev = np.linalg.eigvalsh(h)
    assert ev.min() >= -1e-10 * ev.max()
    with pytest.raises(orc.OracleError) as e:
        orc.explicit_jtj(gauss_factors(orc, [4, 4, 4], 3, 37), var_cap=10)
    assert e.value.code == 6


def test_preconditioner_kats(orc):
    # test_gauss_newton.cpp:280-311
    p = orc.preconditioner(np.eye(2)[None], np.eye(2)[None, None], 1.0)
    assert np.allclose(p[0], 0.5 * np.eye(2))
    d = np.diag([1.0, 3.0])
    p = orc.preconditioner(d[None], d[None, None], 0.0)
    assert np.allclose(p[0], np.diag([1.0, 1.0 / 3.0]))
    f = gauss_factors(orc, [4, 4, 4], 3, 41)
    grams, pair = orc.gamma_set(f)
    p = orc.preconditioner(grams, pair, 1e-3)
    for n in range(3):
        assert np.linalg.norm(p[n] @ (pair[n, n] + 1e-3 * np.eye(3)) - np.eye(3)) < 1e-10
    p = orc.preconditioner(grams, pair, 1e-3, shape=1)
    for n in range(3):
        s = pair[n, n].copy()
        s[np.diag_indices(3)] *= 1.001
        assert np.linalg.norm(p[n] @ s - np.eye(3)) < 1e-10


def test_cg_isolated_identity_one_iteration(orc):
    # test_gauss_newton.cpp:323-336
    f = gauss_factors(orc, [3, 3, 3], 2, 47)
    grams, pair = _isolated_identity(3, 2)
    g = gauss_factors(orc, [3, 3, 3], 2, 48)
    v, it, cap, bd = orc.cp_cg(f, grams, pair, g, 0.0, orc.GnConfig(cg_tol=1e-10))
    assert it == 1
    for n in range(3):
        assert np.linalg.norm(v[n] + g[n]) <= 1e-12 * np.linalg.norm(g[n])


def test_cg_zero_gradient(orc):
    # test_gauss_newton.cpp:338-346
    f = gauss_factors(orc, [3, 3, 3], 2, 53)
    grams, pair = orc.gamma_set(f)
    v, it, _, _ = orc.cp_cg(f, grams, pair, [np.zeros((3, 2))] * 3, 1e-3, orc.GnConfig())
    assert it == 0 and all(np.linalg.norm(x) == 0 for x in v)


def test_cg_matches_dense_solve(orc):
    # test_gauss_newton.cpp:348-367 and acceptance c4
    f = gauss_factors(orc, [3, 3, 3], 2, 59)
    x = gauss_tensor(orc, [3, 3, 3], 1234)
    mk = [orc.mttkrp_naive(x, f, n) for n in range(3)]
    grams, pair = orc.gamma_set(f)
    g = orc.gradient(f, mk, grams, pair)
    v, it, _, _ = orc.cp_cg(f, grams, pair, g, 1e-3, orc.GnConfig(cg_tol=1e-10, cg_max_iters=10000))
    h = orc.explicit_jtj(f) + 1e-3 * np.eye(18)
    dense = np.linalg.solve(h, -orc.vec_stack(g))
    assert np.linalg.norm(orc.vec_stack(v) - dense) <= 1e-6 * np.linalg.norm(dense)


def test_cg_stale_denominator_finite(orc):
    # test_gauss_newton.cpp:369-382
    f = gauss_factors(orc, [3, 3, 3], 2, 61)
    x = gauss_tensor(orc, [3, 3, 3], 77)
    mk = [orc.mttkrp_naive(x, f, n) for n in range(3)]
    grams, pair = orc.gamma_set(f)
    g = orc.gradient(f, mk, grams, pair)
    v, _, _, _ = orc.cp_cg(f, grams, pair, g, 1e-2, orc.GnConfig(cg_beta=1, cg_max_iters=50))
    assert all(np.isfinite(a).all() for a in v)


def test_gn_step_exact_fit_halts(orc):
    # test_gauss_newton.cpp:384-407
    f = gauss_factors(orc, [3, 3, 3], 2, 67)
    x = orc.reconstruct(f)
    f2, d = orc.gn_step(x, f, orc.GnConfig(), orc.norm2(x))
    assert d["halt"] == 1 and d["stepped"] == 0
    assert all(np.array_equal(a, b) for a, b in zip(f, f2))
    f3, d = orc.gn_step(x, f, orc.GnConfig(residual_tol=0.0, grad_tol=1e-9), orc.norm2(x))
    assert d["halt"] == 2 and d["grad_norm"] <= 1e-9


def test_gn_step_reduces_residual(orc):
    # test_gauss_newton.cpp:409-424
    t = gauss_factors(orc, [3, 3, 3], 1, 71)
    x = orc.reconstruct(t)
    p = gauss_factors(orc, [3, 3, 3], 1, 72)
    m = [a + 0.01 * b for a, b in zip(t, p)]
    cfg = orc.GnConfig(residual_tol=0.0, reg_mode=0, lambda_=1e-5)
    _, d = orc.gn_step(x, m, cfg, orc.norm2(x))
    assert d["stepped"] == 1 and d["residual_after"] < d["residual_before"]


def test_armijo_backtracks_and_exhausts(orc):
    # test_gauss_newton.cpp:426-467 (one-entry tensor [8] from (1,1,1))
    x = np.array([8.0]).reshape(1, 1, 1)
    m = [np.ones((1, 1))] * 3
    cfg = orc.GnConfig(residual_tol=0.0, reg_mode=0, lambda_=1e-3, armijo=1)
    _, d = orc.gn_step(x, m, cfg, orc.norm2(x))
    assert d["stepped"] == 1 and d["alpha"] < 1.0 and d["armijo_exhausted"] == 0
    assert d["residual_after"] < d["residual_before"]
    cfg = orc.GnConfig(residual_tol=0.0, reg_mode=0, lambda_=1e-3, armijo=1, c1=0.999999,
                       shrink=0.5, max_backtracks=2)
    f2, d = orc.gn_step(x, m, cfg, orc.norm2(x))
    assert d["armijo_exhausted"] == 1 and d["alpha"] == pytest.approx(0.25)
    assert not np.array_equal(f2[0], m[0])


def test_gn_optimize_recovers_rank2(orc):
    # test_gauss_newton.cpp:469-482
    conv = 0
    for seed in range(5):
        t = orc.random_model([4, 4, 4], 2, seed, kind="uniform", a=-1.0, b=1.0)
        x = orc.reconstruct(t)
        init = orc.random_model([4, 4, 4], 2, seed + 900, kind="uniform", a=-1.0, b=1.0)
        _, recs, status = orc.gn_optimize(x, init, orc.GnConfig())
        conv += status == "converged_residual"
    assert conv >= 3


def test_gn_zero_iteration_cap(orc):
    # test_gauss_newton.cpp:484-497
    t = gauss_factors(orc, [3, 3, 3], 2, 73)
    x = orc.reconstruct(t)
    init = gauss_factors(orc, [3, 3, 3], 2, 74)
    f, recs, st = orc.gn_optimize(x, init, orc.GnConfig(max_iters=0))
    assert recs == [] and st == "cap_hit"
    assert all(np.array_equal(a, b) for a, b in zip(f, init))


# ---------------------------------------------------------------- ALS
def test_als_first_subproblem_exact(orc):
    # test_als.cpp:43-59
    t = gauss_factors(orc, [3, 3, 3], 1, 3)
    x = orc.reconstruct(t)
    start = [gauss_matrix(orc, 3, 1, 4), t[1], t[2]]
    f, step, cnt, _ = orc.als_sweep(x, start, 0.0)
    assert np.linalg.norm(f[0] - t[0]) < 1e-12 * np.linalg.norm(t[0])
    assert np.linalg.norm(x - orc.reconstruct(f)) / np.linalg.norm(x) < 1e-12
    assert cnt <= 2


def test_als_huge_lambda_collapses(orc):
    # test_als.cpp:61-75
    t = gauss_factors(orc, [4, 4, 4], 2, 7)
    x = orc.reconstruct(t)
    m = gauss_factors(orc, [4, 4, 4], 2, 8)
    m0 = orc.mttkrp_naive(x, m, 0)
    f, _, _, _ = orc.als_sweep(x, m, 1e12)
    assert np.linalg.norm(f[0]) <= 1e-6 * np.linalg.norm(m0)


def test_als_monotone(orc):
    # test_als.cpp:77-93 and :167-182 (acceptance c5)
    for seed in range(5):
        t = orc.random_model([4, 4, 4], 5, seed, kind="uniform", a=-1.0, b=1.0)
        x = orc.reconstruct(t)
        m = orc.random_model([4, 4, 4], 5, seed + 500, kind="uniform", a=-1.0, b=1.0)
        prev = np.linalg.norm(x - orc.reconstruct(m)) / np.linalg.norm(x)
        for _ in range(40):
            m, _, cnt, _ = orc.als_sweep(x, m, 0.0)
            assert cnt == 2
            cur = np.linalg.norm(x - orc.reconstruct(m)) / np.linalg.norm(x)
            assert cur <= prev + 1e-12
            prev = cur


def test_als_stationary_point(orc):
    # test_als.cpp:95-108
    m = gauss_factors(orc, [3, 3, 3], 2, 13)
    x = orc.reconstruct(m)
    f, _, _, _ = orc.als_sweep(x, m, 0.0)
    for a, b in zip(f, m):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)


def test_als_decay_schedule_kat(orc):
    # test_als.cpp:146-165
    t = orc.random_model([3, 3, 3], 2, 5)
    x = orc.reconstruct(t)
    init = orc.random_model([3, 3, 3], 2, 77)
    cfg = orc.AlsConfig(max_sweeps=7, residual_tol=0.0, step_tol=0.0, lambda0=0.01,
                        decay_factor=2.0, decay_every=3)
    _, recs, _ = orc.als_optimize(x, init, cfg)
    assert [r["lambda"] for r in recs] == pytest.approx(
        [0.01, 0.01, 0.01, 0.005, 0.005, 0.005, 0.0025])


def test_als_rank1_converges(orc):
    # test_als.cpp:110-125
    conv = 0
    for seed in range(10):
        t = orc.random_model([3, 3, 3], 1, seed, kind="gaussian")
        x = orc.reconstruct(t)
        init = orc.random_model([3, 3, 3], 1, seed + 1000, kind="gaussian")
        _, _, st = orc.als_optimize(x, init, orc.AlsConfig(max_sweeps=50, step_tol=0.0))
        conv += st == "converged_residual"
    assert conv >= 9
