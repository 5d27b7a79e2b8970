"""CPU baseline arm: the reference's ALS and GN-CG path with BLAS products.

TEST / BENCH INFRASTRUCTURE ONLY (bench.py's cpu_baseline and --impl
reference legs, tests/). The product never imports it.

The reference (Eigen 3, single-threaded: proj/src/CMakeLists.txt:14-15) cannot
be built here. oracle/cpkit_oracle.cpp restates it with
fixed-order loops for parity; those loops are far slower than Eigen. This
module restates the same algorithm with the dense products on OpenBLAS
(numpy / scipy), so the timed CPU baseline is a tuned-BLAS CPU implementation
of the reference path, at 1 thread (the reference's own setting) or on all
host cores. It follows, per call:

  als_sweep      als.cpp:22-52 (grams, Gamma^(n), tree MTTKRP, spd_solve,
                 step norm, workspace invalidation)
  mttkrp tree    mttkrp.cpp:160-189 (front/back split h = ceil(N/2); the root
                 partial of the back modes serves modes < h, the front one
                 modes >= h; cached until a contracted factor changes)
  residual       kruskal.cpp:94-118 (fast formula, clamp at 0)
  gn_step        gauss_newton.cpp:360-449 without Armijo (the default):
                 tree MTTKRPs, Gamma set, residual, gradient, cp_cg, update,
                 then the reference's third (naive) contraction for
                 residual_after (:442-444)
  cp_cg          gauss_newton.cpp:279-349 (PCG, sum-of-norms stop test, cap
                 min(sum s R, 10 R), breakdown on <W,Q> <= 0)
  hessian_matvec gauss_newton.cpp:96-136 (per (n, p) pair, as the reference)
"""
import math
import string

import numpy as np
import scipy.linalg as sla

try:
    from threadpoolctl import threadpool_limits
except ImportError:  # pragma: no cover - threadpoolctl is in the image
    threadpool_limits = None


def threads(n):
    """Context manager limiting the BLAS threads to n."""
    if threadpool_limits is None:
        import contextlib
        return contextlib.nullcontext()
    return threadpool_limits(limits=int(n), user_api="blas")


def gram(a):  # matrix_ops.cpp:30-34
    s = a.T @ a
    return 0.5 * (s + s.T)


def krp(factors):
    """Khatri-Rao product, first factor's index slowest (row-major over modes)."""
    k = factors[0]
    for a in factors[1:]:
        k = (k[:, None, :] * a[None, :, :]).reshape(-1, a.shape[1])
    return k


def _reduce_kept(p, dims, keep, factors):
    """Root partial over kept modes (dims, last axis R) -> M^(keep): every other
    kept mode contracted against its factor (mttkrp.cpp:63-75)."""
    R = p.shape[-1]
    if len(dims) == 1:
        return p.reshape(dims[0], R)
    letters = string.ascii_lowercase
    idx = letters[:len(dims)]
    ops = [p.reshape(*dims, R)]
    subs = [idx + "z"]
    for j in range(len(dims)):
        if j != keep:
            ops.append(factors[j])
            subs.append(idx[j] + "z")
    return np.einsum(",".join(subs) + "->" + idx[keep] + "z", *ops, optimize=True)


class Tree:
    """MttkrpWorkspace (mttkrp.hpp:35-54): the two root partials, cached."""

    def __init__(self, x):
        self.x = x
        self.N = x.ndim
        self.h = (self.N + 1) // 2
        self.F = int(np.prod(x.shape[:self.h]))
        self.B = int(np.prod(x.shape[self.h:]))
        self.pf = None  # back modes contracted: F x R
        self.pb = None  # front modes contracted: B x R
        self.contractions = 0

    def note_factor_update(self, n):  # mttkrp.cpp:136-145
        if n >= self.h:
            self.pf = None
        else:
            self.pb = None

    def mttkrp(self, factors, n):
        xm = self.x.reshape(self.F, self.B)
        if n < self.h:
            if self.pf is None:
                self.pf = xm @ krp(factors[self.h:])
                self.contractions += 1
            return _reduce_kept(self.pf, self.x.shape[:self.h], n, factors[:self.h])
        if self.pb is None:
            self.pb = xm.T @ krp(factors[:self.h])
            self.contractions += 1
        return _reduce_kept(self.pb, self.x.shape[self.h:], n - self.h, factors[self.h:])


def _factor_shifted(s, lam):  # matrix_ops.cpp:41-56
    shifted = s + lam * np.eye(s.shape[0])
    try:
        return sla.cho_factor(shifted, lower=True, check_finite=False)
    except np.linalg.LinAlgError:
        shifted = shifted + (1e-12 * np.trace(s) / s.shape[0]) * np.eye(s.shape[0])
        return sla.cho_factor(shifted, lower=True, check_finite=False)


def spd_solve(s, b, lam):  # matrix_ops.cpp:60-70: Y (S + lam I) = B
    return sla.cho_solve(_factor_shifted(s, lam), b.T, check_finite=False).T


def spd_inverse(s, lam):  # matrix_ops.cpp:72-81
    inv = sla.cho_solve(_factor_shifted(s, lam), np.eye(s.shape[0]), check_finite=False)
    return 0.5 * (inv + inv.T)


def residual_fitness(factors, m_last, xnorm2):  # kruskal.cpp:94-118
    cross = float(np.sum(m_last * factors[-1]))
    g = np.ones((factors[0].shape[1],) * 2)
    for a in factors:
        g = g * gram(a)
    res2 = max(0.0, xnorm2 - 2.0 * cross + float(g.sum()))
    r = math.sqrt(res2 / xnorm2)
    return r, 1.0 - r


def als_sweep(tree, factors, lam):  # als.cpp:22-52
    N = len(factors)
    factors = [a.copy() for a in factors]
    grams = [gram(a) for a in factors]
    step = 0.0
    tree.contractions = 0
    m_last = None
    R = factors[0].shape[1]
    for n in range(N):
        gamma = np.ones((R, R))
        for m in range(N):
            if m != n:
                gamma = gamma * grams[m]
        m_n = tree.mttkrp(factors, n)
        a_new = spd_solve(gamma, m_n, lam)
        step += float(np.linalg.norm(a_new - factors[n]))
        factors[n] = a_new
        tree.note_factor_update(n)
        grams[n] = gram(a_new)
        if n == N - 1:
            m_last = m_n
    return factors, step, tree.contractions, m_last


# ---- GN (gauss_newton.cpp) -------------------------------------------------------------
def gamma_set(factors):  # kruskal.cpp:42-65
    N = len(factors)
    R = factors[0].shape[1]
    grams = [gram(a) for a in factors]
    pair = [[None] * N for _ in range(N)]
    for n in range(N):
        for p in range(n, N):
            g = np.ones((R, R))
            for m in range(N):
                if m != n and m != p:
                    g = g * grams[m]
            pair[n][p] = pair[p][n] = g
    return pair


def hessian_matvec(factors, pair, w, lam):  # gauss_newton.cpp:96-136 (identity shape)
    N = len(factors)
    u = []
    for n in range(N):
        un = lam * w[n] + w[n] @ pair[n][n]
        for p in range(N):
            if p != n:
                b = factors[p].T @ w[p]
                un = un + factors[n] @ (pair[n][p] * b).T
        u.append(un)
    return u


def cp_cg(factors, pair, g, lam, cg_tol=1e-3, cap=None):  # gauss_newton.cpp:279-349
    N = len(factors)
    R = factors[0].shape[1]
    if cap is None:
        cap = min(sum(a.shape[0] for a in factors) * R, 10 * R)
    v = [np.zeros_like(gn) for gn in g]
    gnorm = sum(float(np.linalg.norm(gn)) for gn in g)
    if gnorm == 0.0:
        return v, 0, False, False
    pinv = [spd_inverse(pair[n][n], lam) for n in range(N)]
    rres = [-gn for gn in g]
    z = [rres[n] @ pinv[n] for n in range(N)]
    w = [zn.copy() for zn in z]
    rz = sum(float(np.sum(rres[n] * z[n])) for n in range(N))
    it, hit_cap, breakdown = 0, False, False
    while sum(float(np.linalg.norm(rn)) for rn in rres) > cg_tol * gnorm:
        if it >= cap:
            hit_cap = True
            break
        q = hessian_matvec(factors, pair, w, lam)
        wq = sum(float(np.sum(w[n] * q[n])) for n in range(N))
        if not wq > 0.0:
            breakdown = True
            break
        alpha = rz / wq
        for n in range(N):
            v[n] = v[n] + alpha * w[n]
            rres[n] = rres[n] - alpha * q[n]
            z[n] = rres[n] @ pinv[n]
        rz_new = sum(float(np.sum(rres[n] * z[n])) for n in range(N))
        beta = rz_new / rz
        for n in range(N):
            w[n] = z[n] + beta * w[n]
        rz = rz_new
        it += 1
    return v, it, hit_cap, breakdown


def gn_step(x, factors, lam, xnorm2, tree=None, residual_tol=5e-5):
    """One default GN step (gauss_newton.cpp:360-449, no Armijo) at lambda."""
    if tree is None:
        tree = Tree(x)
    N = len(factors)
    m = [tree.mttkrp(factors, n) for n in range(N)]
    pair = gamma_set(factors)
    res, _ = residual_fitness(factors, m[-1], xnorm2)
    diag = {"residual_before": res, "residual_after": res, "stepped": False, "cg_iters": 0}
    if res < residual_tol:
        return factors, diag
    g = [factors[n] @ pair[n][n] - m[n] for n in range(N)]
    v, it, cap, bd = cp_cg(factors, pair, g, lam)
    new = [factors[n] + v[n] for n in range(N)]
    for n in range(N):
        tree.note_factor_update(n)
    # the reference's residual_after: a naive (uncached) last-mode MTTKRP (:442-444)
    naive = Tree(x)
    r_after, _ = residual_fitness(new, naive.mttkrp(new, N - 1), xnorm2)
    diag.update(residual_after=r_after, stepped=True, cg_iters=it, cg_hit_cap=cap, cg_breakdown=bd,
                step_norm=sum(float(np.linalg.norm(vn)) for vn in v))
    return new, diag


def schedule_next(lam, direction, mu=2.0, lower=1e-6, upper=1e-2):  # gauss_newton.cpp:47-59
    if direction == 0:
        lam /= mu
        if lam < lower:
            direction = 1
    else:
        lam *= mu
        if lam > upper:
            direction = 0
    return lam, direction


def als_optimize(x, factors, max_sweeps=10000, residual_tol=5e-5, step_tol=1e-7, lambda0=0.0,
                 decay_factor=2.0, decay_every=None):  # als.cpp:54-94
    """Outer ALS loop: lambda_k = lambda0 / decay^floor((k-1)/every), a record
    per sweep from the residual of the sweep's own last-mode MTTKRP, stop on
    residual_tol (converged_residual) or step_tol (converged_step), else cap_hit."""
    xnorm2 = float(np.dot(x.ravel(), x.ravel()))
    if not xnorm2 > 0.0:
        raise ValueError("als_optimize: tensor norm must be positive")
    tree = Tree(x)
    records, status = [], "cap_hit"
    for sweep in range(1, max_sweeps + 1):
        lam = lambda0 / decay_factor ** ((sweep - 1) // decay_every) if decay_every else lambda0
        factors, step, _, m_last = als_sweep(tree, factors, lam)
        r, f = residual_fitness(factors, m_last, xnorm2)
        records.append({"iter": sweep, "residual": r, "fitness": f, "lambda": lam, "cg_iters": 0})
        if r < residual_tol:
            status = "converged_residual"
            break
        if step < step_tol:
            status = "converged_step"
            break
    return factors, records, status


def gn_optimize(x, factors, max_iters=500, residual_tol=5e-5, step_tol=1e-7, upper=1e-2, lower=1e-6, mu=2.0):
    """Outer GN loop with the default varying schedule (gauss_newton.cpp:451-494,
    :10-59): lambda starts at `upper`, a record per stepped iteration
    {iter, residual_after, 1 - r, lambda, cg_iters}, stop on residual_tol
    (converged_residual) or step_tol (converged_step), else cap_hit."""
    xnorm2 = float(np.dot(x.ravel(), x.ravel()))
    if not xnorm2 > 0.0:
        raise ValueError("gn_optimize: tensor norm must be positive")
    tree = Tree(x)
    lam, direction = upper, 0
    records, status = [], "cap_hit"
    for it in range(1, max_iters + 1):
        factors, d = gn_step(x, factors, lam, xnorm2, tree, residual_tol)
        if not d["stepped"]:
            status = "converged_residual"
            break
        r = d["residual_after"]
        records.append({"iter": it, "residual": r, "fitness": 1.0 - r, "lambda": lam, "cg_iters": d["cg_iters"]})
        if r < residual_tol:
            status = "converged_residual"
            break
        if d["step_norm"] < step_tol:
            status = "converged_step"
            break
        lam, direction = schedule_next(lam, direction, mu, lower, upper)
    return factors, records, status
