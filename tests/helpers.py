"""Shared seeded-input helpers for the parity tests.

Random draws use the reference's keyed SplitMix RNG (rng.hpp:11-46) through the
oracle, so every test input is a pure function of (seed, stream, index).
"""
import numpy as np


def gauss_matrix(orc, rows, cols, seed, stream=0x7E57):
    return np.array([[orc.gaussian(seed, stream, i * cols + j) for j in range(cols)]
                     for i in range(rows)], dtype=np.float64).reshape(rows, cols)


def gauss_factors(orc, dims, rank, seed):
    return orc.random_model(dims, rank, seed, kind="gaussian")


def gauss_tensor(orc, dims, seed):
    """selftest.cpp:16-23 random_dense_tensor: gaussian(seed, 0xDD, flat)."""
    n = int(np.prod(dims))
    return np.array([orc.gaussian(seed, 0xDD, f) for f in range(n)]).reshape(dims)


def rel_err(got, exp):
    """Frobenius-relative error (test_tensor_core.cpp:30-32)."""
    got = np.asarray(got)
    exp = np.asarray(exp)
    return float(np.linalg.norm((got - exp).ravel()) / np.linalg.norm(exp.ravel()))


def vec_rel_err(got, exp):
    num = sum(float(np.sum((np.asarray(g) - np.asarray(e)) ** 2)) for g, e in zip(got, exp))
    den = sum(float(np.sum(np.asarray(e) ** 2)) for e in exp)
    return (num / den) ** 0.5


def khatri_rao(a, b):
    """matrix_ops.cpp:9-21: column k = kron(a_k, b_k)."""
    return np.einsum("ir,jr->ijr", a, b).reshape(a.shape[0] * b.shape[0], a.shape[1])


def matricize(x, mode):
    """tensor.cpp:111-132: rows i_mode, remaining modes ascending, last fastest."""
    return np.moveaxis(x, mode, 0).reshape(x.shape[mode], -1)


def mttkrp_unfold(x, factors, mode):
    kr = np.ones((1, factors[0].shape[1]))
    for m, f in enumerate(factors):
        if m != mode:
            kr = khatri_rao(kr, f)
    return matricize(x, mode) @ kr


def swamp_factors(orc, dims, rank, seed, c=0.9):
    """BASELINE config 3 ("swamp"): column r of mode n is sqrt(c) u_n + sqrt(1-c) v_{n,r},
    normalised; u, v ~ N(0,1) from the keyed RNG on streams 0x5701+n / 0x5801+n."""
    out = []
    for n, s in enumerate(dims):
        u = np.array([orc.gaussian(seed, 0x5701 + n, i) for i in range(s)])
        a = np.empty((s, rank))
        for r in range(rank):
            v = np.array([orc.gaussian(seed, 0x5801 + n, r * s + i) for i in range(s)])
            col = np.sqrt(c) * u + np.sqrt(1 - c) * v
            a[:, r] = col / np.linalg.norm(col)
        out.append(a)
    return out
