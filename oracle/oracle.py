"""ctypes front end for the CPU oracle (oracle/cpkit_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py. The product package
(paper_1910_12331_b200) never imports this module.

Factor sets are lists of float64 numpy arrays of shape (s_n, R), row-major,
exactly the reference's Matrix layout (matrix_ops.hpp:9-10).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libcpkit_oracle.so")

_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class GnConfig(C.Structure):
    """Flat mirror of GnConfig (gauss_newton.hpp:50-62); defaults per :53-59."""

    _fields_ = [
        ("grad_tol", C.c_double), ("residual_tol", C.c_double), ("step_tol", C.c_double),
        ("max_iters", C.c_int), ("cg_tol", C.c_double), ("cg_max_iters", C.c_int),
        ("reg_mode", C.c_int), ("reg_shape", C.c_int),
        ("lambda_", C.c_double), ("mu", C.c_double), ("lower", C.c_double), ("upper", C.c_double),
        ("armijo", C.c_int), ("c1", C.c_double), ("shrink", C.c_double),
        ("max_backtracks", C.c_int), ("cg_beta", C.c_int),
    ]

    def __init__(self, **kw):
        d = dict(grad_tol=0.0, residual_tol=5e-5, step_tol=1e-7, max_iters=500, cg_tol=1e-3,
                 cg_max_iters=0, reg_mode=1, reg_shape=0, lambda_=1e-2, mu=2.0, lower=1e-6,
                 upper=1e-2, armijo=0, c1=1e-4, shrink=0.5, max_backtracks=20, cg_beta=0)
        d.update(kw)
        super().__init__(**d)


class AlsConfig(C.Structure):
    """Flat mirror of AlsConfig (als.hpp:11-22); decay_every 0 = unset."""

    _fields_ = [("max_sweeps", C.c_int), ("residual_tol", C.c_double), ("step_tol", C.c_double),
                ("lambda0", C.c_double), ("decay_factor", C.c_double), ("decay_every", C.c_int)]

    def __init__(self, **kw):
        d = dict(max_sweeps=10000, residual_tol=5e-5, step_tol=1e-7, lambda0=0.0,
                 decay_factor=2.0, decay_every=0)
        d.update(kw)
        super().__init__(**d)


class Record(C.Structure):
    _fields_ = [("iteration", C.c_int), ("residual", C.c_double), ("fitness", C.c_double),
                ("lambda_", C.c_double), ("cg_iters", C.c_int), ("seconds", C.c_double)]


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build() -> str:
    """Compile the oracle with its committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        for name in ("orc_mix64",):
            getattr(L, name).restype = C.c_uint64
            getattr(L, name).argtypes = [C.c_uint64]
        L.orc_keyed.restype = C.c_uint64
        L.orc_keyed.argtypes = [C.c_uint64] * 4
        L.orc_uniform.restype = C.c_double
        L.orc_uniform.argtypes = [C.c_uint64] * 3 + [C.c_double] * 2
        L.orc_gaussian.restype = C.c_double
        L.orc_gaussian.argtypes = [C.c_uint64] * 3
        L.orc_problem_seed.restype = C.c_uint64
        L.orc_problem_seed.argtypes = [C.c_uint64, C.c_int, C.c_int]
        L.orc_init_seed.restype = C.c_uint64
        L.orc_init_seed.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int]
        L.orc_norm2.restype = C.c_double
        L.orc_norm2.argtypes = [_u64p, C.c_int, _dp]
        L.orc_noise_gaussian.restype = C.c_double
        L.orc_noise_gaussian.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_add_noise.argtypes = [_u64p, C.c_int, _dp, C.c_uint64, C.c_double, _dp]
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def _chk(rc: int) -> None:
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def _dims(dims: Sequence[int]):
    a = (C.c_uint64 * len(dims))(*[int(d) for d in dims])
    return a


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _cat(blocks: Sequence[np.ndarray]) -> np.ndarray:
    return np.ascontiguousarray(np.concatenate([np.ascontiguousarray(b, dtype=np.float64).ravel()
                                                for b in blocks]))


def _split(buf: np.ndarray, rows: Sequence[int], rank: int) -> List[np.ndarray]:
    out, at = [], 0
    for s in rows:
        out.append(buf[at:at + s * rank].reshape(s, rank).copy())
        at += s * rank
    return out


def _tensor(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


# ---- rng (rng.hpp:11-46) and seeds (harness.cpp:378-391)
def mix64(x: int) -> int:
    return lib().orc_mix64(x)


def keyed(seed, stream, index, salt) -> int:
    return lib().orc_keyed(seed, stream, index, salt)


def uniform(seed, stream, index, a=0.0, b=1.0) -> float:
    return lib().orc_uniform(seed, stream, index, a, b)


def gaussian(seed, stream, index) -> float:
    return lib().orc_gaussian(seed, stream, index)


def noise_gaussian(seed: int, gidx: int) -> float:
    """The keyed noise draw (stream 0x4E01, portable log/cos) at global flat index gidx."""
    return lib().orc_noise_gaussian(seed, gidx)


def add_noise(x: np.ndarray, seed: int, rel: float):
    """x += scale * E in place (C-contiguous float64 tensor); returns (scale, ||X||^2, ||E||^2)."""
    if not (x.dtype == np.float64 and x.flags.c_contiguous):
        raise ValueError("add_noise: need a C-contiguous float64 tensor")
    out = np.empty(3)
    _chk(lib().orc_add_noise(_dims(x.shape), x.ndim, _dptr(x), seed, rel, _dptr(out)))
    return float(out[0]), float(out[1]), float(out[2])


def problem_seed(master: int, rank: int, problem: int) -> int:
    return lib().orc_problem_seed(master, rank, problem)


def init_seed(master: int, rank: int, problem: int, init: int) -> int:
    return lib().orc_init_seed(master, rank, problem, init)


def random_model(dims, rank, seed, kind="uniform", a=0.0, b=1.0) -> List[np.ndarray]:
    """generators.cpp:59-76: entry (i,r) of mode n = draw(seed, n, i*R+r)."""
    n = sum(int(d) for d in dims) * rank
    out = np.empty(n, dtype=np.float64)
    _chk(lib().orc_random_model(_dims(dims), len(dims), C.c_int64(rank), C.c_uint64(seed),
                                0 if kind == "uniform" else 1, C.c_double(a), C.c_double(b),
                                _dptr(out)))
    return _split(out, dims, rank)


def reconstruct(factors: Sequence[np.ndarray]) -> np.ndarray:
    """kruskal.cpp:67-92 per-entry order (sum over r of the mode-ordered product)."""
    dims = [f.shape[0] for f in factors]
    rank = factors[0].shape[1]
    out = np.empty(int(np.prod(dims)), dtype=np.float64)
    _chk(lib().orc_reconstruct(_dims(dims), len(dims), C.c_int64(rank), _dptr(_cat(factors)),
                               _dptr(out)))
    return out.reshape(dims)


def norm2(x: np.ndarray) -> float:
    x = _tensor(x)
    return lib().orc_norm2(_dims(x.shape), x.ndim, _dptr(x))


def mttkrp_naive(x: np.ndarray, factors, mode: int) -> np.ndarray:
    x = _tensor(x)
    rank = factors[0].shape[1]
    out = np.empty((x.shape[mode] if 0 <= mode < x.ndim else 1, rank), dtype=np.float64)
    _chk(lib().orc_mttkrp_naive(_dims(x.shape), x.ndim, _dptr(x), C.c_int64(rank),
                                _dptr(_cat(factors)), mode, _dptr(out)))
    return out


def mttkrp_tree_all(x: np.ndarray, factors):
    """All modes through one MttkrpWorkspace; returns (list of M^(n), contractions)."""
    x = _tensor(x)
    rank = factors[0].shape[1]
    out = np.empty(sum(x.shape) * rank, dtype=np.float64)
    cnt = C.c_int(0)
    _chk(lib().orc_mttkrp_tree_all(_dims(x.shape), x.ndim, _dptr(x), C.c_int64(rank),
                                   _dptr(_cat(factors)), _dptr(out), C.byref(cnt)))
    return _split(out, x.shape, rank), cnt.value


def gram(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = np.empty((a.shape[1], a.shape[1]))
    _chk(lib().orc_gram(_dptr(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]), _dptr(out)))
    return out


def gamma_set(factors):
    """kruskal.cpp:42-65 -> (grams[N,R,R], pairwise[N,N,R,R])."""
    dims = [f.shape[0] for f in factors]
    n, rank = len(dims), factors[0].shape[1]
    grams = np.empty((n, rank, rank))
    pair = np.empty((n, n, rank, rank))
    _chk(lib().orc_gamma_set(_dims(dims), n, C.c_int64(rank), _dptr(_cat(factors)), _dptr(grams),
                             _dptr(pair)))
    return grams, pair


def residual(x: np.ndarray, factors, xnorm2: float, last_mttkrp: Optional[np.ndarray] = None):
    x = _tensor(x)
    rank = factors[0].shape[1]
    r, f = C.c_double(), C.c_double()
    lm = None if last_mttkrp is None else np.ascontiguousarray(last_mttkrp, dtype=np.float64)
    _chk(lib().orc_residual(_dims(x.shape), x.ndim, _dptr(x), C.c_int64(rank), _dptr(_cat(factors)),
                            C.c_double(xnorm2), None if lm is None else _dptr(lm), C.byref(r),
                            C.byref(f)))
    return r.value, f.value


def gradient(factors, mttkrps, grams, pair):
    dims = [f.shape[0] for f in factors]
    rank = factors[0].shape[1]
    out = np.empty(sum(dims) * rank)
    _chk(lib().orc_gradient(_dims(dims), len(dims), C.c_int64(rank), _dptr(_cat(factors)),
                            _dptr(_cat(mttkrps)), _dptr(np.ascontiguousarray(grams)),
                            _dptr(np.ascontiguousarray(pair)), _dptr(out)))
    return _split(out, dims, rank)


def hessian_matvec(factors, grams, pair, w, lam: float, shape: int = 0):
    dims = [f.shape[0] for f in factors]
    rank = factors[0].shape[1]
    out = np.empty(sum(dims) * rank)
    _chk(lib().orc_hessian_matvec(_dims(dims), len(dims), C.c_int64(rank), _dptr(_cat(factors)),
                                  _dptr(np.ascontiguousarray(grams)),
                                  _dptr(np.ascontiguousarray(pair)), _dptr(_cat(w)),
                                  C.c_double(lam), shape, _dptr(out)))
    return _split(out, dims, rank)


def explicit_jtj(factors, var_cap: int = 2000) -> np.ndarray:
    dims = [f.shape[0] for f in factors]
    rank = factors[0].shape[1]
    nv = sum(dims) * rank
    out = np.empty((nv, nv))
    _chk(lib().orc_explicit_jtj(_dims(dims), len(dims), C.c_int64(rank), _dptr(_cat(factors)),
                                C.c_uint64(var_cap), _dptr(out)))
    return out


def vec_stack(ms) -> np.ndarray:
    """gauss_newton.cpp:209-222: mode-major, column-major within each factor."""
    return np.concatenate([np.asarray(m).T.ravel() for m in ms])


def preconditioner(grams, pair, lam: float, shape: int = 0):
    n, rank = grams.shape[0], grams.shape[1]
    out = np.empty((n, rank, rank))
    _chk(lib().orc_preconditioner(n, C.c_int64(rank), _dptr(np.ascontiguousarray(grams)),
                                  _dptr(np.ascontiguousarray(pair)), C.c_double(lam), shape,
                                  _dptr(out)))
    return out


def spd_solve(s: np.ndarray, b: np.ndarray, lam: float) -> np.ndarray:
    s = np.ascontiguousarray(s, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.empty_like(b)
    _chk(lib().orc_spd_solve(_dptr(s), C.c_int64(s.shape[0]), _dptr(b), C.c_int64(b.shape[0]),
                             C.c_double(lam), _dptr(out)))
    return out


def spd_inverse(s: np.ndarray, lam: float) -> np.ndarray:
    s = np.ascontiguousarray(s, dtype=np.float64)
    out = np.empty_like(s)
    _chk(lib().orc_spd_inverse(_dptr(s), C.c_int64(s.shape[0]), C.c_double(lam), _dptr(out)))
    return out


def cp_cg(factors, grams, pair, g, lam: float, cfg: GnConfig):
    dims = [f.shape[0] for f in factors]
    rank = factors[0].shape[1]
    out = np.empty(sum(dims) * rank)
    it, cap, bd = C.c_int(), C.c_int(), C.c_int()
    _chk(lib().orc_cp_cg(_dims(dims), len(dims), C.c_int64(rank), _dptr(_cat(factors)),
                         _dptr(np.ascontiguousarray(grams)), _dptr(np.ascontiguousarray(pair)),
                         _dptr(_cat(g)), C.c_double(lam), C.byref(cfg), _dptr(out), C.byref(it),
                         C.byref(cap), C.byref(bd)))
    return _split(out, dims, rank), it.value, bool(cap.value), bool(bd.value)


GN_DIAG_FIELDS = ("halt", "stepped", "residual_before", "residual_after", "grad_norm", "lambda",
                  "cg_iters", "step_norm", "alpha", "armijo_exhausted", "cg_hit_cap",
                  "cg_breakdown")


def gn_step(x: np.ndarray, factors, cfg: GnConfig, xnorm2: float):
    x = _tensor(x)
    rank = factors[0].shape[1]
    buf = _cat(factors)
    diag = np.empty(12)
    _chk(lib().orc_gn_step(_dims(x.shape), x.ndim, _dptr(x), C.c_int64(rank), _dptr(buf),
                           C.byref(cfg), C.c_double(xnorm2), _dptr(diag)))
    return _split(buf, x.shape, rank), dict(zip(GN_DIAG_FIELDS, diag.tolist()))


STATUS = ("converged_residual", "converged_step", "cap_hit", "numerical_failure")


def _records(recs, n):
    return [dict(iter=recs[i].iteration, residual=recs[i].residual, fitness=recs[i].fitness,
                 **{"lambda": recs[i].lambda_}, cg_iters=recs[i].cg_iters,
                 seconds=recs[i].seconds) for i in range(n)]


def gn_optimize(x: np.ndarray, factors, cfg: GnConfig):
    x = _tensor(x)
    rank = factors[0].shape[1]
    buf = _cat(factors)
    recs = (Record * max(1, cfg.max_iters))()
    n, st = C.c_int(), C.c_int()
    _chk(lib().orc_gn_optimize(_dims(x.shape), x.ndim, _dptr(x), C.c_int64(rank), _dptr(buf),
                               C.byref(cfg), recs, C.byref(n), C.byref(st)))
    return _split(buf, x.shape, rank), _records(recs, n.value), STATUS[st.value]


def als_sweep(x: np.ndarray, factors, lam: float):
    x = _tensor(x)
    rank = factors[0].shape[1]
    buf = _cat(factors)
    sn, cnt = C.c_double(), C.c_int()
    last = np.empty((x.shape[-1], rank))
    _chk(lib().orc_als_sweep(_dims(x.shape), x.ndim, _dptr(x), C.c_int64(rank), _dptr(buf),
                             C.c_double(lam), C.byref(sn), C.byref(cnt), _dptr(last)))
    return _split(buf, x.shape, rank), sn.value, cnt.value, last


def als_optimize(x: np.ndarray, factors, cfg: AlsConfig):
    x = _tensor(x)
    rank = factors[0].shape[1]
    buf = _cat(factors)
    recs = (Record * max(1, cfg.max_sweeps))()
    n, st = C.c_int(), C.c_int()
    _chk(lib().orc_als_optimize(_dims(x.shape), x.ndim, _dptr(x), C.c_int64(rank), _dptr(buf),
                                C.byref(cfg), recs, C.byref(n), C.byref(st)))
    return _split(buf, x.shape, rank), _records(recs, n.value), STATUS[st.value]


def schedule_next(mode: int, lam: float, mu: float, lower: float, upper: float, direction: int):
    l, d = C.c_double(lam), C.c_int(direction)
    lib().orc_schedule_next(mode, C.byref(l), C.c_double(mu), C.c_double(lower),
                            C.c_double(upper), C.byref(d))
    return l.value, d.value
