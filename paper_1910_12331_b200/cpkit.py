"""Python host mirror of the cpkit C ABI (include/cpkit.h, include/cpkit_dev.h).

The product is libcpkit_b200.so (sm_100a kernels + C++ drivers). This module
only binds it with ctypes so tests and the bench call the same entry points a
C caller would (the reference's own CLI links only its C ABI,
proj/tools/CMakeLists.txt:1-5). There is no fallback: if the library is
missing, every call raises.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libcpkit_b200.so")

STATUS_NAMES = ("ok", "invalid_argument", "parse_error", "io_error", "singular_system",
                "numerical_failure", "limit_exceeded", "internal_error")

# Every exported symbol of include/cpkit.h and include/cpkit_dev.h.
CPKIT_SYMBOLS = (
    "cpkit_version", "cpkit_status_name", "cpkit_last_error", "cpkit_string_free",
    "cpkit_tensor_create", "cpkit_tensor_load", "cpkit_tensor_save", "cpkit_tensor_order",
    "cpkit_tensor_extent", "cpkit_tensor_element_count", "cpkit_tensor_data",
    "cpkit_tensor_destroy", "cpkit_model_load", "cpkit_model_save", "cpkit_model_order",
    "cpkit_model_rank", "cpkit_model_extent", "cpkit_model_factor", "cpkit_model_reconstruct",
    "cpkit_model_destroy", "cpkit_generate_low_rank", "cpkit_matmul_tensor", "cpkit_decompose",
    "cpkit_run_trace", "cpkit_run_likelihood", "cpkit_run_matmul", "cpkit_run_bench_matvec",
    "cpkit_run_selftest_oracle", "cpkit_report_emit", "cpkit_report_to_json",
    "cpkit_report_config", "cpkit_report_ok", "cpkit_report_destroy",
)
CPKIT_DEV_SYMBOLS = (
    "cpkit_dev_problem_create", "cpkit_dev_nccl_unique_id", "cpkit_dev_problem_create_sharded",
    "cpkit_dev_problem_destroy", "cpkit_dev_slab", "cpkit_dev_upload_tensor",
    "cpkit_dev_generate_tensor", "cpkit_dev_set_factors", "cpkit_dev_get_factors",
    "cpkit_dev_norm2", "cpkit_dev_mttkrp", "cpkit_dev_mttkrp_naive",
    "cpkit_dev_note_factor_update", "cpkit_dev_full_contractions",
    "cpkit_dev_reset_contraction_counter", "cpkit_dev_gamma_set", "cpkit_dev_set_gamma_set",
    "cpkit_dev_residual", "cpkit_dev_gradient", "cpkit_dev_jtj_matvec",
    "cpkit_dev_preconditioner", "cpkit_dev_cp_cg", "cpkit_dev_spd_solve",
    "cpkit_dev_spd_inverse", "cpkit_dev_als_sweep", "cpkit_dev_gn_step", "cpkit_dev_optimize",
    "cpkit_dev_time_als_sweeps", "cpkit_dev_time_roots", "cpkit_dev_profile",
    "cpkit_dev_profile_read", "cpkit_dev_time_jtj",
    "cpkit_dev_time_norm2", "cpkit_dev_time_second_level", "cpkit_dev_probe_dmma_peak", "cpkit_dev_kernel_launches",
    "cpkit_dev_guard_violations", "cpkit_dev_guard_selftest",
    "cpkit_dev_time_gn_steps", "cpkit_dev_random_factors", "cpkit_dev_problem_seed",
    "cpkit_dev_init_seed", "cpkit_dev_download_tensor", "cpkit_dev_shard_range",
    "cpkit_dev_problem_create_loopback", "cpkit_dev_load_tensor",
)


class CpkitError(RuntimeError):
    def __init__(self, code: int, message: str):
        name = STATUS_NAMES[code] if 0 <= code < len(STATUS_NAMES) else str(code)
        super().__init__(f"{name}: {message}")
        self.code = code
        self.status = name


_lib = None
_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_u64 = C.c_uint64


def load():
    """Load libcpkit_b200.so (built by __graft_entry__.build()); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.cpkit_version.restype = C.c_char_p
    L.cpkit_status_name.restype = C.c_char_p
    L.cpkit_last_error.restype = C.c_char_p
    L.cpkit_tensor_data.restype = _dp
    L.cpkit_tensor_data.argtypes = [_vp]
    for f in ("cpkit_tensor_order", "cpkit_tensor_element_count", "cpkit_model_order",
              "cpkit_model_rank"):
        getattr(L, f).restype = _u64
        getattr(L, f).argtypes = [_vp]
    for f in ("cpkit_tensor_extent", "cpkit_model_extent"):
        getattr(L, f).restype = _u64
        getattr(L, f).argtypes = [_vp, _u64]
    L.cpkit_model_factor.restype = _dp
    L.cpkit_model_factor.argtypes = [_vp, _u64]
    for f in ("cpkit_tensor_destroy", "cpkit_model_destroy", "cpkit_report_destroy",
              "cpkit_dev_problem_destroy", "cpkit_string_free"):
        getattr(L, f).argtypes = [_vp]
        getattr(L, f).restype = None
    L.cpkit_dev_full_contractions.argtypes = [_vp]
    L.cpkit_dev_reset_contraction_counter.argtypes = [_vp]
    L.cpkit_dev_reset_contraction_counter.restype = None
    L.cpkit_dev_kernel_launches.restype = _u64
    L.cpkit_dev_guard_violations.restype = _u64
    L.cpkit_report_ok.argtypes = [_vp]
    L.cpkit_dev_problem_seed.restype = _u64
    L.cpkit_dev_problem_seed.argtypes = [_u64, C.c_int, C.c_int]
    L.cpkit_dev_init_seed.restype = _u64
    L.cpkit_dev_init_seed.argtypes = [_u64, C.c_int, C.c_int, C.c_int]
    _lib = L
    return L


def _chk(rc: int) -> None:
    if rc != 0:
        raise CpkitError(rc, load().cpkit_last_error().decode())


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _dims(dims):
    return (C.c_uint64 * len(dims))(*[int(d) for d in dims])


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_dp)


def stack(blocks: Sequence[np.ndarray]) -> np.ndarray:
    """Stacked factor layout of cpkit_dev.h: mode-major row-major blocks."""
    return np.ascontiguousarray(np.concatenate([_f64(b).ravel() for b in blocks]))


def unstack(buf: np.ndarray, dims: Sequence[int], rank: int) -> List[np.ndarray]:
    out, at = [], 0
    for s in dims:
        out.append(buf[at:at + s * rank].reshape(s, rank).copy())
        at += s * rank
    return out


def version() -> str:
    return load().cpkit_version().decode()


def status_name(code: int) -> str:
    return load().cpkit_status_name(code).decode()


# ------------------------------------------------------------------ cpkit.h objects
class Tensor:
    """cpkit_tensor handle (host copy, row-major)."""

    def __init__(self, handle):
        self._h = handle if isinstance(handle, C.c_void_p) else _vp(handle)

    @classmethod
    def create(cls, x: np.ndarray) -> "Tensor":
        x = _f64(x)
        h = _vp()
        _chk(load().cpkit_tensor_create(_dims(x.shape), _u64(x.ndim), _ptr(x), C.byref(h)))
        return cls(h)

    @classmethod
    def load_file(cls, path: str) -> "Tensor":
        h = _vp()
        _chk(load().cpkit_tensor_load(path.encode(), C.byref(h)))
        return cls(h)

    def save(self, path: str) -> None:
        _chk(load().cpkit_tensor_save(self._h, path.encode()))

    @property
    def shape(self):
        L = load()
        return tuple(L.cpkit_tensor_extent(self._h, m) for m in range(L.cpkit_tensor_order(self._h)))

    def numpy(self) -> np.ndarray:
        L = load()
        n = L.cpkit_tensor_element_count(self._h)
        p = L.cpkit_tensor_data(self._h)
        return np.ctypeslib.as_array(p, shape=(n,)).reshape(self.shape).copy()

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cpkit_tensor_destroy(self._h)
            self._h = None


class Model:
    """cpkit_model handle."""

    def __init__(self, handle):
        self._h = handle if isinstance(handle, C.c_void_p) else _vp(handle)

    @classmethod
    def load_file(cls, path: str) -> "Model":
        h = _vp()
        _chk(load().cpkit_model_load(path.encode(), C.byref(h)))
        return cls(h)

    def save(self, path: str) -> None:
        _chk(load().cpkit_model_save(self._h, path.encode()))

    @property
    def rank(self) -> int:
        return load().cpkit_model_rank(self._h)

    @property
    def dims(self):
        L = load()
        return tuple(L.cpkit_model_extent(self._h, m) for m in range(L.cpkit_model_order(self._h)))

    def factors(self) -> List[np.ndarray]:
        L = load()
        out = []
        for m, s in enumerate(self.dims):
            p = L.cpkit_model_factor(self._h, m)
            out.append(np.ctypeslib.as_array(p, shape=(s * self.rank,)).reshape(s, self.rank).copy())
        return out

    def reconstruct(self) -> Tensor:
        h = _vp()
        _chk(load().cpkit_model_reconstruct(self._h, C.byref(h)))
        return Tensor(h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cpkit_model_destroy(self._h)
            self._h = None


class Report:
    def __init__(self, handle):
        self._h = handle if isinstance(handle, C.c_void_p) else _vp(handle)

    def to_json(self) -> dict:
        return json.loads(self.to_json_text())

    def to_json_text(self) -> str:
        s = C.c_char_p()
        _chk(load().cpkit_report_to_json(self._h, C.byref(s)))
        try:
            return s.value.decode()
        finally:
            load().cpkit_string_free(C.cast(s, _vp))

    def config(self) -> dict:
        s = C.c_char_p()
        _chk(load().cpkit_report_config(self._h, C.byref(s)))
        try:
            return json.loads(s.value.decode())
        finally:
            load().cpkit_string_free(C.cast(s, _vp))

    def emit(self, fmt: str, path: str) -> None:
        _chk(load().cpkit_report_emit(self._h, fmt.encode(), path.encode()))

    def ok(self) -> bool:
        return bool(load().cpkit_report_ok(self._h))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cpkit_report_destroy(self._h)
            self._h = None


def generate_low_rank(spec: dict):
    m, t = _vp(), _vp()
    _chk(load().cpkit_generate_low_rank(json.dumps(spec).encode(), C.byref(m), C.byref(t)))
    return Model(m), Tensor(t)


def matmul_tensor(n: int) -> Tensor:
    h = _vp()
    _chk(load().cpkit_matmul_tensor(_u64(n), C.byref(h)))
    return Tensor(h)


def decompose(tensor: Tensor, config: dict, init: Optional[Model] = None):
    """cpkit_decompose (reference cpkit_c.cpp:229-297): returns (Model, Report)."""
    m, r = _vp(), _vp()
    _chk(load().cpkit_decompose(tensor._h, json.dumps(config).encode(),
                                None if init is None else init._h, C.byref(m), C.byref(r)))
    return Model(m), Report(r)


def run_trace(config: dict) -> Report:
    r = _vp()
    _chk(load().cpkit_run_trace(json.dumps(config).encode(), C.byref(r)))
    return Report(r)


def run_likelihood(config: dict) -> Report:
    """harness.cpp:488-550 on the device: one CTA per (rank, problem, init) instance."""
    r = _vp()
    _chk(load().cpkit_run_likelihood(json.dumps(config).encode(), C.byref(r)))
    return Report(r)


def run_bench_matvec(config: dict) -> Report:
    """selftest.cpp:275-318: the implicit J^T J matvec timed on the device over sizes."""
    r = _vp()
    _chk(load().cpkit_run_bench_matvec(json.dumps(config).encode(), C.byref(r)))
    return Report(r)


def run_selftest_oracle(config: dict) -> Report:
    """selftest.cpp:198-271: device operators vs dense routes evaluated on the device."""
    r = _vp()
    _chk(load().cpkit_run_selftest_oracle(json.dumps(config).encode(), C.byref(r)))
    return Report(r)


def run_matmul(config: dict) -> Report:
    """harness.cpp:552-653 on the device: three arms per init, one CTA per instance."""
    r = _vp()
    _chk(load().cpkit_run_matmul(json.dumps(config).encode(), C.byref(r)))
    return Report(r)


# ------------------------------------------------------------------ cpkit_dev.h
class DeviceProblem:
    """cpkit_dev_problem: tensor slab + factors + workspace resident on one GPU."""

    def __init__(self, dims: Sequence[int], rank: int, device: int = 0, shard: int = 0,
                 world: int = 1, nccl_id: Optional[bytes] = None):
        self.dims = [int(d) for d in dims]
        self.rank = int(rank)
        h = _vp()
        L = load()
        if world == 1 and nccl_id is None:
            _chk(L.cpkit_dev_problem_create(device, _dims(self.dims), _u64(len(self.dims)),
                                            _u64(self.rank), C.byref(h)))
        else:
            buf = C.create_string_buffer(nccl_id, 128)
            _chk(L.cpkit_dev_problem_create_sharded(device, _dims(self.dims), _u64(len(self.dims)),
                                                    _u64(self.rank), shard, world, buf, C.byref(h)))
        self._h = h
        self.stacked = sum(self.dims) * self.rank

    @classmethod
    def loopback(cls, dims: Sequence[int], rank: int, world: int, device: int = 0) -> List["DeviceProblem"]:
        """TEST ONLY: `world` last-mode shards on one GPU joined by the in-process
        loopback group (cpkit_dev_problem_create_loopback). Drive each shard from
        its own thread with the same call sequence."""
        hs = (_vp * world)()
        _chk(load().cpkit_dev_problem_create_loopback(device, _dims(dims), _u64(len(dims)), _u64(rank), world,
                                                      hs))
        out = []
        for r in range(world):
            p = cls.__new__(cls)
            p.dims = [int(d) for d in dims]
            p.rank = int(rank)
            p._h = _vp(hs[r])
            p.stacked = sum(p.dims) * p.rank
            out.append(p)
        return out

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cpkit_dev_problem_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def slab(self):
        lo, hi, n = _u64(), _u64(), _u64()
        _chk(load().cpkit_dev_slab(self._h, C.byref(lo), C.byref(hi), C.byref(n)))
        return lo.value, hi.value, n.value

    # The cpkit_dev_* entries take bare pointers sized by the problem; every
    # buffer is checked here so a wrong shape or dtype raises ValueError
    # instead of reading or writing past the end of a host array.
    def _factor_stack(self, blocks, what="factors") -> np.ndarray:
        if len(blocks) != len(self.dims):
            raise ValueError(f"{what}: expected {len(self.dims)} blocks, got {len(blocks)}")
        for n, b in enumerate(blocks):
            if np.shape(b) != (self.dims[n], self.rank):
                raise ValueError(f"{what}[{n}]: expected shape {(self.dims[n], self.rank)}, got {np.shape(b)}")
        return stack(blocks)

    def _slab_array(self, x, what) -> np.ndarray:
        n = self.slab()[2]
        if np.size(x) != n:
            raise ValueError(f"{what}: expected {n} elements (the local slab), got {np.size(x)}")
        return _f64(x)

    def upload(self, x_local: np.ndarray):
        x = self._slab_array(x_local, "upload")
        _chk(load().cpkit_dev_upload_tensor(self._h, _ptr(x)))

    def load_file(self, path: str):
        """CPKT1 file -> this shard's slab on the device, streamed (cpkit_dev_load_tensor)."""
        _chk(load().cpkit_dev_load_tensor(self._h, path.encode()))

    def generate(self, truth: Sequence[np.ndarray], noise_seed: int = 0, noise_rel: float = 0.0):
        buf = self._factor_stack(truth, "truth")
        _chk(load().cpkit_dev_generate_tensor(self._h, _ptr(buf), _u64(noise_seed),
                                              C.c_double(noise_rel)))

    def set_factors(self, factors):
        buf = self._factor_stack(factors)
        _chk(load().cpkit_dev_set_factors(self._h, _ptr(buf)))

    def get_factors(self):
        buf = np.empty(self.stacked)
        _chk(load().cpkit_dev_get_factors(self._h, _ptr(buf)))
        return unstack(buf, self.dims, self.rank)

    def norm2(self) -> float:
        v = C.c_double()
        _chk(load().cpkit_dev_norm2(self._h, C.byref(v)))
        return v.value

    def mttkrp(self, mode: int, download: bool = True):
        rows = self.dims[mode] if 0 <= mode < len(self.dims) else 1
        out = np.empty((rows, self.rank)) if download else None
        _chk(load().cpkit_dev_mttkrp(self._h, _u64(mode), _ptr(out)))
        return out

    def mttkrp_naive(self, mode: int):
        rows = self.dims[mode] if 0 <= mode < len(self.dims) else 1
        out = np.empty((rows, self.rank))
        _chk(load().cpkit_dev_mttkrp_naive(self._h, _u64(mode), _ptr(out)))
        return out

    def note_factor_update(self, mode: int):
        _chk(load().cpkit_dev_note_factor_update(self._h, _u64(mode)))

    @property
    def full_contractions(self) -> int:
        return load().cpkit_dev_full_contractions(self._h)

    def reset_contraction_counter(self):
        load().cpkit_dev_reset_contraction_counter(self._h)

    def gamma_set(self):
        n, r = len(self.dims), self.rank
        g = np.empty((n, r, r))
        p = np.empty((n, n, r, r))
        _chk(load().cpkit_dev_gamma_set(self._h, _ptr(g), _ptr(p)))
        return g, p

    def set_gamma_set(self, grams, pair):
        n, r = len(self.dims), self.rank
        if np.size(grams) != n * r * r or np.size(pair) != n * n * r * r:
            raise ValueError("set_gamma_set: expected N*R*R grams and N*N*R*R pairwise blocks")
        g, p = _f64(grams), _f64(pair)
        _chk(load().cpkit_dev_set_gamma_set(self._h, _ptr(g), _ptr(p)))

    def residual(self, xnorm2: float):
        r, f = C.c_double(), C.c_double()
        _chk(load().cpkit_dev_residual(self._h, C.c_double(xnorm2), C.byref(r), C.byref(f)))
        return r.value, f.value

    def gradient(self, mttkrps=None):
        out = np.empty(self.stacked)
        m = None if mttkrps is None else self._factor_stack(mttkrps, "mttkrps")
        _chk(load().cpkit_dev_gradient(self._h, _ptr(m), _ptr(out)))
        return unstack(out, self.dims, self.rank)

    def jtj_matvec(self, w, lam: float, shape: int = 0):
        wb = self._factor_stack(w, "w")
        out = np.empty(self.stacked)
        _chk(load().cpkit_dev_jtj_matvec(self._h, _ptr(wb), C.c_double(lam), shape, _ptr(out)))
        return unstack(out, self.dims, self.rank)

    def preconditioner(self, lam: float, shape: int = 0):
        out = np.empty((len(self.dims), self.rank, self.rank))
        _chk(load().cpkit_dev_preconditioner(self._h, C.c_double(lam), shape, _ptr(out)))
        return out

    def cp_cg(self, g, lam: float, gn: Optional[dict] = None):
        gb = self._factor_stack(g, "g")
        out = np.empty(self.stacked)
        it, cap, bd = C.c_int(), C.c_int(), C.c_int()
        _chk(load().cpkit_dev_cp_cg(self._h, _ptr(gb), C.c_double(lam),
                                    None if gn is None else json.dumps(gn).encode(), _ptr(out),
                                    C.byref(it), C.byref(cap), C.byref(bd)))
        return unstack(out, self.dims, self.rank), it.value, bool(cap.value), bool(bd.value)

    def spd_solve(self, s, b, lam: float):
        s, b = _f64(s), _f64(b)
        r = self.rank
        if s.shape != (r, r) or b.ndim != 2 or b.shape[1] != r:
            raise ValueError(f"spd_solve: need S ({r}, {r}) and B (rows, {r})")
        out = np.empty_like(b)
        _chk(load().cpkit_dev_spd_solve(self._h, _ptr(s), _ptr(b), _u64(b.shape[0]),
                                        C.c_double(lam), _ptr(out)))
        return out

    def spd_inverse(self, s, lam: float):
        s = _f64(s)
        if s.shape != (self.rank, self.rank):
            raise ValueError(f"spd_inverse: need S ({self.rank}, {self.rank})")
        out = np.empty_like(s)
        _chk(load().cpkit_dev_spd_inverse(self._h, _ptr(s), C.c_double(lam), _ptr(out)))
        return out

    def als_sweep(self, lam: float):
        sn, cnt = C.c_double(), C.c_int()
        _chk(load().cpkit_dev_als_sweep(self._h, C.c_double(lam), C.byref(sn), C.byref(cnt)))
        return sn.value, cnt.value

    def gn_step(self, gn: Optional[dict], xnorm2: float):
        d = np.empty(12)
        _chk(load().cpkit_dev_gn_step(self._h, None if gn is None else json.dumps(gn).encode(),
                                      C.c_double(xnorm2), _ptr(d)))
        keys = ("halt", "stepped", "residual_before", "residual_after", "grad_norm", "lambda",
                "cg_iters", "step_norm", "alpha", "armijo_exhausted", "cg_hit_cap",
                "cg_breakdown")
        return dict(zip(keys, d.tolist()))

    def optimize(self, config: dict, init=None):
        ib = None if init is None else self._factor_stack(init, "init")
        out = np.empty(self.stacked)
        r = _vp()
        _chk(load().cpkit_dev_optimize(self._h, json.dumps(config).encode(), _ptr(ib), _ptr(out),
                                       C.byref(r)))
        return unstack(out, self.dims, self.rank), Report(r)

    # ---- timing (CUDA events on the problem's own stream)
    def time_als_sweeps(self, lam: float, sweeps: int) -> float:
        ms = C.c_double()
        _chk(load().cpkit_dev_time_als_sweeps(self._h, C.c_double(lam), sweeps, C.byref(ms)))
        return ms.value

    def time_roots(self, reps: int):
        a, b = C.c_double(), C.c_double()
        _chk(load().cpkit_dev_time_roots(self._h, reps, C.byref(a), C.byref(b)))
        return a.value, b.value

    def profile(self, enable: bool):
        _chk(load().cpkit_dev_profile(self._h, 1 if enable else 0))

    def profile_read(self):
        ms = (C.c_double * 3)()
        cnt = (C.c_int * 3)()
        _chk(load().cpkit_dev_profile_read(self._h, ms, cnt))
        return list(ms), list(cnt)

    def time_jtj(self, reps: int) -> float:
        ms = C.c_double()
        _chk(load().cpkit_dev_time_jtj(self._h, reps, C.byref(ms)))
        return ms.value

    def download(self) -> np.ndarray:
        lo, hi, n = self.slab()
        out = np.empty(n)
        _chk(load().cpkit_dev_download_tensor(self._h, _ptr(out)))
        return out.reshape(self.dims[:-1] + [hi - lo])

    def download_into(self, out: np.ndarray) -> None:
        n = self.slab()[2]
        if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.flags.c_contiguous
                and out.flags.writeable and out.size == n):
            raise ValueError(f"download_into: need a writable C-contiguous float64 array of {n} elements")
        _chk(load().cpkit_dev_download_tensor(self._h, _ptr(out)))

    def time_gn_steps(self, gn: Optional[dict], steps: int):
        ms, cg = C.c_double(), C.c_int()
        _chk(load().cpkit_dev_time_gn_steps(self._h, None if gn is None else json.dumps(gn).encode(),
                                            steps, C.byref(ms), C.byref(cg)))
        return ms.value, cg.value

    def time_norm2(self, reps: int) -> float:
        ms = C.c_double()
        _chk(load().cpkit_dev_time_norm2(self._h, reps, C.byref(ms)))
        return ms.value


    def time_second_level(self, reps: int):
        """(ms per pass, bytes of the back-root partial) of the second tree level, mode 0."""
        ms, nbytes = C.c_double(), C.c_double()
        _chk(load().cpkit_dev_time_second_level(self._h, reps, C.byref(ms), C.byref(nbytes)))
        return ms.value, nbytes.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _chk(load().cpkit_dev_nccl_unique_id(buf))
    return buf.raw


def probe_dmma_peak(device: int = 0) -> float:
    v = C.c_double()
    _chk(load().cpkit_dev_probe_dmma_peak(device, C.byref(v)))
    return v.value


def random_factors(dims, rank, seed, kind="uniform", a=0.0, b=1.0):
    """generators.cpp:59-76 seeded factor draws, computed by the library."""
    out = np.empty(sum(int(d) for d in dims) * rank)
    _chk(load().cpkit_dev_random_factors(_dims(dims), _u64(len(dims)), _u64(rank), _u64(seed),
                                         0 if kind == "uniform" else 1, C.c_double(a),
                                         C.c_double(b), _ptr(out)))
    return unstack(out, dims, rank)


def shard_range(extent: int, shard: int, world: int):
    """Rows [lo, hi) of the last mode owned by `shard` (no GPU needed)."""
    lo, hi = C.c_uint64(), C.c_uint64()
    _chk(load().cpkit_dev_shard_range(_u64(extent), shard, world, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def problem_seed(master: int, rank: int, problem: int) -> int:
    return int(load().cpkit_dev_problem_seed(master, rank, problem))


def init_seed(master: int, rank: int, problem: int, init: int) -> int:
    return int(load().cpkit_dev_init_seed(master, rank, problem, init))


def kernel_launches() -> int:
    return int(load().cpkit_dev_kernel_launches())


def guard_violations() -> int:
    """Released device buffers whose red zones were overwritten (CPKIT_GUARD=1 mode)."""
    return int(load().cpkit_dev_guard_violations())


def guard_selftest() -> bool:
    """Positive control of the guard mode (needs CPKIT_GUARD=1 in the environment)."""
    d = C.c_int()
    _chk(load().cpkit_dev_guard_selftest(C.byref(d)))
    return bool(d.value)
