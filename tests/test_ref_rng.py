"""The oracle's keyed RNG (cpkit_oracle.cpp, SplitMix restatement of
rng.hpp:11-46) pinned bit for bit to the REFERENCE's own header: against golden
vectors made from it (tests/golden/ref_rng.json) and, where the reference
source tree is present, against oracle/_ref/libref_rng.so compiled from it
(oracle/Makefile) on a random sample. The device generators are in turn
bitwise equal to the oracle (tests/test_gpu_noise.py, test_golden.py)."""
import ctypes as C
import json
import os
import struct

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REFLIB = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "libref_rng.so")


def hx(v):
    return struct.pack(">d", float(v)).hex()


def test_oracle_matches_reference_rng_golden(orc):
    with open(os.path.join(HERE, "golden", "ref_rng.json")) as fh:
        rows = json.load(fh)["rows"]
    assert len(rows) >= 300
    for r in rows:
        s, st, i = r["seed"], r["stream"], r["index"]
        assert hx(orc.uniform(s, st, i, 0.0, 1.0)) == r["uniform01"], r
        assert hx(orc.uniform(s, st, i, -2.0, 3.0)) == r["uniform_m2_3"], r
        assert hx(orc.gaussian(s, st, i)) == r["gaussian"], r


@pytest.mark.skipif(not os.path.exists(REFLIB), reason="reference source tree not present (GPU box)")
def test_oracle_matches_reference_rng_sampled(orc):
    L = C.CDLL(REFLIB)
    u64 = C.c_uint64
    L.ref_uniform.restype = C.c_double
    L.ref_uniform.argtypes = [u64, u64, u64, C.c_double, C.c_double]
    L.ref_gaussian.restype = C.c_double
    L.ref_gaussian.argtypes = [u64, u64, u64]
    rng = np.random.default_rng(2024)
    for _ in range(3000):
        s, st, i = (int(v) for v in rng.integers(0, 2**62, size=3))
        st %= 0x10000
        assert orc.uniform(s, st, i, 0.0, 1.0) == L.ref_uniform(s, st, i, 0.0, 1.0)
        g1, g2 = orc.gaussian(s, st, i), L.ref_gaussian(s, st, i)
        assert hx(g1) == hx(g2), (s, st, i, g1, g2)


REF_HARNESS = "/root/reference/proj/src/core/harness.cpp"


@pytest.mark.skipif(not (os.path.exists(REFLIB) and os.path.exists(REF_HARNESS)),
                    reason="reference source tree not present (GPU box)")
def test_seed_derivation_matches_reference(orc):
    """harness.cpp:378-391 problem_seed / init_seed: the reference's derive /
    mix64 chain (from rng.hpp, via the shim) with the tag constants read from
    the reference source, against the oracle's derivation."""
    import re
    src = open(REF_HARNESS).read()
    tags = {k: int(v, 0) for k, v in re.findall(r"(kProblemTag|kInitTag)\s*=\s*(0x[0-9A-Fa-f]+)", src)}
    assert set(tags) == {"kProblemTag", "kInitTag"}
    L = C.CDLL(REFLIB)
    for f in ("ref_mix64", "ref_derive"):
        getattr(L, f).restype = C.c_uint64
    L.ref_mix64.argtypes = [C.c_uint64]
    L.ref_derive.argtypes = [C.c_uint64, C.c_uint64]
    for master in (0, 1, 7, 2**40 + 3):
        for rank in (1, 5, 100, 200):
            for prob in (0, 1, 29):
                ps = L.ref_derive(L.ref_derive(L.ref_derive(L.ref_mix64(master), tags["kProblemTag"]), rank), prob)
                assert orc.problem_seed(master, rank, prob) == ps
                for init in (0, 4):
                    h = L.ref_derive(L.ref_derive(L.ref_derive(L.ref_mix64(master), tags["kInitTag"]), rank), prob)
                    assert orc.init_seed(master, rank, prob, init) == L.ref_derive(h, init)
