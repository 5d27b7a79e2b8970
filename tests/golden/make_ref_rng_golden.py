"""Golden vectors of the REFERENCE's keyed RNG (proj/src/core/rng.hpp), taken
from oracle/_ref/libref_rng.so, which oracle/Makefile compiles from the
reference's own header. Run here (where /root/reference exists):
    make -C oracle && python tests/golden/make_ref_rng_golden.py
"""
import ctypes as C
import json
import os
import struct

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def cases():
    out = []
    for seed in (0, 1, 5, 12345, 2**63 + 7):
        for stream in (0, 1, 2, 3, 4, 0xDD, 0x4E01, 0x5701, 0x5802):
            for index in (0, 1, 2, 99, 4999, 10**9 + 3, 2**40 + 5):
                out.append((seed, stream, index))
    return out


def main():
    L = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libref_rng.so"))
    u64 = C.c_uint64
    L.ref_uniform.restype = C.c_double
    L.ref_uniform.argtypes = [u64, u64, u64, C.c_double, C.c_double]
    L.ref_gaussian.restype = C.c_double
    L.ref_gaussian.argtypes = [u64, u64, u64]
    L.ref_keyed.restype = u64
    L.ref_keyed.argtypes = [u64, u64, u64, u64]
    hx = lambda v: struct.pack(">d", v).hex()
    rows = []
    for s, st, i in cases():
        rows.append({"seed": s, "stream": st, "index": i,
                     "uniform01": hx(L.ref_uniform(s, st, i, 0.0, 1.0)),
                     "uniform_m2_3": hx(L.ref_uniform(s, st, i, -2.0, 3.0)),
                     "gaussian": hx(L.ref_gaussian(s, st, i)),
                     "keyed_salt0": str(L.ref_keyed(s, st, i, 0))})
    with open(os.path.join(HERE, "ref_rng.json"), "w") as fh:
        json.dump({"source": "reference proj/src/core/rng.hpp via oracle/ref_rng_shim.cpp", "rows": rows}, fh, indent=0)


if __name__ == "__main__":
    main()
