"""Generate tests/golden/golden_r01.json from the CPU oracle.

The reference ships no golden files and cannot be built here,
so these fixtures are produced by the oracle AFTER it passes every reference
known-answer test (tests/test_oracle_kats.py). They freeze seeded RNG draws
(bitwise, as IEEE-754 hex), seed derivations, a bit-exact reconstruction and
small-problem outputs of every hot-path function, so later rounds (and the
device path) are checked against the same numbers.

Run:  python tests/golden/make_golden.py
"""
import json
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as orc  # noqa: E402


def hexd(v):
    return struct.pack(">d", float(v)).hex()


def arr(a):
    return np.asarray(a, dtype=np.float64).ravel().tolist()


def main():
    g = {"generator": "oracle/cpkit_oracle.cpp via tests/golden/make_golden.py", "rng": {}, "seeds": {}}
    for x in (0, 1, 12345, 2**63):
        g["rng"][f"mix64({x})"] = orc.mix64(x)
    for seed, stream, idx in ((0, 0, 0), (7, 1, 99), (2**40 + 3, 0x4E01, 123456)):
        g["rng"][f"keyed({seed},{stream},{idx},0)"] = orc.keyed(seed, stream, idx, 0)
        g["rng"][f"uniform({seed},{stream},{idx})"] = hexd(orc.uniform(seed, stream, idx, 0.0, 1.0))
        g["rng"][f"gaussian({seed},{stream},{idx})"] = hexd(orc.gaussian(seed, stream, idx))
    for m, r, p in ((0, 100, 0), (0, 5, 0), (42, 7, 3)):
        g["seeds"][f"problem_seed({m},{r},{p})"] = orc.problem_seed(m, r, p)
        g["seeds"][f"init_seed({m},{r},{p},0)"] = orc.init_seed(m, r, p, 0)

    dims, rank = [4, 3, 5], 2
    truth = orc.random_model(dims, rank, orc.problem_seed(0, rank, 0))
    x = orc.reconstruct(truth)
    init = orc.random_model(dims, rank, orc.init_seed(0, rank, 0, 0), kind="gaussian")
    ms, cnt = orc.mttkrp_tree_all(x, init)
    grams, pair = orc.gamma_set(init)
    xn2 = orc.norm2(x)
    grad = orc.gradient(init, ms, grams, pair)
    w = orc.random_model(dims, rank, 99, kind="gaussian")
    mv = orc.hessian_matvec(init, grams, pair, w, 1e-2)
    v, it, cap, bd = orc.cp_cg(init, grams, pair, grad, 1e-2, orc.GnConfig())
    r, f = orc.residual(x, init, xn2, ms[-1])
    f_gn, d_gn = orc.gn_step(x, init, orc.GnConfig(), xn2)
    f_als, step, c_als, _ = orc.als_sweep(x, init, 1e-3)
    _, recs_gn, st_gn = orc.gn_optimize(x, init, orc.GnConfig(max_iters=30))
    _, recs_als, st_als = orc.als_optimize(x, init, orc.AlsConfig(max_sweeps=30))
    g["small"] = {
        "dims": dims, "rank": rank,
        "truth": [arr(a) for a in truth], "x_hex_first8": [hexd(v) for v in x.ravel()[:8]],
        "x": arr(x), "init": [arr(a) for a in init], "xnorm2": xn2,
        "mttkrp": [arr(a) for a in ms], "contractions": cnt,
        "grams": arr(grams), "pairwise": arr(pair), "residual": [r, f],
        "gradient": [arr(a) for a in grad], "w": [arr(a) for a in w], "matvec_lambda": 1e-2,
        "matvec": [arr(a) for a in mv],
        "cg": {"lambda": 1e-2, "v": [arr(a) for a in v], "iterations": it, "hit_cap": cap, "breakdown": bd},
        "gn_step": {"diag": d_gn, "factors": [arr(a) for a in f_gn]},
        "als_sweep": {"lambda": 1e-3, "factors": [arr(a) for a in f_als], "step_norm": step, "contractions": c_als},
        "gn_trace": {"max_iters": 30, "status": st_gn, "records": recs_gn},
        "als_trace": {"max_sweeps": 30, "status": st_als, "records": recs_als},
    }
    for rec in g["small"]["gn_trace"]["records"] + g["small"]["als_trace"]["records"]:
        rec.pop("seconds", None)
    with open(os.path.join(HERE, "golden_r01.json"), "w") as fh:
        json.dump(g, fh, indent=1)
    print("wrote", os.path.join(HERE, "golden_r01.json"))


if __name__ == "__main__":
    main()
