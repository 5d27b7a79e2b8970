"""Small workload for the guarded allocation mode (CPKIT_GUARD=1,
tests/test_gpu_guard.py; compute-sanitizer itself is closed on the GPU pool):
every device kernel
family of the product on shapes that take the same code paths as the BASELINE
configs (TMA + mbarrier root GEMM with its tail launch, split-K TN root,
cluster Gram, blocked Cholesky, cooperative tile-resident and streaming CG with
the software grid barrier, pipelined GN/ALS drivers with CUDA graphs, batched
tiny instances), sized to finish in seconds.

Checks the MTTKRPs against numpy so a run whose buffers were corrupted fails. Not a test: tests/ holds the parity
suite."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit  # noqa: E402

SMALL = os.environ.get("SAN_SMALL") == "1"


def mttkrp_ref(x, f, n):
    N = x.ndim
    letters = "abcdefgh"[:N]
    ops, subs = [x], [letters]
    for m in range(N):
        if m != n:
            ops.append(f[m])
            subs.append(letters[m] + "z")
    return np.einsum(",".join(subs) + "->" + letters[n] + "z", *ops)


def case(dims, R, seed):
    truth = cpkit.random_factors(dims, R, seed)
    p = cpkit.DeviceProblem(dims, R)
    p.generate(truth, noise_seed=seed, noise_rel=1e-3)
    init = cpkit.random_factors(dims, R, seed + 100)
    p.set_factors(init)
    x = p.download() if np.prod(dims) <= 4_000_000 else None
    for n in range(len(dims)):
        got = p.mttkrp(n)
        if x is not None:
            ref = mttkrp_ref(x, init, n)
            err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            assert err < 1e-10, (dims, R, n, err)
    xn2 = p.norm2()
    p.set_factors(init)
    for _ in range(2):
        p.als_sweep(1e-3)
    p.set_factors(init)
    p.gn_step({"cg_max_iters": 15}, xn2)
    p.set_factors(init)
    rep = p.optimize({"optimizer": "als", "als": {"max_sweeps": 4}})
    rep = p.optimize({"optimizer": "gn", "gn": {"max_iters": 3, "cg_max_iters": 10}})
    p.gamma_set()
    g = cpkit.random_factors(dims, R, seed + 7, kind="gaussian")
    p.jtj_matvec(g, 1e-3)
    p.cp_cg(g, 1e-3, {"cg_max_iters": 12})
    s = cpkit.random_factors([R], R, seed + 9)[0]
    s = s.T @ s + np.eye(R)
    p.spd_inverse(s, 1e-3)
    p.close()
    print("case ok", dims, R, flush=True)


def main():
    cases = [([40, 36, 33], 24, 1), ([24, 20, 18, 16], 12, 2), ([9, 7, 5], 3, 3)]
    if not SMALL:
        cases += [([120, 100, 96], 100, 4), ([48, 40, 36, 32], 50, 5)]
    for dims, R, seed in cases:
        case(dims, R, seed)
    rep = cpkit.run_likelihood({"problem": {"family": "uniform01", "dims": [4, 4, 4], "ranks": [2]},
                                "optimizer": "gn", "problems": 1, "inits": 4, "seed": 5,
                                "gn": {"max_iters": 10}}).to_json()
    assert rep["ranks"][0]["problems"][0]["inits"], rep
    print("sanitize driver done; kernels launched:", cpkit.kernel_launches(), flush=True)


if __name__ == "__main__":
    main()
