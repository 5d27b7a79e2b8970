"""Cluster mode of the tile-resident CG (kernels_cg_res.cu, CLU): the nct
column tiles of a row block form a thread-block cluster and exchange sibling
columns through distributed shared memory. Every CTA still computes the same
operands in the same order, so the solve must be BITWISE equal to the L2-gather
version (CPKIT_CG_NO_CLUSTER=1), and both must match the oracle's cp_cg."""
import os

import numpy as np
import pytest

from tests.helpers import vec_rel_err

pytestmark = pytest.mark.gpu

CASES = [([120, 100, 96], 100), ([60, 50, 40], 64), ([80, 70, 66], 50), ([50, 45, 40], 75),
         ([30, 28, 26, 24], 40), ([400, 400, 400], 100)]


@pytest.mark.parametrize("dims,R", CASES)
def test_cluster_cg_bitwise_equals_gather_cg(orc, dims, R):
    from paper_1910_12331_b200 import cpkit
    f = cpkit.random_factors(dims, R, 3)
    g = cpkit.random_factors(dims, R, 4, kind="gaussian")
    out = {}
    for mode in ("cluster", "gather"):
        if mode == "gather":
            os.environ["CPKIT_CG_NO_CLUSTER"] = "1"
        try:
            p = cpkit.DeviceProblem(dims, R)
            p.set_factors(f)
            p.gamma_set()
            out[mode] = p.cp_cg(g, 1e-3, {"cg_max_iters": 60, "cg_tol": 1e-10})
            p.close()
        finally:
            os.environ.pop("CPKIT_CG_NO_CLUSTER", None)
    (v1, it1, c1, b1), (v2, it2, c2, b2) = out["cluster"], out["gather"]
    assert (it1, c1, b1) == (it2, c2, b2)
    for a, b in zip(v1, v2):
        assert np.array_equal(a, b)
    if np.prod(dims) <= 400_000:
        cfg = orc.GnConfig(cg_max_iters=60, cg_tol=1e-10)
        grams, pair = orc.gamma_set(f)
        v_ref, it_ref, cap_ref, bd_ref = orc.cp_cg(f, grams, pair, g, 1e-3, cfg)
        assert (it1, c1, b1) == (it_ref, cap_ref, bd_ref)
        assert vec_rel_err(v1, v_ref) < 1e-9
