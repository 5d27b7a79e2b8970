"""The BLAS CPU-baseline arm (oracle/blas_arm.py) agrees with the pinned
oracle restatement: it times the same algorithm the GPU is compared with."""
import numpy as np
import pytest

from oracle import blas_arm as ba
from tests.helpers import rel_err, vec_rel_err


@pytest.mark.parametrize("dims,rank", [([7, 6, 5], 3), ([6, 5, 4, 3], 4), ([4, 3, 5, 2, 3], 2)])
def test_tree_mttkrp(orc, dims, rank):
    x = np.random.default_rng(1).standard_normal(dims)
    f = orc.random_model(dims, rank, 4, kind="gaussian")
    ref, cnt = orc.mttkrp_tree_all(x, f)
    t = ba.Tree(x)
    for n in range(len(dims)):
        assert rel_err(t.mttkrp(f, n), ref[n]) < 1e-12
    assert t.contractions == cnt


@pytest.mark.parametrize("dims,rank", [([9, 8, 7], 3), ([6, 5, 4, 3], 2)])
def test_als_and_gn_steps(orc, dims, rank):
    truth = orc.random_model(dims, rank, 7)
    x = orc.reconstruct(truth)
    orc.add_noise(x, 2, 1e-3)
    init = orc.random_model(dims, rank, 8)
    f_ref, step_ref, cnt_ref, _ = orc.als_sweep(x, init, 1e-3)
    f, step, cnt, _ = ba.als_sweep(ba.Tree(x), init, 1e-3)
    assert vec_rel_err(f, f_ref) < 1e-10 and abs(step - step_ref) < 1e-10 * step_ref and cnt == cnt_ref
    xn2 = orc.norm2(x)
    f_ref, d_ref = orc.gn_step(x, init, orc.GnConfig(), xn2)
    f, d = ba.gn_step(x, init, 1e-2, xn2)
    assert d["cg_iters"] == d_ref["cg_iters"]
    assert abs(d["residual_after"] - d_ref["residual_after"]) < 1e-10
    assert vec_rel_err(f, f_ref) < 1e-9


def test_als_optimize_matches_oracle(orc):
    dims, rank = [8, 7, 6], 3
    truth = orc.random_model(dims, rank, 11)
    x = orc.reconstruct(truth)
    init = orc.random_model(dims, rank, 12)
    f_ref, recs, st = orc.als_optimize(x, init, orc.AlsConfig(max_sweeps=60, lambda0=1e-3, decay_every=5))
    f, recs2, st2 = ba.als_optimize(x, init, max_sweeps=60, lambda0=1e-3, decay_every=5)
    assert st2 == st and len(recs2) == len(recs)
    for a, b in zip(recs2, recs):
        assert a["lambda"] == b["lambda"] and abs(a["residual"] - b["residual"]) < 1e-9
    assert vec_rel_err(f, f_ref) < 1e-8


def test_gn_optimize_matches_oracle(orc):
    dims, rank = [8, 7, 6], 3
    truth = orc.random_model(dims, rank, 21)
    x = orc.reconstruct(truth)
    orc.add_noise(x, 3, 1e-4)
    init = orc.random_model(dims, rank, 22)
    f_ref, recs, st = orc.gn_optimize(x, init, orc.GnConfig(max_iters=15))
    f, recs2, st2 = ba.gn_optimize(x, init, max_iters=15)
    assert st2 == st and len(recs2) == len(recs)
    for a, b in zip(recs2, recs):
        assert a["lambda"] == b["lambda"] and a["cg_iters"] == b["cg_iters"]
        assert abs(a["residual"] - b["residual"]) < 1e-9
    assert vec_rel_err(f, f_ref) < 1e-7
