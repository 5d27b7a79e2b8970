"""The sharded (NCCL) code path on one GPU: a one-rank NCCL communicator routes
every collective of DeviceProblem (all-reduce of M^(n) partials, all-gather of
M^(N-1) slab rows, scalar all-reduces) through libnccl. Results must equal the
unsharded path bit for bit (a one-rank all-reduce/all-gather is a copy)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_one_rank_nccl_path_matches_unsharded(orc):
    from paper_1910_12331_b200 import cpkit
    dims, R = [24, 20, 28], 6
    truth = orc.random_model(dims, R, 3)
    x = orc.reconstruct(truth)
    init = orc.random_model(dims, R, 4)
    plain = cpkit.DeviceProblem(dims, R)
    plain.upload(x)
    shard = cpkit.DeviceProblem(dims, R, shard=0, world=1, nccl_id=cpkit.nccl_unique_id())
    assert shard.slab() == (0, dims[-1], x.size)
    shard.upload(x)
    assert shard.norm2() == plain.norm2()
    for p in (plain, shard):
        p.set_factors(init)
    for n in range(3):
        assert np.array_equal(plain.mttkrp(n), shard.mttkrp(n))
    f1, r1 = plain.optimize({"optimizer": "als", "als": {"max_sweeps": 5}}, init)
    f2, r2 = shard.optimize({"optimizer": "als", "als": {"max_sweeps": 5}}, init)
    for a, b in zip(f1, f2):
        assert np.array_equal(a, b)
    f1, r1 = plain.optimize({"optimizer": "gn", "gn": {"max_iters": 3}}, init)
    f2, r2 = shard.optimize({"optimizer": "gn", "gn": {"max_iters": 3}}, init)
    assert [r["cg_iters"] for r in r1.to_json()["records"]] == [r["cg_iters"] for r in r2.to_json()["records"]]
    for a, b in zip(f1, f2):
        assert np.array_equal(a, b)
