"""The product's sharded code path (last-mode slabs, NCCL
all-reduce of the s x R MTTKRP partials, all-gather of the last-mode rows,
scalar all-reduces) run on ONE GPU with 2 and 4 shards joined by the
in-process loopback group (cpkit_dev_problem_create_loopback): the same
DeviceProblem code and collective sequence as a multi-GPU job, each shard on
its own host thread. Every result is compared with the UNSHARDED oracle.

Sharded sums associate differently from the unsharded ones (partials summed
over ranks), so kernel outputs are held at 1e-11 and trajectories at the
north star's tolerances; generation is bit-exact (shard-invariant order).
"""
import threading

import numpy as np
import pytest

from tests.helpers import rel_err, vec_rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ck():
    from paper_1910_12331_b200 import cpkit
    cpkit.load()
    return cpkit


def on_ranks(probs, fn):
    """fn(rank, problem) on one thread per shard; returns the per-rank results."""
    out, errs = [None] * len(probs), []

    def run(r):
        try:
            out[r] = fn(r, probs[r])
        except Exception as exc:  # re-raised below
            errs.append((r, exc))

    ts = [threading.Thread(target=run, args=(r,)) for r in range(len(probs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errs, errs
    return out


def slab_of(x, r, world):
    s = x.shape[-1] // world
    return np.ascontiguousarray(x[..., r * s:(r + 1) * s])


CASES = [([12, 10, 8], 3, 2), ([12, 10, 8], 3, 4), ([6, 5, 7, 8], 4, 2), ([6, 5, 7, 8], 4, 4),
         ([40, 36, 32], 10, 4)]


@pytest.mark.parametrize("dims,rank,world", CASES)
def test_sharded_generation_is_bitwise(orc, ck, dims, rank, world):
    truth = orc.random_model(dims, rank, orc.problem_seed(2, rank, 0))
    x = orc.reconstruct(truth)
    orc.add_noise(x, 9, 1e-3)
    probs = ck.DeviceProblem.loopback(dims, rank, world)
    slabs = on_ranks(probs, lambda r, p: (p.generate(truth, noise_seed=9, noise_rel=1e-3), p.download())[1])
    for r in range(world):
        assert np.array_equal(slabs[r], slab_of(x, r, world)), r
    xn = on_ranks(probs, lambda r, p: p.norm2())
    assert len(set(xn)) == 1 and abs(xn[0] - orc.norm2(x)) <= 1e-13 * orc.norm2(x)


@pytest.mark.parametrize("dims,rank,world", CASES)
def test_sharded_mttkrp_every_mode(orc, ck, dims, rank, world):
    rng = np.random.default_rng(len(dims) * 10 + world)
    x = rng.standard_normal(dims)
    f = orc.random_model(dims, rank, 5, kind="gaussian")
    ref, _ = orc.mttkrp_tree_all(x, f)
    probs = ck.DeviceProblem.loopback(dims, rank, world)

    def run(r, p):
        p.upload(slab_of(x, r, world))
        p.set_factors(f)
        return [p.mttkrp(n) for n in range(len(dims))]

    got = on_ranks(probs, run)
    for r in range(world):
        for n in range(len(dims)):
            assert rel_err(got[r][n], ref[n]) < 1e-11, (r, n)
            assert np.array_equal(got[r][n], got[0][n])  # collectives leave every rank the same bits


@pytest.mark.parametrize("dims,rank,world", CASES)
def test_sharded_als_sweeps(orc, ck, dims, rank, world):
    truth = orc.random_model(dims, rank, orc.problem_seed(1, rank, 0))
    x = orc.reconstruct(truth)
    orc.add_noise(x, 3, 1e-4)
    init = orc.random_model(dims, rank, orc.init_seed(1, rank, 0, 0))
    probs = ck.DeviceProblem.loopback(dims, rank, world)

    def run(r, p):
        p.upload(slab_of(x, r, world))
        p.set_factors(init)
        steps = [p.als_sweep(1e-3)[0] for _ in range(4)]
        return steps, p.get_factors()

    got = on_ranks(probs, run)
    f = init
    for k in range(4):
        f, step, _, _ = orc.als_sweep(x, f, 1e-3)
        for r in range(world):
            assert abs(got[r][0][k] - step) <= 1e-9 * max(step, 1.0), (k, r)
    for r in range(world):
        assert vec_rel_err(got[r][1], f) < 1e-9, r
        for a, b in zip(got[r][1], got[0][1]):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("dims,rank,world", CASES)
def test_sharded_gn_steps(orc, ck, dims, rank, world):
    truth = orc.random_model(dims, rank, orc.problem_seed(4, rank, 0))
    x = orc.reconstruct(truth)
    orc.add_noise(x, 6, 1e-4)
    # a start 5% off the truth: GN converges, so a step is well conditioned (a
    # diverging random start makes the capped CG's V roundoff-sensitive)
    pert = orc.random_model(dims, rank, 99, kind="gaussian")
    init = [t + 0.05 * q for t, q in zip(truth, pert)]
    xn2 = orc.norm2(x)
    # per-step parity from identical states (a free-running GN trajectory can
    # move a CG count by one once roundoff differs)
    fs, ds = [init], []
    for k in range(3):  # cpkit_dev_gn_step starts a fresh schedule per call, as the oracle's gn_step
        f, d = orc.gn_step(x, fs[-1], orc.GnConfig(cg_max_iters=50), xn2)
        fs.append(f)
        ds.append(d)
    probs = ck.DeviceProblem.loopback(dims, rank, world)

    def run(r, p):
        p.upload(slab_of(x, r, world))
        out = []
        for k in range(3):
            p.set_factors(fs[k])
            out.append((p.gn_step({"cg_max_iters": 50}, xn2), p.get_factors()))
        return out

    got = on_ranks(probs, run)
    for k in range(3):
        for r in range(world):
            dg, fg = got[r][k]
            assert int(dg["cg_iters"]) == ds[k]["cg_iters"], (k, r, dg, ds[k])
            assert abs(dg["residual_after"] - ds[k]["residual_after"]) < 1e-9, (k, r)
            assert vec_rel_err(fg, fs[k + 1]) < 1e-8, (k, r)


@pytest.mark.parametrize("optimizer", ["als", "gn"])
def test_sharded_optimize_trace(orc, ck, optimizer):
    """The pipelined drivers (als_optimize / gn_optimize) on 4 shards against the
    unsharded oracle: same record count, lambda and CG counts, residuals <= 1e-8."""
    dims, rank, world = [20, 18, 16], 4, 4
    truth = orc.random_model(dims, rank, orc.problem_seed(3, rank, 0))
    x = orc.reconstruct(truth)
    orc.add_noise(x, 2, 1e-5)
    init = orc.random_model(dims, rank, orc.init_seed(3, rank, 0, 0))
    cfg = {"optimizer": optimizer, "als": {"max_sweeps": 30}, "gn": {"max_iters": 12, "cg_max_iters": 40}}
    probs = ck.DeviceProblem.loopback(dims, rank, world)

    def run(r, p):
        p.upload(slab_of(x, r, world))
        f, rep = p.optimize(cfg, init)
        return f, rep.to_json()

    got = on_ranks(probs, run)
    if optimizer == "als":
        _, recs, st = orc.als_optimize(x, init, orc.AlsConfig(max_sweeps=30))
    else:
        _, recs, st = orc.gn_optimize(x, init, orc.GnConfig(max_iters=12, cg_max_iters=40))
    for r in range(world):
        rr = got[r][1]["records"]
        assert len(rr) == len(recs) and got[r][1]["status"] == st, (r, len(rr), len(recs))
        for a, b in zip(rr, recs):
            assert a["cg_iters"] == b["cg_iters"] and a["lambda"] == b["lambda"]
            assert abs(a["residual"] - b["residual"]) < 1e-8


@pytest.mark.slow
@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_c5s_matches_unsharded(ck, world):
    """bench.py's multi-GPU configuration itself: the C5s tensor (order 4, s=200,
    R=200, noise 1e-4) generated per shard and sharded on mode 4 over `world`
    shards (the tile plans of the short local slabs, split-K front roots, the
    collectives), against the unsharded device run: every mode's MTTKRP at
    1e-11, one ALS sweep and one GN step at the trajectory tolerances."""
    dims, R = [200, 200, 200, 200], 200
    truth = ck.random_factors(dims, R, ck.problem_seed(0, R, 0))
    init = ck.random_factors(dims, R, ck.init_seed(0, R, 0, 0))
    ref = ck.DeviceProblem(dims, R)
    ref.generate(truth, noise_seed=1, noise_rel=1e-4)
    ref.set_factors(init)
    m_ref = [ref.mttkrp(n) for n in range(4)]
    xn2 = ref.norm2()
    step_ref, _ = ref.als_sweep(0.0)
    f_als = ref.get_factors()
    ref.set_factors(init)
    d_ref = ref.gn_step({}, xn2)
    f_gn = ref.get_factors()
    ref.close()
    probs = ck.DeviceProblem.loopback(dims, R, world)

    def run(r, p):
        p.generate(truth, noise_seed=1, noise_rel=1e-4)
        p.set_factors(init)
        m = [p.mttkrp(n) for n in range(4)]
        n2 = p.norm2()
        step, _ = p.als_sweep(0.0)
        fa = p.get_factors()
        p.set_factors(init)
        d = p.gn_step({}, n2)
        return m, n2, step, fa, d, p.get_factors()

    got = on_ranks(probs, run)
    for p in probs:
        p.close()
    for r in range(world):
        m, n2, step, fa, d, fg = got[r]
        for n in range(4):
            assert rel_err(m[n], m_ref[n]) < 1e-11, (r, n)
        assert abs(n2 - xn2) <= 1e-13 * xn2
        assert abs(step - step_ref) <= 1e-10 * step_ref
        assert vec_rel_err(fa, f_als) < 1e-10
        assert int(d["cg_iters"]) == int(d_ref["cg_iters"])
        assert abs(d["residual_after"] - d_ref["residual_after"]) < 1e-10
        assert vec_rel_err(fg, f_gn) < 1e-9
