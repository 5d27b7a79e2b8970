"""World-size-2 gloo tests of the last-mode sharding plan, on CPU.

The B200 library shards the tensor along its last mode (cpkit_dev_shard_range),
all-reduces the s_n x R MTTKRP partials of modes n < N-1, all-gathers the slab
rows of M^(N-1) and all-reduces ||X||^2 (solver.cu second_level_back/front,
norm2). These tests run that exact plan on two gloo ranks with the CPU oracle
computing each rank's local pieces, and check the reassembled results (and a
full sharded ALS sweep) against the unsharded oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, port, dims, rank_r, q):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from oracle import oracle as orc
        from paper_1910_12331_b200 import cpkit
        N = len(dims)
        lo, hi = cpkit.shard_range(dims[-1], rank, WORLD)
        x = np.random.default_rng(5).standard_normal(dims)
        f = orc.random_model(dims, rank_r, 7, kind="gaussian")
        x_loc = np.ascontiguousarray(x[..., lo:hi])
        f_loc = f[:-1] + [np.ascontiguousarray(f[-1][lo:hi])]
        errs = {}
        # ||X||^2: local partial + all-reduce
        t = torch.tensor([orc.norm2(x_loc)], dtype=torch.float64)
        dist.all_reduce(t)
        errs["norm2"] = abs(t.item() - orc.norm2(x)) / orc.norm2(x)
        # M^(n), n < N-1: local partial over the slab + all-reduce
        for n in range(N - 1):
            m = torch.from_numpy(orc.mttkrp_naive(x_loc, f_loc, n))
            dist.all_reduce(m)
            ref = orc.mttkrp_naive(x, f, n)
            errs[f"m{n}"] = float(np.linalg.norm(m.numpy() - ref) / np.linalg.norm(ref))
        # M^(N-1): complete local rows, all-gather (equal slabs)
        ml = torch.from_numpy(orc.mttkrp_naive(x_loc, f_loc, N - 1))
        parts = [torch.empty_like(ml) for _ in range(WORLD)]
        dist.all_gather(parts, ml)
        full = torch.cat(parts).numpy()
        ref = orc.mttkrp_naive(x, f, N - 1)
        errs["mlast"] = float(np.linalg.norm(full - ref) / np.linalg.norm(ref))
        # one sharded ALS sweep (als.cpp:22-52): solves replicated on every rank
        a = [fi.copy() for fi in f]
        for n in range(N):
            aloc = a[:-1] + [np.ascontiguousarray(a[-1][lo:hi])]
            if n < N - 1:
                m = torch.from_numpy(orc.mttkrp_naive(x_loc, aloc, n))
                dist.all_reduce(m)
                m = m.numpy()
            else:
                ml = torch.from_numpy(orc.mttkrp_naive(x_loc, aloc, n))
                parts = [torch.empty_like(ml) for _ in range(WORLD)]
                dist.all_gather(parts, ml)
                m = torch.cat(parts).numpy()
            gam = np.ones((rank_r, rank_r))
            for mm in range(N):
                if mm != n:
                    gam = gam * orc.gram(a[mm])
            a[n] = orc.spd_solve(gam, m, 1e-3)
        ref_f, _, _, _ = orc.als_sweep(x, f, 1e-3)
        errs["als"] = max(float(np.linalg.norm(u - v) / np.linalg.norm(v)) for u, v in zip(a, ref_f))
        q.put((rank, lo, hi, errs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,rank_r", [([6, 5, 8], 3), ([4, 3, 5, 6], 2)])
def test_sharded_plan_matches_unsharded_oracle(dims, rank_r):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, dims, rank_r, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    assert out[0][1] == 0 and out[-1][2] == dims[-1] and out[0][2] == out[1][1]  # slabs tile the mode
    for _, _, _, errs in out:
        for k, v in errs.items():
            assert v < 1e-12, (k, v)


def test_shard_range_balanced():
    from paper_1910_12331_b200 import cpkit
    for extent in (1, 7, 400, 401):
        for world in (1, 2, 3, 8):
            spans = [cpkit.shard_range(extent, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == extent
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
