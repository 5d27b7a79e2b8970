"""CPKT1 ingest streamed to the device (tensor.cpp:197-239).

cpkit_dev_load_tensor reads whole last-mode rows in chunks into two pinned
staging buffers while the previous chunk crosses to HBM, copies only the
shard's slab columns, and runs read_tensor's finiteness check on the device.
The loaded tensor equals the file bit for bit on every layout (order-3
permuted copies, order >= 4 X^T copy, odd padded rows, last-mode shards), and
the reference's error codes are kept (bad magic / truncated: parse; NaN,
wrong extents: invalid argument; missing file: io).
"""
import threading

import numpy as np
import pytest

from tests.helpers import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ck():
    from paper_1910_12331_b200 import cpkit
    cpkit.load()
    return cpkit


@pytest.mark.parametrize("dims,rank", [([30, 20, 25], 4), ([9, 8, 7, 6], 3), ([5, 7, 9, 3], 2), ([300, 200, 150], 8)])
def test_streamed_load_bitwise(orc, ck, tmp_path, dims, rank):
    x = np.random.default_rng(sum(dims)).standard_normal(dims)
    path = str(tmp_path / "x.cpkt")
    ck.Tensor.create(x).save(path)
    p = ck.DeviceProblem(dims, rank)
    p.load_file(path)
    assert np.array_equal(p.download(), x)
    f = orc.random_model(dims, rank, 3, kind="gaussian")
    p.set_factors(f)
    ref, _ = orc.mttkrp_tree_all(x, f)  # the layout copies were built from the streamed tensor
    for n in range(len(dims)):
        assert rel_err(p.mttkrp(n), ref[n]) < 1e-11


def test_streamed_load_errors(ck, tmp_path):
    dims = [4, 5, 6]
    x = np.random.default_rng(1).standard_normal(dims)
    good = str(tmp_path / "g.cpkt")
    ck.Tensor.create(x).save(good)
    p = ck.DeviceProblem(dims, 2)
    with pytest.raises(ck.CpkitError) as e:
        p.load_file(str(tmp_path / "missing.cpkt"))
    assert e.value.status == "io_error"
    raw = open(good, "rb").read()
    trunc = tmp_path / "t.cpkt"
    trunc.write_bytes(raw[:-8])
    with pytest.raises(ck.CpkitError) as e:
        p.load_file(str(trunc))
    assert e.value.status == "parse_error"
    bad = tmp_path / "b.cpkt"
    bad.write_bytes(b"NOPE1" + raw[5:])
    with pytest.raises(ck.CpkitError) as e:
        p.load_file(str(bad))
    assert e.value.status == "parse_error"
    nan = tmp_path / "n.cpkt"
    arr = bytearray(raw)
    arr[-8:] = np.array([np.nan]).tobytes()
    nan.write_bytes(bytes(arr))
    with pytest.raises(ck.CpkitError) as e:
        p.load_file(str(nan))
    assert e.value.status == "invalid_argument"
    other = ck.DeviceProblem([4, 5, 7], 2)
    with pytest.raises(ck.CpkitError) as e:
        other.load_file(good)
    assert e.value.status == "invalid_argument"


@pytest.mark.parametrize("world", [2, 4])
def test_streamed_load_sharded(ck, tmp_path, world):
    dims = [14, 12, 8]
    x = np.random.default_rng(world).standard_normal(dims)
    path = str(tmp_path / "s.cpkt")
    ck.Tensor.create(x).save(path)
    probs = ck.DeviceProblem.loopback(dims, 3, world)
    out = [None] * world

    def run(r):
        probs[r].load_file(path)
        out[r] = probs[r].download()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    s = dims[-1] // world
    for r in range(world):
        assert np.array_equal(out[r], x[..., r * s:(r + 1) * s])


def test_decompose_from_loaded_tensor(orc, ck, tmp_path):
    """cpkit_tensor_load reads straight into the tensor's (pinned) storage and
    cpkit_decompose uploads it without another host copy: same result as from
    cpkit_tensor_create."""
    dims, R = [20, 18, 16], 3
    truth = orc.random_model(dims, R, 8)
    x = orc.reconstruct(truth)
    path = str(tmp_path / "d.cpkt")
    ck.Tensor.create(x).save(path)
    cfg = {"optimizer": "als", "rank": R, "seed": 2, "als": {"max_sweeps": 20}}
    m1, r1 = ck.decompose(ck.Tensor.load_file(path), cfg)
    m2, r2 = ck.decompose(ck.Tensor.create(x), cfg)
    strip = lambda rep: [{k: v for k, v in rec.items() if k != "seconds"} for rec in rep.to_json()["records"]]
    assert strip(r1) == strip(r2)
    for a, b in zip(m1.factors(), m2.factors()):
        assert np.array_equal(a, b)
