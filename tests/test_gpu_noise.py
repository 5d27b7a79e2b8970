"""On-device tensor generation (generators.cpp:78-94,
kruskal.cpp:67-92) against the CPU restatement, bit for bit.

reconstruct(truth) follows the reference's per-entry order with separate
multiply and add; the keyed noise (stream 0x4E01, keyed_noise.cuh) uses a
portable log/cos and a column-block norm order, so the device tensor equals
oracle.reconstruct + oracle.add_noise exactly - including the odd-row-stride
(padded) layout and BASELINE config 2 at its full size.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ck():
    from paper_1910_12331_b200 import cpkit
    cpkit.load()
    return cpkit


def test_noise_draws_match_cpu(orc):
    # the CPU restatement of the portable Box-Muller stays close to rng::gaussian
    for g in range(0, 5000, 37):
        a, b = orc.noise_gaussian(11, g), orc.gaussian(11, 0x4E01, g)
        assert abs(a - b) <= 4e-15 * max(1.0, abs(b)), (g, a, b)  # a few ulp from glibc log/cos


@pytest.mark.parametrize("dims,rank,rel", [
    ([13, 11, 10], 3, 1e-3),
    ([5, 7, 9, 3], 2, 1e-2),     # odd back extent: padded row stride on the device
    ([6, 5, 4, 3, 7], 4, 1e-4),  # order 5
    ([50, 50, 50], 5, 1e-6),
])
def test_generated_tensor_bitwise(orc, ck, dims, rank, rel):
    truth = orc.random_model(dims, rank, orc.problem_seed(0, rank, 0))
    p = ck.DeviceProblem(dims, rank)
    p.generate(truth, noise_seed=5, noise_rel=rel)
    got = p.download()
    x = orc.reconstruct(truth)
    scale, nx, ne = orc.add_noise(x, 5, rel)
    assert np.array_equal(got, x), np.max(np.abs(got - x))
    assert abs(np.linalg.norm(got - orc.reconstruct(truth)) / np.sqrt(nx) - rel) < 1e-12


def test_generated_noiseless_bitwise(orc, ck):
    dims, rank = [17, 9, 12], 4
    truth = orc.random_model(dims, rank, 77, kind="gaussian")
    p = ck.DeviceProblem(dims, rank)
    p.generate(truth)
    assert np.array_equal(p.download(), orc.reconstruct(truth))


@pytest.mark.slow
def test_c2_generation_bitwise_full_size(orc, ck):
    """BASELINE config 2 (s=400, R=100, noise 1e-6 ||X||): 512 MB, device vs CPU bit for bit."""
    dims, rank = [400, 400, 400], 100
    orc.set_threads(16)
    truth = orc.random_model(dims, rank, orc.problem_seed(0, rank, 0))
    p = ck.DeviceProblem(dims, rank)
    p.generate(truth, noise_seed=1, noise_rel=1e-6)
    got = p.download()
    p.close()
    x = orc.reconstruct(truth)
    orc.add_noise(x, 1, 1e-6)
    assert np.array_equal(got, x)
