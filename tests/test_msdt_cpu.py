"""CPU check of the order-3 multi-sweep dimension tree as an
algorithm: a numpy restatement of DeviceProblem::mttkrp_msdt's root rotation
(P_c = X x_c A_c, reused for the next two mode updates, c = 2, 1, 0, ...)
drives ALS sweeps that must track the oracle's reference-tree sweeps
(als.cpp:22-52, mttkrp.cpp:160-189) at roundoff level, with 3 first-level
contractions per 2 sweeps. The device implementation is checked against the
oracle in tests/test_gpu_parity.py::test_als_msdt_tracks_oracle."""
import numpy as np
import pytest

from tests.helpers import vec_rel_err


class MsdtAls:
    """Host model of the device's order-3 ALS mode loop with the MSDT cache."""

    def __init__(self, x, factors):
        self.x = x
        self.a = [f.copy() for f in factors]
        self.root = None  # (c, P_c) with P_c kept modes ascending, rank last
        self.contractions = 0

    def _mttkrp(self, n):
        if self.root is None or self.root[0] == n:
            c = (n + 2) % 3  # updated neither now nor next
            p = np.tensordot(self.x, self.a[c], axes=([c], [0]))  # kept modes ascending, then r
            self.root = (c, p)
            self.contractions += 1
        c, p = self.root
        kept = [m for m in range(3) if m != c]
        other = kept[1] if kept[0] == n else kept[0]
        # contract the other kept index with its (current) factor, Hadamard in r
        return np.einsum("ijr,jr->ir", p, self.a[other]) if kept[0] == n else \
            np.einsum("jir,jr->ir", p, self.a[other])

    def sweep(self, lam):
        step = 0.0
        grams = [f.T @ f for f in self.a]
        for n in range(3):
            g = np.ones_like(grams[0])
            for m in range(3):
                if m != n:
                    g = g * grams[m]
            m_n = self._mttkrp(n)
            new = np.linalg.solve(g + lam * np.eye(g.shape[0]), m_n.T).T
            step += np.linalg.norm(new - self.a[n])
            self.a[n] = new
            grams[n] = new.T @ new
            if self.root is not None and self.root[0] == n:
                self.root = None  # note_factor_update(n) drops the root that kept A_n
        return step


@pytest.mark.parametrize("dims,rank", [([6, 5, 4], 3), ([9, 7, 8], 4), ([12, 5, 10], 6)])
def test_msdt_rotation_tracks_reference_tree(orc, dims, rank):
    t = orc.random_model(dims, rank, 3)
    x = orc.reconstruct(t) + 1e-3 * np.random.default_rng(5).standard_normal(dims)
    f = orc.random_model(dims, rank, 4)
    model = MsdtAls(x, f)
    counts = []
    for sweep in range(6):
        c0 = model.contractions
        step = model.sweep(1e-4)
        f, step_ref, cnt_ref, _ = orc.als_sweep(x, f, 1e-4)
        counts.append(model.contractions - c0)
        assert cnt_ref == 2  # the reference tree: two first-level contractions per sweep
        assert abs(step - step_ref) <= 1e-9 * step_ref, sweep
        assert vec_rel_err(model.a, f) < 1e-10, sweep
    assert counts == [2, 1, 2, 1, 2, 1]
