"""Single-rank GPU runs of the multi-GPU paths (the decomposition itself is
tested at world size 2 with gloo in test_parallel.py)."""

import numpy as np
import pytest

import oracle
from paper_1711_05017_b200 import parallel
from paper_1711_05017_b200.descriptor import ComplexField, SampleGrid
from paper_1711_05017_b200.energy import Configuration, PartAsset, evaluate, score_field

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def assets():
    rng = np.random.default_rng(4)
    g = SampleGrid(3, (32, 32, 32), (-1.6, -1.6, -1.6), 0.1)
    mk = lambda: ComplexField(g, rng.normal(size=g.node_count) + 1j * rng.normal(size=g.node_count))  # noqa: E731
    return PartAsset.from_field("a", mk()), PartAsset.from_field("b", mk(), movable=True)


def test_pose_sweep_matches_evaluate(assets):
    a1, a2 = assets
    Rs, ts = oracle.bench_poses(40, 0.5, seed=1)
    for prec, tol in (("fp64", 1e-10), ("fp32", 1e-4)):
        out = parallel.pose_sweep(a1, a2, Rs, ts, m_prime=16 ** 3, precision=prec)
        assert out.shape == (40, 7)
        from paper_1711_05017_b200 import backend

        backend.set_precision(prec)
        try:
            for i in range(0, 40, 7):
                ev = evaluate(a1, a2, Configuration(Rs[i], ts[i]), 16 ** 3)
                assert abs(out[i, 0] - ev.score) <= tol * max(abs(ev.score), 1e-3)
                np.testing.assert_allclose(out[i, 1:4].real, ev.force, rtol=tol, atol=tol * np.max(np.abs(ev.force)))
        finally:
            backend.set_precision("fp32")


@pytest.mark.parametrize("mp", [16 ** 3, None])
def test_score_field_slab_equals_score_field(assets, mp):
    a1, a2 = assets
    R = oracle.quat_rotation([0.7, -0.3, 0.2, 0.4])
    full = score_field(a1, a2, R, mp).values.reshape(32, 32, 32)
    slab = parallel.score_field_slab(a1, a2, R, mp).cpu().numpy()
    np.testing.assert_allclose(slab, full, atol=1e-11 * np.max(np.abs(full)))
