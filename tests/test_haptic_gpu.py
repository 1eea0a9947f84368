"""Haptic session driver: the batched backtracking step makes exactly the
decision of the reference's sequential loop (service.py:105-126)."""

import numpy as np
import pytest

from paper_1711_05017_b200 import backend, scenes
from paper_1711_05017_b200.descriptor import KernelSpec, affinity_field
from paper_1711_05017_b200.energy import Configuration, PartAsset, evaluate
from paper_1711_05017_b200.haptic import HapticSession

pytestmark = pytest.mark.gpu


def sequential_step(fixed, moving, modes, R, t, ev, damping, dt, spacing):
    step = (ev.force / damping) * dt
    norm = float(np.linalg.norm(step))
    if norm > 0.5 * spacing:
        step = step * (0.5 * spacing / norm)
    for _ in range(4):
        trial = t + step
        if evaluate(fixed, moving, Configuration(R, trial), modes).energy <= ev.energy:
            return trial
        step = 0.5 * step
    return t


def test_step_damped_matches_sequential_backtracking():
    peg = scenes.get_scene("peg3d")
    g = peg.grid(16)
    a1 = PartAsset.from_field("f", affinity_field(peg.fixed, g, KernelSpec()), solid_box=peg.fixed.bbox)
    a2 = PartAsset.from_field("m", affinity_field(peg.moving, g, KernelSpec()), movable=True, solid_box=peg.moving.bbox)
    backend.set_precision("fp64")
    try:
        rng = np.random.default_rng(3)
        for k in range(6):
            t0 = rng.uniform(-0.4, 0.4, 3)
            s = HapticSession(a1, a2, 512, damping=0.05, frame_dt=1e-3, translation=t0)
            ev = s.eval_current()
            want = sequential_step(a1, a2, 512, np.eye(3), t0, ev, 0.05, 1e-3, g.spacing)
            s.step_damped(ev)
            np.testing.assert_allclose(s.translation, want, rtol=0, atol=1e-15)
        import os

        aff, pol = os.sched_getaffinity(0), os.sched_getscheduler(0)
        stats = s.run([np.eye(3)] * 20, [t0] * 20, rate_hz=2000.0)
        assert stats["frames"] == 20 and stats["p99_us"] > 0
        assert 0 <= stats["max_frame"] < 20 and isinstance(stats["realtime"], bool)
        # the servo thread's affinity and scheduling policy are restored after the run
        assert os.sched_getaffinity(0) == aff and os.sched_getscheduler(0) == pol
    finally:
        backend.set_precision("fp32")
