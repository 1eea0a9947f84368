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


def test_landscape_export_runs_beside_a_session():
    """SPEC.md:348 / service.py:305-318: a landscape export from a worker
    thread completes while a 1 kHz session serves frames from a resident
    grid held to part of the GPU (max_sms), and the frames stay inside the
    1 ms budget at p99."""
    import threading

    import torch

    from paper_1711_05017_b200.descriptor import SampleGrid
    from paper_1711_05017_b200.energy import score_field_device

    n, w = 256, 64
    g = SampleGrid(3, (n,) * 3, (-2.0,) * 3, 4.0 / n)
    rng = np.random.default_rng(5)

    class _A:
        def __init__(self, win, wrap):
            self.grid, self._w = g, (win, wrap)

        def window(self, m_prime=None):
            return self._w

        def max_modes(self):
            return w ** 3

    def win(side):
        k2 = (np.arange(side) - side // 2).astype(np.float64) ** 2
        amp = 1.0 / (1.0 + k2[:, None, None] + k2[None, :, None] + k2[None, None, :])
        return backend.DeviceWindow((rng.standard_normal((side,) * 3) + 1j * rng.standard_normal((side,) * 3)) * amp)

    q1, q2 = win(w), win(w)  # the session's truncated windows
    f1, f2 = win(n), win(n)  # full spectra for the 256^3 export
    frames = 1000
    th = np.linspace(0.0, np.pi, frames)
    R = np.stack([np.array([[np.cos(a), -np.sin(a), 0], [np.sin(a), np.cos(a), 0], [0, 0, 1.0]]) for a in th])
    t = np.stack([np.array([0.0, 0.0, 0.2 * a]) for a in th])
    done = {}

    def export():
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            land = score_field_device(_A(f1, True), _A(f2, True), R[frames // 2], None, precision=32)
            stream.synchronize()
        done["ok"] = bool(torch.isfinite(land.abs()).all())

    sess = HapticSession(_A(q1, False), _A(q2, False), None)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    worker = threading.Thread(target=export)
    worker.start()
    run = sess.run(R, t, rate_hz=1000.0, max_sms=sms * 3 // 4)
    worker.join(timeout=60)
    assert not worker.is_alive() and done.get("ok"), "the export did not finish beside the session"
    assert run["frames"] == frames and run["p99_us"] < 1000.0, run
