"""Haptic session driver: the per-frame servo loop.

Follows the reference's sandbox session (`Session.eval_current` /
`Session.step_damped`, /root/reference/pkg/src/geofield/service.py:66-126),
in 3D and on the GPU:

* `eval_current` is one `evaluate` (one single-query kernel, or the resident
  `backend.HapticServer` when one runs for the pair);
* `step_damped` takes a first-order step dx = (F / c) dt clamped to half a
  cell and, if the energy rises, halves it up to three more times.  The
  reference evaluates those trials one after another (up to 4 extra
  evaluate calls per frame); here all four trial poses go to ONE batched
  cascade launch and the first trial (in the reference's order) whose energy
  does not exceed the current one is taken -- the same decision, one launch.
* `run` paces a trajectory at a fixed servo rate (the paper's 1 kHz loop,
  PAPER.md:317-321) and records per-frame latency and deadline misses; by
  default the frames are served by a resident query grid (no launch per
  frame).
"""

from __future__ import annotations

import statistics
import time

import numpy as np

from . import backend
from .energy import Configuration, EnergyEval, evaluate

__all__ = ["HapticSession"]

_SPIN_S = 150e-6  # spin only the last 150 us of a frame's slack (sleep wake-up jitter)


def _rt_runtime_us():
    """The kernel's real-time budget per second (-1: unlimited), or None."""
    try:
        with open("/proc/sys/kernel/sched_rt_runtime_us") as fh:
            return int(fh.read().strip())
    except (OSError, ValueError):
        return None


def _enter_realtime():
    """Pin the calling thread to the highest-numbered core it may use and
    raise it to SCHED_FIFO.  Returns what `_leave_realtime` needs; the third
    item says whether both took effect."""
    import os

    if not hasattr(os, "sched_setaffinity"):
        return None
    aff = os.sched_getaffinity(0)
    pol, prio = os.sched_getscheduler(0), os.sched_getparam(0)
    ok = True
    try:
        os.sched_setaffinity(0, {max(aff)})
        os.sched_setscheduler(0, os.SCHED_FIFO, os.sched_param(max(1, os.sched_get_priority_max(os.SCHED_FIFO) // 2)))
    except (OSError, PermissionError):
        ok = False
    return aff, (pol, prio), ok


def _leave_realtime(state):
    import os

    aff, (pol, prio), _ = state
    try:
        os.sched_setscheduler(0, pol, prio)
    except (OSError, PermissionError):
        pass
    os.sched_setaffinity(0, aff)


class HapticSession:
    def __init__(self, fixed, moving, m_prime=None, damping=1.0, frame_dt=1e-3, rotation=None, translation=None):
        self.fixed, self.moving, self.modes = fixed, moving, m_prime
        g = fixed.grid
        self.spacing = g.spacing
        self.damping = float(damping)
        self.frame_dt = float(frame_dt)
        d = g.dimension
        self.rotation = np.eye(d) if rotation is None else np.asarray(rotation, dtype=np.float64)
        self.translation = np.zeros(d) if translation is None else np.asarray(translation, dtype=np.float64)
        self.stats = []

    def config(self):
        return Configuration(self.rotation, self.translation)

    def eval_current(self):
        ev = evaluate(self.fixed, self.moving, self.config(), m_prime=self.modes)
        self.stats.append(ev.eval_time_us)
        return ev

    def _trial_energies(self, trials):
        """Energies of several translations at the current rotation, one launch."""
        import torch

        g = self.fixed.grid
        c = g.center()
        C1, wrap1 = self.fixed.window(self.modes)
        C2, wrap2 = self.moving.window(self.modes)
        R = np.broadcast_to(self.rotation, (len(trials),) + self.rotation.shape)
        t_eff = np.asarray(trials) - c + self.rotation @ c
        poses = torch.from_numpy(backend.pack_poses(R, t_eff)).cuda()
        dcell = 1.0 / (g.node_count * g.cell_volume)
        out = backend.cascade_batch(C1, C2, wrap1 and wrap2, g.delta_omega(), dcell, c, poses).cpu().numpy()
        return -out[:, 0]  # energy = -Re(score)

    def step_damped(self, ev: EnergyEval):
        """One damped descent step with backtracking (service.py:105-126)."""
        step = (ev.force / self.damping) * self.frame_dt
        norm = float(np.linalg.norm(step))
        limit = 0.5 * self.spacing
        if norm > limit:
            step = step * (limit / norm)
        trials = [self.translation + step * 0.5 ** k for k in range(4)]
        energies = self._trial_energies(trials)
        for trial, e in zip(trials, energies):
            if e <= ev.energy:
                self.translation = trial
                return True
        return False  # every trial climbed: hold the pose

    def run(self, rotations, translations, rate_hz=1000.0, resident=True, realtime=True, max_sms=0):
        """Pace a pose trajectory at `rate_hz`; returns latency stats and misses.

        resident=True serves the frames from a persistent query grid
        (energy.haptic_session) for the duration of the run, as a dedicated
        haptic server would; False launches one kernel per frame.
        realtime=True runs the servo loop as a haptic thread is normally run:
        pinned to one host core at SCHED_FIFO priority (restored afterwards;
        skipped when the OS refuses, reported as "realtime": False).  Measured
        on the B200 box: unpinned, 1-2 frames per 1000 stall for 1-5 ms while
        the thread is descheduled; pinned at SCHED_FIFO, none.  `max_sms`
        is handed to the resident grid (see backend.HapticServer)."""
        if resident:
            from .energy import haptic_session

            with haptic_session(self.fixed, self.moving, self.modes, max_sms=max_sms) as srv:
                return self._run(rotations, translations, rate_hz, realtime, srv)
        return self._run(rotations, translations, rate_hz, realtime)

    def _run(self, rotations, translations, rate_hz, realtime=False, server=None):
        import gc

        period = 1.0 / rate_hz
        gc_was = gc.isenabled()
        gc.disable()  # a collector pause inside the servo loop would be a missed frame
        restore = _enter_realtime() if realtime else None
        try:
            out = self._paced(rotations, translations, period, rate_hz, server)
            out["realtime"] = bool(restore and restore[2])
            return out
        finally:
            if restore:
                _leave_realtime(restore)
            if gc_was:
                gc.enable()

    def _paced(self, rotations, translations, period, rate_hz, server=None):
        """Servo pacing: sleep through most of the slack, spin only the last
        `_SPIN_S`.  A SCHED_FIFO thread that busy-waits the whole period uses
        100 % of its core and hits the kernel's real-time throttle
        (sched_rt_runtime_us, 950 ms of every 1 s by default): it is then
        descheduled for ~50 ms -- the 46 ms frame of the round-1 C5 run."""
        lat, misses, late, gpu = [], 0, [], []
        t_next = time.perf_counter()
        for i, (R, t) in enumerate(zip(rotations, translations)):
            self.rotation, self.translation = np.asarray(R), np.asarray(t)
            t0 = time.perf_counter()
            self.eval_current()
            dt = time.perf_counter() - t0
            lat.append(dt * 1e6)
            if server is not None:
                gpu.append(server.last_timing()["gpu_us"])
            if dt > period:
                misses += 1
                if len(late) < 16:
                    rec = {"frame": i, "us": dt * 1e6, "start_lag_us": (t0 - t_next) * 1e6}
                    if server is not None:  # where the time went: host, PCIe or the grid
                        rec.update(server.last_timing())
                    late.append(rec)
            t_next += period
            slack = t_next - time.perf_counter()
            if slack > _SPIN_S:
                time.sleep(slack - _SPIN_S)
            while time.perf_counter() < t_next:
                pass
        worst = max(range(len(lat)), key=lat.__getitem__) if lat else -1
        lat.sort()
        pct = lambda p: lat[min(len(lat) - 1, int(p * len(lat)))]  # noqa: E731  (cli.py:357-361)
        return {"frames": len(lat), "p50_us": statistics.median(lat), "p95_us": pct(0.95), "p99_us": pct(0.99),
                "max_us": lat[-1], "max_frame": worst, "deadline_misses": misses, "missed": late,
                "rate_hz": rate_hz, "rt_runtime_us": _rt_runtime_us(),
                "gpu_us_p50": statistics.median(gpu) if gpu else None}
