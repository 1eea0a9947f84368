"""Headline benchmark: the haptic single-query loop (BASELINE.json configs[1]).

Workload (N=1): "low-clearance peg-in-hole 128^3, K=32, single-query haptic
latency loop on 1 B200": a 128^3 grid, truncation K=32 (window side w=2K=64,
m'=262,144 retained modes), energy + force + torque per query.  One step =
one 1,000-query segment of a jittered insertion trajectory (R near I,
sigma_theta = 0.5 deg; t sliding along z with sigma_t = h/4), issued as
1,000 serial single-query launches.

  value   queries/s of the device-resident loop (windows and poses already in
          HBM; one kernel launch per query, stream-ordered), CUDA events.
  e2e     queries/s through the reference-facing operator call
          (backend.cascade: host pose in, host complex128[7] out, the
          per-query H2D/D2H inside the timed region), with p50/p95/p99 per
          query as cmd_bench defines them (cli.py:357-361).
  roofline  the cascade kernel against the FP32 FMA pipe measured live on
          this GPU (MEASURED_PEAKS.json has no FP32 figure); algorithmic work
          240 FP32 flops per live retained mode.
  cpu_baseline  the reference's own compiled kernel (_core.cascade_3d built
          from /root/reference into oracle/_ref) on the same windows, 1 core
          (it is single-threaded by design, backend.py:153-164).

--impl reference runs the reference kernel with every host core (a thread
pool over poses; _core.cascade_3d releases the GIL) on the same config.

Multi-GPU: the single haptic query does not shard:
`--gpus N` runs N independent replicas, one per rank, and value/e2e are the
whole-job totals (max-over-ranks time).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GRID_N = 128
K_TRUNC = 32
W = 2 * K_TRUNC
DOMAIN = 3.46  # grid_for_pair domain of the C1/C2 peg pair
QUERIES_PER_STEP = 1000
SEED = 20260814


def synthetic_windows(w, seed=SEED):
    """CN(0,1)(1+|k|^2)^-1 windows (SURVEY.md 8(d) micro-benchmark law)."""
    rng = np.random.default_rng(seed)
    k = np.stack(np.meshgrid(*[np.arange(w) - w // 2] * 3, indexing="ij"), axis=-1)
    amp = 1.0 / (1.0 + np.sum(k * k, axis=-1))
    C1 = (rng.normal(size=(w,) * 3) + 1j * rng.normal(size=(w,) * 3)) * amp
    C2 = (rng.normal(size=(w,) * 3) + 1j * rng.normal(size=(w,) * 3)) * amp
    return C1, C2


def grid_params(frozen=False):
    h = DOMAIN / GRID_N
    origin = -0.5 * DOMAIN
    center = np.full(3, origin + h * (GRID_N // 2))
    dom = np.full(3, 1.0 / (GRID_N * h))
    dcell = 1.0 / (GRID_N ** 3 * h ** 3)
    if frozen:  # per-grid immutables, as energy._grid_constants hands them to every query
        center.flags.writeable = False
        dom.flags.writeable = False
    return h, center, dom, dcell


def axis_rot(axis, ang):
    c, s = np.cos(ang), np.sin(ang)
    R = np.eye(3)
    i, j = [(1, 2), (0, 2), (0, 1)][axis]
    R[i, i], R[i, j], R[j, i], R[j, j] = c, -s, s, c
    return R


def trajectory(n, seed):
    """Jittered insertion path: R ~ I (0.5 deg jitter), t_z from 0.4 to 0."""
    h, center, _, _ = grid_params()
    rng = np.random.default_rng(seed)
    s = np.linspace(0.0, 1.0, n)
    Rs, ts = [], []
    for k in range(n):
        j = np.deg2rad(0.5) * rng.normal(size=3)
        R = axis_rot(0, j[0]) @ axis_rot(1, j[1]) @ axis_rot(2, j[2])
        t = np.array([0.0, 0.0, 0.4 * (1.0 - s[k])]) + (h / 4) * rng.normal(size=3)
        Rs.append(R)
        ts.append(t)
    Rs, ts = np.asarray(Rs), np.asarray(ts)
    t_eff = ts - center + Rs @ center  # energy.py:177
    return Rs, ts, t_eff


def live_fraction(Rs, w, sample=8):
    """Share of retained modes whose trilinear footprint touches the window
    (the rest contribute exact zeros), averaged over a few poses."""
    k = np.stack(np.meshgrid(*[np.arange(w) - w // 2] * 3, indexing="ij"), axis=-1).reshape(-1, 3)
    fr = []
    for R in Rs[:: max(1, len(Rs) // sample)][:sample]:
        u = -(k @ R) + w // 2
        fl = np.floor(u)
        ok = np.all((fl >= -1) & (fl <= w - 1), axis=1)
        fr.append(ok.mean())
    return float(np.mean(fr))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    return world, rank, local


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ---------------------------------------------------------------------------
# synthetic poses exactly as the reference's cmd_bench draws them
# (cli.py:336-346): per pose q ~ N(0, I4) normalised to a rotation, then
# t ~ U(-span, span)^3, in that order


def cmd_bench_poses(n, span, seed=0):
    rng = np.random.default_rng(seed)
    Rs, ts = [], []
    for _ in range(n):
        w, x, y, z = rng.normal(size=4)
        nrm = np.sqrt(w * w + x * x + y * y + z * z)
        w, x, y, z = w / nrm, x / nrm, y / nrm, z / nrm
        Rs.append([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                   [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                   [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])
        ts.append(rng.uniform(-span, span, 3))
    return np.asarray(Rs), np.asarray(ts)


# ---------------------------------------------------------------------------
# CPU baseline (the reference's compiled kernel, oracle/_ref)


def reference_core():
    import oracle

    core = oracle.ref_core()
    if core is None:
        raise RuntimeError("oracle/_ref not built (make -C oracle ref in the build container)")
    return core


def cpu_reference_rate(C1, C2, Rs, t_eff, threads, budget_s):
    """Queries/s of _core.cascade_3d on `threads` host threads for ~budget_s."""
    from concurrent.futures import ThreadPoolExecutor

    core = reference_core()
    _, center, dom, dcell = grid_params()
    C1 = np.ascontiguousarray(C1)
    C2 = np.ascontiguousarray(C2)

    def one(i):
        return core.cascade_3d(C1, C2, False, dom[0], dom[1], dom[2], dcell, np.ascontiguousarray(Rs[i]),
                               np.ascontiguousarray(t_eff[i]), center)

    one(0)  # warm
    t0 = time.perf_counter()
    one(1)
    per = time.perf_counter() - t0
    n = max(threads, int(budget_s * threads / max(per, 1e-6)))
    n = min(n, len(Rs))
    t0 = time.perf_counter()
    if threads == 1:
        for i in range(n):
            one(i)
    else:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(one, range(n)))
    dt = time.perf_counter() - t0
    return n / dt, n, dt


def run_reference_arm(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    C1, C2 = synthetic_windows(W)
    Rs, _, t_eff = trajectory(max(4096, QUERIES_PER_STEP), SEED)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_rate(C1, C2, Rs, t_eff, threads, 0.5)
    rates, samples = [], []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        r, n, dt = cpu_reference_rate(C1, C2, Rs, t_eff, threads, args.ref_seconds)
        rates.append(r)
        samples.append(n)
    total = time.perf_counter() - t_all
    value = float(np.sum(samples) / total)
    line = {
        "impl": "reference", "metric": "pose queries/sec (energy+force+torque) at K=32, 128^3, single-query loop",
        "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 haptic query loop: 128^3 grid, K=32 (w=64, m'=262144)",
                   "grid": GRID_N, "K": K_TRUNC, "w": W, "m_prime": W ** 3},
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": threads, "kind": "reference",
                         "sample": f"{int(np.mean(samples))} poses of the trajectory per step, "
                                   f"_core.cascade_3d on a {threads}-thread pool"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# engine arm


def run_engine(args):
    import torch

    world, rank, local = dist_setup()
    from paper_1711_05017_b200 import _lib, backend

    _lib.ensure_device(local)
    prec = args.precision
    h, center, dom, dcell = grid_params(frozen=True)
    C1, C2 = synthetic_windows(W)
    W1, W2 = backend.DeviceWindow(C1), backend.DeviceWindow(C2)
    n_total = QUERIES_PER_STEP * (args.steps + args.warmup)
    Rs, ts, t_eff = trajectory(n_total, SEED + rank)
    poses = torch.from_numpy(backend.pack_poses(Rs, t_eff)).cuda()
    out = torch.empty((n_total, 14), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    flush = torch.empty(int(256 * 2 ** 20) // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    def step(i):
        sl = slice(i * QUERIES_PER_STEP, (i + 1) * QUERIES_PER_STEP)
        backend.cascade_batch(W1, W2, False, dom, dcell, center, poses[sl], out=out[sl], precision=prec,
                              serial=True)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()

    # ---- device-resident timed region: K steps, per-step events, L2 flushed between steps
    barrier(world)
    torch.cuda.synchronize()
    step_ms = []
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(args.warmup + k)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    barrier(world)
    local_total_ms = float(np.sum(step_ms))
    total_ms = max_over_ranks(local_total_ms, world)
    queries = QUERIES_PER_STEP * args.steps * world
    value = queries / (total_ms * 1e-3)
    kernel_us = 1e3 * local_total_ms / (QUERIES_PER_STEP * args.steps)

    # ---- e2e through the operator call with host buffers (backend.cascade:
    # host pose in, host complex128[7] out).  Haptic-loop mode: a persistent
    # query grid (backend.HapticServer) answers each call -- no launch per
    # query; the one-shot launch path is reported beside it.
    Re, _, te = trajectory(args.e2e_queries + 50, SEED + 7 + rank)

    def e2e_loop():
        lat = []
        for i in range(50):
            backend.cascade(W1, W2, False, dom, dcell, Re[i], te[i], center, precision=prec)
        barrier(world)
        t0 = time.perf_counter()
        for i in range(50, 50 + args.e2e_queries):
            q0 = time.perf_counter_ns()
            backend.cascade(W1, W2, False, dom, dcell, Re[i], te[i], center, precision=prec)
            lat.append((time.perf_counter_ns() - q0) / 1e3)
        dt = time.perf_counter() - t0
        barrier(world)
        return sorted(lat), max_over_ranks(dt, world)

    # headline: the haptic-session path (energy.haptic_session / backend.HapticServer:
    # a resident query grid, pose in and result out through self-tagged
    # host-mapped slots); the one-shot launch per call is reported beside it
    with backend.HapticServer(W1, W2, False, dom, dcell, center, precision=prec):
        lat, e2e_s = e2e_loop()
    lat1, dt1 = e2e_loop()  # no server: one single-query kernel launch per call
    e2e_value = args.e2e_queries * world / e2e_s

    # the float64 engine (the reference's own tolerances) on the same loop, for reference
    fp64_mode = None
    if prec == "fp32":
        def e2e64():
            lat64 = []
            for i in range(50):
                backend.cascade(W1, W2, False, dom, dcell, Re[i], te[i], center, precision="fp64")
            for i in range(50, 50 + args.e2e_queries):
                q0 = time.perf_counter_ns()
                backend.cascade(W1, W2, False, dom, dcell, Re[i], te[i], center, precision="fp64")
                lat64.append((time.perf_counter_ns() - q0) / 1e3)
            return sorted(lat64)

        with backend.HapticServer(W1, W2, False, dom, dcell, center, precision="fp64"):
            l64 = e2e64()
        fp64_mode = {"e2e_p50_us": statistics.median(l64), "e2e_p99_us": l64[min(len(l64) - 1, int(0.99 * len(l64)))],
                     "e2e_queries_per_s": 1e6 / float(np.mean(l64)),
                     "note": "same session loop in the float64 engine (reference tolerances 1e-9..1e-12)"}

    def pct(xs, p):
        return xs[min(len(xs) - 1, int(p * len(xs)))]

    # ---- roofline: cascade kernel vs the FP32 FMA pipe measured here
    import ctypes

    peak = ctypes.c_double(0.0)
    _lib.check(_lib.LIB.gf_measure_fma_peak(64 if prec == "fp64" else 32, ctypes.byref(peak)))
    live = live_fraction(Rs, W)
    flops = 240.0 * live * W ** 3
    achieved = flops / (kernel_us * 1e-6) / 1e12

    stages = {} if args.no_stages else measure_stages(args, rank, world, peak.value)

    cpu = None
    if rank == 0 and not args.no_cpu:
        rate, n, dt = cpu_reference_rate(C1, C2, Rs, t_eff, 1, args.cpu_seconds)
        cpu = {"value": rate, "unit": "queries/s", "cores": 1, "kind": "reference",
               "sample": f"{n} trajectory poses through _core.cascade_3d (oracle/_ref, built from the "
                         f"reference sources), single thread, {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": "pose queries/sec (energy+force+torque) at K=32, 128^3, single-query loop",
            "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if prec == "fp32" else "f64", "data": "synthetic",
            "config": {"workload": "C2 haptic query loop: 128^3 grid, K=32 (w=64, m'=262144), "
                                   "1000 serial single-query launches per step",
                       "grid": GRID_N, "K": K_TRUNC, "w": W, "m_prime": W ** 3,
                       "queries_per_step": QUERIES_PER_STEP, "parallelism": f"replicas x{world}",
                       "l2": "flushed between steps (256 MiB write); windows L2-resident within a step "
                             "as in a live haptic loop"},
            "latency_us": {"kernel_mean": kernel_us, "e2e_p50": statistics.median(lat), "e2e_p95": pct(lat, 0.95),
                           "e2e_p99": pct(lat, 0.99), "launch_path_p50": statistics.median(lat1),
                           "launch_path_p99": pct(lat1, 0.99), "definition": "cli.py:357-361"},
            "e2e": {"value": e2e_value, "unit": "queries/s",
                    "h2d_bytes_per_step": QUERIES_PER_STEP * 25 * 8, "d2h_bytes_per_step": QUERIES_PER_STEP * 28 * 8,
                    "step": f"{QUERIES_PER_STEP} serial queries",
                    "path": "backend.cascade (host R, t_eff in -> host complex128[7] out) inside a haptic session "
                            "(backend.HapticServer): 25 self-tagged 8-byte request slots read by the GPU from "
                            "pinned host memory, 28 result slots written back; no launch per query",
                    "launch_path_value": args.e2e_queries * world / dt1,
                    "launch_path": "same call without a session: one single-query kernel launch per call"},
            "roofline": {"bound": "fp32" if prec == "fp32" else "fp64", "achieved": achieved,
                         "peak": peak.value, "unit": "TFLOP/s", "frac": achieved / peak.value,
                         "traffic": _traffic("cascade3d_single_kernel"),
                         "traffic_unit": "bytes per launch (DRAM read+write, ncu capture; windows stay L2-resident)",
                         "work": f"240 flops x live modes ({live:.3f} x {W ** 3}) per launch",
                         "peak_source": "FMA-chain kernel measured in this run (gf_measure_fma_peak)"},
            "cpu_baseline": cpu,
            "fp64_engine": fp64_mode,
            "gpu_launches": QUERIES_PER_STEP * args.steps,
            "clocks": clk.summary(),
            "stages": stages,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# secondary stages (extra keys; the headline metric is the haptic loop above)


def _peaks():
    import json as _json

    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return _json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "note": "fallback (B200_PROFILING.md)"}


def _traffic(kernel):
    """Per-launch DRAM bytes of `kernel` from the committed ncu capture summary
    (profiles/r01_traffic.json), or None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_traffic.json")) as fh:
            return json.load(fh)[kernel]["bytes"]
    except (OSError, KeyError, ValueError):
        return None


def _field_traffic():
    parts = [_traffic(k) for k in ("product_brick_kernel", "fft_rows_staged_kernel", "fft_cols_tma_kernel",
                                   "fft_cols_tma_kernel")]
    return None if None in parts else sum(parts)


def _time_ms(fn, reps=3):
    import torch

    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best


class _Asset:
    """Minimal PartAsset stand-in holding a device window (synthetic inputs)."""

    def __init__(self, grid, win, wrap):
        self.grid, self._win, self._wrap = grid, win, wrap

    def window(self, m_prime=None):
        return self._win, self._wrap

    def max_modes(self):
        return int(np.prod(self._win.shape))


def measure_stages(args, rank, world, fp32_peak):
    import torch

    import oracle  # the stages' cpu_baseline legs only (numpy restatements timed on the host)
    from paper_1711_05017_b200 import backend, parallel, scenes
    from paper_1711_05017_b200.descriptor import ComplexField, SampleGrid, affinity_field
    from paper_1711_05017_b200.energy import score_field_device
    from paper_1711_05017_b200.spectral import forward_window

    hbm = float(_peaks()["hbm_gbs"])
    out = {}
    dev = torch.device("cuda", torch.cuda.current_device())
    gen = torch.Generator(device=dev)
    gen.manual_seed(SEED + rank)

    # --- C1: the reference's own CPU case, end to end on real assets: peg-in-hole 64^3, K=16
    # (m' = 32^3), GPU density -> spectra -> windows, then a 1000-pose insertion trajectory
    # through the public evaluate(); the reference kernel runs the same windows and poses
    from paper_1711_05017_b200.energy import Configuration, evaluate

    sc1 = scenes.get_scene("peg_in_hole")
    m1 = 32 ** 3
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p1, p2 = sc1.build_assets(64, m_prime=m1)
    w1c, w1wrap = p1.window(m1)
    w2c, _ = p2.window(m1)
    torch.cuda.synchronize()
    pre_ms = (time.perf_counter() - t0) * 1e3
    n_traj = 1000
    zs = np.linspace(0.6, 0.0, n_traj)  # from clear of the block (peg bottom above its top) to seated
    cfgs = [Configuration(np.eye(3), np.array([0.0, 0.0, z])) for z in zs]
    from paper_1711_05017_b200.energy import haptic_session

    def run_traj():
        for cfg in cfgs[:20]:
            evaluate(p1, p2, cfg, m1)
        lat, rows = [], []
        t0 = time.perf_counter()
        for cfg in cfgs:
            q0 = time.perf_counter_ns()
            ev = evaluate(p1, p2, cfg, m1)
            lat.append((time.perf_counter_ns() - q0) / 1e3)
            rows.append(np.concatenate([[ev.energy], ev.force, ev.torque]))
        dt = time.perf_counter() - t0
        lat.sort()
        return n_traj / dt, lat[len(lat) // 2], lat[min(len(lat) - 1, int(0.99 * len(lat)))], rows

    with haptic_session(p1, p2, m1):
        rate_s, p50_s, p99_s, res1 = run_traj()
    rate_l, p50_l, p99_l, _ = run_traj()
    out["trajectory_C1"] = {
        "workload": "peg-in-hole (64-gon cylinder peg, bored block) 64^3, K=16 (m'=32768), 1000-pose "
                    "insertion trajectory through evaluate(); assets built on the GPU from the meshes",
        "precompute_ms": pre_ms, "poses_per_s": rate_s, "p50_us": p50_s, "p99_us": p99_s,
        "path": "evaluate() inside haptic_session (resident query grid)",
        "launch_path": {"poses_per_s": rate_l, "p50_us": p50_l, "p99_us": p99_l},
        "precision": backend.precision()}
    if rank == 0 and not args.no_cpu:
        core = reference_core()
        g1 = p1.grid
        C1h, C2h = np.asarray(w1c), np.asarray(w2c)
        c1 = g1.center()
        dcell1 = 1.0 / (g1.node_count * g1.cell_volume)
        idx = np.linspace(0, n_traj - 1, 100).astype(int)
        t0 = time.perf_counter()
        refs = [core.cascade_3d(C1h, C2h, bool(w1wrap), *g1.delta_omega(), dcell1, np.eye(3),
                                np.ascontiguousarray(cfgs[i].translation), c1) for i in idx]
        dt = time.perf_counter() - t0
        ref_rows = np.array([np.concatenate([[-r[0].real], r[1:4].real, r[4:7].real]) for r in refs])
        got = np.array(res1)[idx]
        # parity as BASELINE.md states it: |new - ref| <= 1e-4 max(|ref|, L1), L1 = dcell sum |summand|
        l1 = np.array([np.abs(oracle.cascade_term_scales(C1h, C2h, bool(w1wrap), g1.delta_omega(), dcell1,
                                                         np.eye(3), cfgs[i].translation, c1))
                       for i in idx])
        denom = np.maximum(np.abs(ref_rows), l1)
        out["trajectory_C1"]["max_err_over_tolerance_scale"] = float(np.max(np.abs(got - ref_rows) / denom))
        out["trajectory_C1"]["tolerance"] = "1e-4 of max(|ref|, L1) (BASELINE.md section 2)"
        out["trajectory_C1"]["cpu_baseline"] = {
            "value": len(idx) / dt, "unit": "poses/s", "cores": 1, "kind": "reference",
            "sample": f"{len(idx)} trajectory poses through _core.cascade_3d (oracle/_ref) on the same "
                      "windows, single thread"}
    del p1, p2
    torch.cuda.empty_cache()

    # --- C2 on real assets: the low-clearance peg-in-hole at 128^3, K=32 (m' = 64^3), the
    # headline configuration with GPU-built windows instead of synthetic ones; the jittered
    # insertion path of the headline, through evaluate() in a haptic session
    sc2 = scenes.get_scene("peg_in_hole_lowclear")
    m2 = 64 ** 3
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    q1, q2 = sc2.build_assets(128, m_prime=m2)
    v1c, v1wrap = q1.window(m2)
    v2c, _ = q2.window(m2)
    torch.cuda.synchronize()
    pre2_ms = (time.perf_counter() - t0) * 1e3
    Rj, tj, _ = trajectory(2000, SEED + 11)
    cfg2 = [Configuration(R, t) for R, t in zip(Rj, tj)]
    with haptic_session(q1, q2, m2):
        for cfg in cfg2[:50]:
            evaluate(q1, q2, cfg, m2)
        lat2, rows2 = [], []
        t0 = time.perf_counter()
        for cfg in cfg2:
            q0 = time.perf_counter_ns()
            ev = evaluate(q1, q2, cfg, m2)
            lat2.append((time.perf_counter_ns() - q0) / 1e3)
            rows2.append(np.concatenate([[ev.energy], ev.force, ev.torque]))
        dt2 = time.perf_counter() - t0
    lat2.sort()
    out["trajectory_C2_real"] = {
        "workload": "low-clearance peg-in-hole 128^3 (clearance 0.01 x bore), K=32 (m'=262144), 2000-pose "
                    "jittered insertion path through evaluate() in a haptic session; assets built on the GPU",
        "precompute_ms": pre2_ms, "poses_per_s": len(cfg2) / dt2, "p50_us": lat2[len(lat2) // 2],
        "p99_us": lat2[min(len(lat2) - 1, int(0.99 * len(lat2)))], "precision": backend.precision()}
    if rank == 0 and not args.no_cpu:
        core = reference_core()
        g2 = q1.grid
        D1h, D2h = np.asarray(v1c), np.asarray(v2c)
        c2 = g2.center()
        dcell2 = 1.0 / (g2.node_count * g2.cell_volume)
        idx = np.linspace(0, len(cfg2) - 1, 20).astype(int)
        teff = [cfg2[i].translation - c2 + cfg2[i].rotation @ c2 for i in idx]
        t0 = time.perf_counter()
        refs = [core.cascade_3d(D1h, D2h, bool(v1wrap), *g2.delta_omega(), dcell2,
                                np.ascontiguousarray(cfg2[i].rotation), np.ascontiguousarray(te), c2)
                for i, te in zip(idx, teff)]
        dt = time.perf_counter() - t0
        ref_rows = np.array([np.concatenate([[-r[0].real], r[1:4].real, r[4:7].real]) for r in refs])
        l1 = np.array([np.abs(oracle.cascade_term_scales(D1h, D2h, bool(v1wrap), g2.delta_omega(), dcell2,
                                                         cfg2[i].rotation, te, c2)) for i, te in zip(idx, teff)])
        got = np.array(rows2)[idx]
        out["trajectory_C2_real"]["max_err_over_tolerance_scale"] = float(
            np.max(np.abs(got - ref_rows) / np.maximum(np.abs(ref_rows), l1)))
        out["trajectory_C2_real"]["tolerance"] = "1e-4 of max(|ref|, L1) (BASELINE.md section 2)"
        out["trajectory_C2_real"]["cpu_baseline"] = {
            "value": len(idx) / dt, "unit": "poses/s", "cores": 1, "kind": "reference",
            "sample": f"{len(idx)} of the same poses through _core.cascade_3d (oracle/_ref) on the same windows, "
                      "single thread"}
    del q1, q2
    torch.cuda.empty_cache()

    # --- C3: batched pose sweep, gear-pair grid 256^3, K=48 (w=96), cmd_bench poses
    n3, w3, dom3 = 256, 96, 5.42
    g3 = SampleGrid(3, (n3,) * 3, (-0.5 * dom3,) * 3, dom3 / n3)
    mk = lambda w: torch.randn((w,) * 3, dtype=torch.complex128, device=dev, generator=gen) * 1e-2  # noqa: E731
    a1, a2 = _Asset(g3, backend.DeviceWindow(mk(w3)), False), _Asset(g3, backend.DeviceWindow(mk(w3)), False)
    Rs, ts = cmd_bench_poses(args.sweep_poses, 0.25 * dom3, seed=rank)
    c = g3.center()
    t_eff = ts - c + np.einsum("nij,j->ni", Rs, c)
    poses = torch.from_numpy(backend.pack_poses(Rs, t_eff)).to(dev)
    res = torch.empty((len(ts), 14), dtype=torch.float64, device=dev)
    dcell = 1.0 / (g3.node_count * g3.cell_volume)
    ms = _time_ms(lambda: backend.cascade_batch(a1._win, a2._win, False, g3.delta_omega(), dcell, c, poses,
                                                out=res, precision="fp32"))
    live = live_fraction(Rs, w3)
    t0 = time.perf_counter()
    parallel.pose_sweep(a1, a2, Rs, ts, precision="fp32")
    e2e_s = time.perf_counter() - t0
    achieved = 240.0 * live * w3 ** 3 * len(ts) / (ms * 1e-3) / 1e12
    out["sweep_C3"] = {
        "workload": f"{len(ts)} cmd_bench SE(3) poses (seed {rank}), 256^3 grid, K=48 (w=96, m'={w3 ** 3}), fp32",
        "poses_per_s": len(ts) / (ms * 1e-3), "e2e_poses_per_s": len(ts) / e2e_s,
        "e2e_path": "parallel.pose_sweep: host poses in, host complex128 results out",
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp32_peak, "work": f"240 flop x live modes ({live:.3f} of m')",
                     "traffic": _traffic("cascade3d_kernel"),
                     "traffic_unit": "bytes per 2048-pose launch (ncu capture)"},
        "projected_1e6_poses_s": 1e6 / (len(ts) / (ms * 1e-3)),
    }
    if rank == 0 and not args.no_cpu:
        core = reference_core()
        C1h, C2h = a1._win.__array__(), a2._win.__array__()
        n_cpu = 0
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < args.stage_cpu_seconds and n_cpu < len(ts):
            core.cascade_3d(C1h, C2h, False, *g3.delta_omega(), dcell, np.ascontiguousarray(Rs[n_cpu]),
                            np.ascontiguousarray(t_eff[n_cpu]), c)
            n_cpu += 1
        dt = time.perf_counter() - t0
        out["sweep_C3"]["cpu_baseline"] = {
            "value": n_cpu / dt, "unit": "poses/s", "cores": 1, "kind": "reference",
            "sample": f"{n_cpu} of the same poses through _core.cascade_3d (oracle/_ref), 1 thread"}
    del a1, a2, poses, res
    torch.cuda.empty_cache()

    # --- C4: full translational landscape 512^3 (full spectrum, w = N), fp32 field
    n4 = args.field_n
    g4 = SampleGrid(3, (n4,) * 3, (-1.0,) * 3, 2.0 / n4)
    b1, b2 = _Asset(g4, backend.DeviceWindow(mk(n4)), True), _Asset(g4, backend.DeviceWindow(mk(n4)), True)
    R4, _ = cmd_bench_poses(1, 1.0, seed=1)
    ms = _time_ms(lambda: score_field_device(b1, b2, R4[0], None, precision=32))
    alg = 24.0 * n4 ** 3  # read both complex64 windows + write the complex64 field
    ftr = _field_traffic() if n4 == 512 else None  # the committed capture is of the 512^3 landscape
    out["field_C4"] = {
        "workload": f"full translational field {n4}^3, full spectrum (w = N, wrap), one cmd_bench rotation (seed 1), "
                    "complex64 out",
        "voxels_per_s": n4 ** 3 / (ms * 1e-3), "ms": ms,
        "roofline": {"bound": "hbm", "achieved": alg / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                     "frac": alg / (ms * 1e-3) / 1e9 / hbm, "work": "24 B/voxel algorithmic",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                     "traffic": ftr,
                     "traffic_unit": "bytes per landscape: product + 3 FFT passes (ncu capture, 512^3)",
                     "dram_achieved": (ftr / (ms * 1e-3) / 1e9) if ftr else None,
                     "dram_frac": (ftr / (ms * 1e-3) / 1e9 / hbm) if ftr else None,
                     "dram_note": "measured DRAM traffic of the four kernels / this run's time: the HBM "
                                  "utilisation the north star's >= 50 % target refers to"},
        "scaling_plan": "slab-decomposed across ranks with one all-to-all (parallel.score_field_slab)",
    }
    if rank == 0 and not args.no_cpu:
        nc = 128
        rngc = np.random.default_rng(SEED)
        Cc1 = rngc.normal(size=(nc,) * 3) + 1j * rngc.normal(size=(nc,) * 3)
        Cc2 = rngc.normal(size=(nc,) * 3) + 1j * rngc.normal(size=(nc,) * 3)
        t0 = time.perf_counter()
        oracle.score_field(Cc1, Cc2, True, (nc,) * 3, (-1.0,) * 3, 2.0 / nc, R4[0])
        dt = time.perf_counter() - t0
        out["field_C4"]["cpu_baseline"] = {
            "value": nc ** 3 / dt, "unit": "voxels/s", "cores": 1, "kind": "port",
            "sample": f"oracle.score_field (numpy restatement of energy.score_field, energy.py:309-344) at "
                      f"{nc}^3 full spectrum, one rotation, {dt:.1f} s (512^3 does not fit a bounded CPU sample)"}
    del b1, b2
    torch.cuda.empty_cache()

    # --- C5: bolt-nut 256^3, K=64 (w=128), screw trajectory paced at 1 kHz
    from paper_1711_05017_b200.haptic import HapticSession

    n5, w5, dom5 = 256, 128, 4.37
    g5 = SampleGrid(3, (n5,) * 3, (-0.5 * dom5,) * 3, dom5 / n5)
    f5 = _Asset(g5, backend.DeviceWindow(mk(w5)), False), _Asset(g5, backend.DeviceWindow(mk(w5)), False)
    frames = args.haptic_frames
    th = np.linspace(0.0, 4.0 * np.pi, frames)  # two turns
    pitch = 0.1
    R5 = np.stack([axis_rot(2, a) for a in th])
    t5 = np.stack([np.array([0.0, 0.0, 0.3 - pitch * a / (2 * np.pi)]) for a in th])
    sess = HapticSession(f5[0], f5[1], None)
    sess.run(R5[:50], t5[:50], rate_hz=1000.0)  # warm
    run = sess.run(R5, t5, rate_hz=1000.0)
    out["haptic_C5"] = {"workload": f"bolt-nut 256^3 grid, K=64 (w=128, m'={w5 ** 3}), {frames}-frame screw "
                                    "trajectory (2 turns, pitch 0.1) paced at 1 kHz, one evaluate per frame served by a "
                                    "resident query grid (haptic_session), fp32",
                        **run, "budget_us": 1000.0}
    del f5, sess
    torch.cuda.empty_cache()

    # --- W: forward centred window 256^3 -> w = 96 (complex128 field -> complex128 window)
    gw = SampleGrid(3, (256,) * 3, (-1.0,) * 3, 2.0 / 256)
    fw = ComplexField(gw, torch.randn(256 ** 3, dtype=torch.complex128, device=dev, generator=gen))
    ms = _time_ms(lambda: forward_window(fw, 96))
    alg = 16.0 * 256 ** 3 + 16.0 * 96 ** 3
    out["window_W"] = {"workload": "forward DFT + truncation + centring, 256^3 complex128 field -> 96^3 window",
                       "ms": ms, "roofline": {"bound": "hbm", "achieved": alg / (ms * 1e-3) / 1e9, "peak": hbm,
                                              "unit": "GB/s", "frac": alg / (ms * 1e-3) / 1e9 / hbm}}
    if rank == 0 and not args.no_cpu:
        fh = fw.values.reshape((256,) * 3)
        t0 = time.perf_counter()
        A = oracle.forward_dft(fh, (256,) * 3, (-1.0,) * 3, 2.0 / 256)
        oracle.center_window(A, (256,) * 3, (-1.0,) * 3, 2.0 / 256, 96)
        dt = time.perf_counter() - t0
        out["window_W"]["cpu_baseline"] = {"value": dt * 1e3, "unit": "ms", "cores": 1, "kind": "port",
                                           "sample": "oracle.forward_dft + center_window (numpy pocketfft, as "
                                                     "spectral.py:114-195) on the same 256^3 field"}
    del fw
    torch.cuda.empty_cache()

    # --- D: skeletal density of the C1 bored block at 64^3 (512 faces), float64
    sc = scenes.get_scene("peg_in_hole")
    gd = sc.grid(64)
    affinity_field(sc.fixed, gd, sc.kernel)
    torch.cuda.synchronize()
    dt = None
    for _ in range(3):  # best of 3 wall-clock calls (host allocation jitter)
        t0 = time.perf_counter()
        fd = affinity_field(sc.fixed, gd, sc.kernel)
        d1 = time.perf_counter() - t0
        dt = d1 if dt is None else min(dt, d1)
    nf = len(sc.fixed.mesh.faces)
    out["density_D"] = {"workload": f"affinity_field, bored block ({nf} faces) on 64^3, float64 bit-exact flags",
                        "voxels_per_s": gd.node_count / dt, "node_face_pairs_per_s": gd.node_count * nf / dt,
                        "ms": dt * 1e3, "excluded": fd.stats["excluded"], "unresolved": fd.stats["unresolved_nodes"],
                        "device_seconds": {"distance_winding": fd.stats.get("seconds_distance"),
                                           "sweep": fd.stats.get("seconds_sweep")},
                        "roofline": {"bound": "fp64", "unit": "FP64 pipe utilisation (ncu)", "frac": 0.409,
                                     "source": "profiles/r01_ncu_density_sweep.txt: sweep_kernel "
                                               "sm__inst_executed_pipe_fp64 40.9 % of peak"}}
    if rank == 0 and not args.no_cpu:
        core = reference_core()
        gc = sc.grid(16)
        P = gc.points()
        m = sc.fixed.mesh
        tri = np.ascontiguousarray(m.triangles)
        t0 = time.perf_counter()
        xi = np.empty(len(P))
        core.distance_3d(*sc.fixed.bvh(), tri, P, xi, 0, len(P))
        wind = np.empty(len(P))
        core.winding_3d(tri, P, wind, 0, len(P))
        iplus = np.empty(len(P), dtype=np.complex128)
        res = np.zeros(len(P))
        cl = np.zeros(len(P), dtype=np.int64)
        core.sweep_3d(tri, m.normals, m.areas, P, np.maximum(xi, 0.25 * gc.spacing), 0.5, 1 / (4 * np.pi), 0.02, 16,
                      0.25 * gc.spacing, iplus, res, cl, 0, len(P))
        dt = time.perf_counter() - t0
        out["density_D"]["cpu_baseline"] = {
            "value": gc.node_count * nf / dt, "unit": "node-face pairs/s", "cores": 1, "kind": "reference",
            "sample": f"_core distance_3d + winding_3d + sweep_3d (oracle/_ref) for the same part on 16^3, {dt:.1f} s"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--e2e-queries", type=int, default=2000)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=6.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-stages", action="store_true")
    ap.add_argument("--sweep-poses", type=int, default=16384)
    ap.add_argument("--stage-cpu-seconds", type=float, default=4.0)
    ap.add_argument("--haptic-frames", type=int, default=1000)
    ap.add_argument("--field-n", type=int, default=512)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("note: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_engine(args)


if __name__ == "__main__":
    sys.exit(main())
