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
  parity  per stage, max |new - ref| / (1e-4 max(|ref|, L1)) (<= 1 passes,
          BASELINE.md section 2) and the plain relative error, against the
          reference kernel (oracle/_ref) or the oracle restatement.
  stages  the other BASELINE configs on their stated inputs (C1 peg-in-hole
          64^3 trajectory, C2 on real assets, C3 gear-pair 10^6-pose sweep,
          C4 512^3 landscape of real spectra, C5 bolt-nut 1 kHz trajectory,
          stage-1 density and stage-2 window), compact.

--impl reference runs the reference kernel with every host core (a thread
pool over poses; _core.cascade_3d releases the GIL) on the same config.

Multi-GPU: `--gpus N` without a torchrun environment re-launches itself
under torch.distributed.run with N ranks.  The single haptic query does not
shard: N independent replicas, whole-job totals
(max-over-ranks time).  The C3 sweep shards its 10^6 poses by rank and the
C4 landscape is slab-decomposed across ranks (parallel.score_field_slab).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
METRIC = "pose queries/sec (energy+force+torque) at K=32, 128^3, single-query loop"
CONFIG = {"workload": "C2 haptic query loop: 128^3 grid, K=32 (w=64, m'=262144), 1000 serial single queries per step",
          "grid": GRID_N, "K": K_TRUNC, "w": W, "m_prime": W ** 3, "queries_per_step": QUERIES_PER_STEP,
          "poses": "jittered insertion path, rng seed 20260814",
          "l2": "flushed between steps (256 MiB write); windows L2-resident within a step as in a live haptic loop",
          "parallelism": "replicas: one independent haptic loop per GPU"}


def r4(x):
    """Compact float for the JSON line (4 significant digits)."""
    if x is None or isinstance(x, (bool, int, str)):
        return x
    return float(f"{float(x):.4g}")


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


# ---------------------------------------------------------------------------
# process topology


def spawn_ranks(args):
    """`--gpus N` outside torchrun: re-launch this script with N ranks
    (torch.distributed.run, loopback rendezvous) and return its exit code."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
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
    q = np.empty((n, 4))
    t = np.empty((n, 3))
    for i in range(n):  # the reference's draw order: 4 normals, then 3 uniforms, per pose
        q[i] = rng.normal(size=4)
        t[i] = rng.uniform(-span, span, 3)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    R = np.stack([np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)], -1),
                  np.stack([2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)], -1),
                  np.stack([2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], -1)], 1)
    return R, t


# ---------------------------------------------------------------------------
# CPU reference (the reference's compiled kernel, oracle/_ref) and parity


def reference_core():
    import oracle

    core = oracle.ref_core()
    if core is None:
        raise RuntimeError("oracle/_ref not built (make -C oracle ref in the build container)")
    return core


def ref_cascade(C1, C2, wrap, dom, dcell, R, t_eff, c):
    core = reference_core()
    wr = lambda x, dt=np.float64: np.require(x, dtype=dt, requirements=["C", "W"])  # noqa: E731  (memoryviews)
    return np.asarray(core.cascade_3d(wr(C1, np.complex128), wr(C2, np.complex128), bool(wrap), *[float(v) for v in dom],
                                      float(dcell), wr(R), wr(t_eff), wr(c)))


def parity_entry(got, want, l1, against):
    """got/want complex [n, 7] (or [n]) arrays; l1 the per-output term scales."""
    got, want, l1 = np.asarray(got), np.asarray(want), np.asarray(l1)
    den = 1e-4 * np.maximum(np.abs(want), l1)
    return {"err_tol": r4(np.max(np.abs(got - want) / den)),
            "rel": r4(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300)),
            "n": int(want.shape[0]) if want.ndim > 1 else int(want.size), "vs": against}


def parity_of_poses(C1, C2, wrap, dom, dcell, c, Rs, t_effs, got, threads=8):
    """Reference kernel (oracle/_ref) on the same windows/poses, in a thread pool."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle

    with ThreadPoolExecutor(max_workers=threads) as pool:
        want = list(pool.map(lambda i: ref_cascade(C1, C2, wrap, dom, dcell, Rs[i], t_effs[i], c), range(len(Rs))))
        l1 = list(pool.map(lambda i: oracle.cascade_term_scales(C1, C2, wrap, dom, dcell, Rs[i], t_effs[i], c),
                           range(len(Rs))))
    return parity_entry(np.asarray(got), np.asarray(want), np.asarray(l1), "oracle/_ref _core.cascade_3d")


def cpu_reference_rate(C1, C2, Rs, t_eff, threads, budget_s, wrap=False, consts=None):
    """Queries/s of _core.cascade_3d on `threads` host threads for ~budget_s."""
    from concurrent.futures import ThreadPoolExecutor

    core = reference_core()
    _, center, dom, dcell = consts or grid_params()
    C1 = np.ascontiguousarray(C1)
    C2 = np.ascontiguousarray(C2)

    def one(i):
        return core.cascade_3d(C1, C2, bool(wrap), dom[0], dom[1], dom[2], dcell, np.ascontiguousarray(Rs[i]),
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
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": CONFIG,
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

    def e2e_loop(precision):
        lat = []
        for i in range(50):
            backend.cascade(W1, W2, False, dom, dcell, Re[i], te[i], center, precision=precision)
        barrier(world)
        t0 = time.perf_counter()
        for i in range(50, 50 + args.e2e_queries):
            q0 = time.perf_counter_ns()
            backend.cascade(W1, W2, False, dom, dcell, Re[i], te[i], center, precision=precision)
            lat.append((time.perf_counter_ns() - q0) / 1e3)
        dt = time.perf_counter() - t0
        barrier(world)
        return sorted(lat), max_over_ranks(dt, world)

    with backend.HapticServer(W1, W2, False, dom, dcell, center, precision=prec):
        lat, e2e_s = e2e_loop(prec)
    lat1, dt1 = e2e_loop(prec)  # no server: one single-query kernel launch per call
    e2e_value = args.e2e_queries * world / e2e_s
    lat64 = None
    if prec == "fp32":  # the float64 engine (the reference's own tolerances) in the same session loop
        with backend.HapticServer(W1, W2, False, dom, dcell, center, precision="fp64"):
            lat64, _ = e2e_loop("fp64")

    def pct(xs, p):
        return xs[min(len(xs) - 1, int(p * len(xs)))]

    # ---- roofline: cascade kernel vs the FP32 FMA pipe measured here
    import ctypes

    peak = ctypes.c_double(0.0)
    _lib.check(_lib.LIB.gf_measure_fma_peak(64 if prec == "fp64" else 32, ctypes.byref(peak)))
    peak64 = ctypes.c_double(0.0)
    _lib.check(_lib.LIB.gf_measure_fma_peak(64, ctypes.byref(peak64)))
    live = live_fraction(Rs, W)
    flops = 240.0 * live * W ** 3
    achieved = flops / (kernel_us * 1e-6) / 1e12

    # ---- parity of the timed loop's own outputs against the reference kernel
    parity = {}
    if rank == 0 and not args.no_cpu:
        idx = np.linspace(args.warmup * QUERIES_PER_STEP, n_total - 1, 6).astype(int)
        got = out[idx].cpu().numpy().view(np.complex128)
        parity["C2_loop"] = parity_of_poses(C1, C2, False, dom, dcell, center, Rs[idx], t_eff[idx], got)

    stages = {} if args.no_stages else measure_stages(args, rank, world, peak.value, peak64.value, parity)

    cpu = None
    if rank == 0 and not args.no_cpu:
        rate, n, dt = cpu_reference_rate(C1, C2, Rs, t_eff, 1, args.cpu_seconds)
        cpu = {"value": rate, "unit": "queries/s", "cores": 1, "kind": "reference",
               "sample": f"{n} trajectory poses through _core.cascade_3d (oracle/_ref, built from the "
                         f"reference sources), single thread, {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if prec == "fp32" else "f64", "data": "synthetic",
            "config": CONFIG,
            "e2e": {"value": e2e_value, "unit": "queries/s",
                    "h2d_bytes_per_step": QUERIES_PER_STEP * 25 * 8, "d2h_bytes_per_step": QUERIES_PER_STEP * 28 * 8,
                    "path": "backend.cascade in a haptic session (resident grid, host-mapped mailbox)",
                    "launch_path_value": r4(args.e2e_queries * world / dt1)},
            "roofline": {"bound": "fp32" if prec == "fp32" else "fp64", "achieved": achieved, "peak": peak.value,
                         "unit": "TFLOP/s", "frac": achieved / peak.value, "traffic": _traffic("cascade3d_single_kernel"),
                         "work": f"240 flop x live modes ({live:.3f} x {W ** 3}) per launch",
                         "peak_source": "FMA-chain kernel measured in this run (gf_measure_fma_peak)"},
            "cpu_baseline": cpu,
            "gpu_launches": QUERIES_PER_STEP * args.steps,
            "clocks": clk.summary(),
            "latency_us": {"kernel_mean": r4(kernel_us), "e2e_p50": r4(statistics.median(lat)),
                           "e2e_p99": r4(pct(lat, 0.99)), "launch_p50": r4(statistics.median(lat1)),
                           "launch_p99": r4(pct(lat1, 0.99)),
                           "fp64_e2e_p50": r4(statistics.median(lat64)) if lat64 else None},
            "parity": parity,
            "stages": stages,
        }
        print(json.dumps(line, separators=(",", ":")), flush=True)
    barrier(world)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# secondary stages: the other BASELINE configs on their stated inputs


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "note": "fallback (B200_PROFILING.md)"}


def _traffic(kernel):
    """Per-launch DRAM bytes of `kernel` from the committed ncu capture summary
    (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh)[kernel]["bytes"]
    except (OSError, KeyError, ValueError):
        return None


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
    """Minimal PartAsset stand-in holding a device window built on the GPU."""

    def __init__(self, grid, win, wrap):
        self.grid, self._win, self._wrap = grid, win, wrap

    def window(self, m_prime=None):
        return self._win, self._wrap

    def max_modes(self):
        return int(np.prod(self._win.shape))


def _gpu_windows(scene, n, w, world, rank):
    """GPU density (node slabs across ranks when world > 1) and the centred
    w^3 windows of both parts (spectral.forward_window); returns the two
    device windows, the grid and the density seconds."""
    import torch

    from paper_1711_05017_b200 import backend, parallel
    from paper_1711_05017_b200.descriptor import affinity_field
    from paper_1711_05017_b200.spectral import forward_window

    sc = scenes_mod().get_scene(scene)
    g = sc.grid(n)
    wins, dens_s = [], 0.0
    for solid in (sc.fixed, sc.moving):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world > 1:
            f = parallel.affinity_field_slab(solid, g, sc.kernel)
        else:
            f = affinity_field(solid, g, sc.kernel)
        torch.cuda.synchronize()
        dens_s += time.perf_counter() - t0
        wins.append(backend.DeviceWindow(forward_window(f, w)))
        del f
    torch.cuda.empty_cache()
    return wins[0], wins[1], g, dens_s


def scenes_mod():
    from paper_1711_05017_b200 import scenes

    return scenes


def measure_stages(args, rank, world, fp32_peak, fp64_peak, parity):
    import torch

    out = {}
    lead = rank == 0
    cpu_ok = lead and not args.no_cpu

    def guarded(key, fn, collective):
        """A stage that fails records its error instead of ending the run (the
        headline line still prints); for the sharded stages every rank learns
        whether any rank failed, so none waits in a collective alone."""
        err = None
        try:
            out[key] = fn()
        except Exception as e:  # noqa: BLE001  (reported in the JSON line)
            err = f"{type(e).__name__}: {e}"[:200]
            out[key] = {"error": err}
        torch.cuda.empty_cache()
        if collective and world > 1:
            flag = torch.tensor([1.0 if err else 0.0], device="cuda")
            import torch.distributed as dist

            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            return flag.item() == 0.0
        return err is None

    if lead:
        guarded("C1C2", lambda: stage_trajectories(args, parity, cpu_ok, fp32_peak), False)
        out.update(out.pop("C1C2") if "error" not in out.get("C1C2", {}) else {"C1C2": out["C1C2"]})
    barrier(world)
    if guarded("C3", lambda: stage_sweep(args, rank, world, fp32_peak, parity, cpu_ok), True):
        barrier(world)
        guarded("C4", lambda: stage_field(args, rank, world, parity, cpu_ok), True)
    barrier(world)
    if lead:
        guarded("C5", lambda: stage_haptic(args, parity, cpu_ok, fp32_peak), False)
        guarded("W", lambda: stage_window(args, parity, cpu_ok), False)
        guarded("D", lambda: stage_density(args, fp64_peak, parity, cpu_ok), False)
    barrier(world)
    return out


def stage_trajectories(args, parity, cpu_ok, fp32_peak):
    """C1 (the reference's CPU case) and C2 on real GPU-built assets, through
    the public evaluate() inside a haptic session; parity vs the reference
    kernel on the very windows the engine uses."""
    import torch

    from paper_1711_05017_b200 import backend
    from paper_1711_05017_b200.energy import Configuration, evaluate, haptic_session

    res = {}
    for key, scene, n, side, npose in (("C1", "peg_in_hole", 64, 32, 1000), ("C2", "peg_in_hole_lowclear", 128, 64,
                                                                              2000)):
        sc = scenes_mod().get_scene(scene)
        m = side ** 3
        sc.build_assets(n, m_prime=m)  # warm-up: first use of the density / spectral kernels
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a1, a2 = sc.build_assets(n, m_prime=m)
        (w1, wrap), (w2, _) = a1.window(m), a2.window(m)
        torch.cuda.synchronize()
        pre_ms = (time.perf_counter() - t0) * 1e3
        if key == "C1":  # insertion trajectory: from clear of the block to seated
            cfgs = [Configuration(np.eye(3), np.array([0.0, 0.0, z])) for z in np.linspace(0.6, 0.0, npose)]
        else:  # the headline's jittered path
            Rj, tj, _ = trajectory(npose, SEED + 11)
            cfgs = [Configuration(R, t) for R, t in zip(Rj, tj)]
        with haptic_session(a1, a2, m) as srv:
            for cfg in cfgs[:50]:
                evaluate(a1, a2, cfg, m)
            lat, rows, gpu = [], [], []
            t0 = time.perf_counter()
            for cfg in cfgs:
                q0 = time.perf_counter_ns()
                ev = evaluate(a1, a2, cfg, m)
                lat.append((time.perf_counter_ns() - q0) / 1e3)
                rows.append(np.concatenate([[ev.score.real], ev.force, ev.torque]))
                gpu.append(srv.last_timing()["gpu_us"])
            dt = time.perf_counter() - t0
        lat.sort()
        gpu_us = statistics.median(gpu)
        live = live_fraction(np.array([c.rotation for c in cfgs[::max(1, len(cfgs) // 8)]]), side)
        achieved = 240.0 * live * m / (gpu_us * 1e-6) / 1e12
        st = {"poses_per_s": r4(len(cfgs) / dt), "p50_us": r4(lat[len(lat) // 2]),
              "p99_us": r4(lat[min(len(lat) - 1, int(0.99 * len(lat)))]), "gpu_us_p50": r4(gpu_us),
              "roofline": {"bound": "fp32", "achieved": r4(achieved), "peak": r4(fp32_peak), "unit": "TFLOP/s",
                           "frac": r4(achieved / fp32_peak)},
              "precompute_ms": r4(pre_ms), "in": f"{scene} {n}^3 GPU assets, evaluate() in a session"}
        if cpu_ok:
            g = a1.grid
            C1h, C2h = np.asarray(w1), np.asarray(w2)
            c, dom, dcell = g.center(), g.delta_omega(), 1.0 / (g.node_count * g.cell_volume)
            idx = np.linspace(0, len(cfgs) - 1, 24).astype(int)
            Rp = np.array([cfgs[i].rotation for i in idx])
            tp = np.array([cfgs[i].translation - c + cfgs[i].rotation @ c for i in idx])
            # evaluate() returns real parts: Re S (energy = -Re S), force = Re T, torque = Re G
            got = np.array([rows[i] for i in idx])
            from concurrent.futures import ThreadPoolExecutor

            import oracle

            with ThreadPoolExecutor(max_workers=8) as pool:
                want = list(pool.map(lambda k: ref_cascade(C1h, C2h, wrap, dom, dcell, Rp[k], tp[k], c),
                                     range(len(idx))))
                l1 = list(pool.map(lambda k: oracle.cascade_term_scales(C1h, C2h, wrap, dom, dcell, Rp[k], tp[k], c),
                                   range(len(idx))))
            want = np.array([np.concatenate([[w_[0].real], w_[1:4].real, w_[4:7].real]) for w_ in want])
            parity[key] = parity_entry(got, want, np.asarray(l1).real, "oracle/_ref _core.cascade_3d")
            t0 = time.perf_counter()
            nref = 0
            while time.perf_counter() - t0 < args.stage_cpu_seconds and nref < len(idx):
                ref_cascade(C1h, C2h, wrap, dom, dcell, Rp[nref], tp[nref], c)
                nref += 1
            st["cpu"] = {"value": r4(nref / (time.perf_counter() - t0)), "unit": "poses/s", "cores": 1,
                         "kind": "reference"}
        res[key] = st
        del a1, a2, w1, w2
        torch.cuda.empty_cache()
    return res


def stage_sweep(args, rank, world, fp32_peak, parity, cpu_ok):
    """C3: 10^6 cmd_bench SE(3) poses of the gear pair (256^3, K=48: w = 96),
    sharded by pose across ranks; device-timed kernel region (poses already
    in HBM, max over ranks) and the e2e parallel.pose_sweep (host poses in,
    gathered host results out)."""
    import torch

    from paper_1711_05017_b200 import backend, parallel

    n3, w3 = 256, 96
    W1, W2, g, dens_s = _gpu_windows("gear_pair", n3, w3, world, rank)
    a1, a2 = _Asset(g, W1, False), _Asset(g, W2, False)
    span = 0.25 * (g.spacing * n3)
    Rs, ts = cmd_bench_poses(args.sweep_poses, span, seed=0)
    c = g.center()
    dom, dcell = g.delta_omega(), 1.0 / (g.node_count * g.cell_volume)
    lo, hi = parallel.shard_range(len(ts), rank, world)
    t_eff = ts[lo:hi] - c + np.einsum("nij,j->ni", Rs[lo:hi], c)
    poses = torch.from_numpy(backend.pack_poses(Rs[lo:hi], t_eff)).cuda()
    res = torch.empty((hi - lo, 14), dtype=torch.float64, device="cuda")

    def run():
        backend.cascade_batch(W1, W2, False, dom, dcell, c, poses, out=res, precision="fp32")

    run()
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    e1.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    barrier(world)
    t0 = time.perf_counter()
    parallel.pose_sweep(a1, a2, Rs, ts, precision="fp32")
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    live = live_fraction(Rs[:64], w3)
    achieved = 240.0 * live * w3 ** 3 * (hi - lo) / (ms * 1e-3) / 1e12
    st = {"poses": len(ts), "n_gpus": world, "poses_per_s": r4(len(ts) / (ms * 1e-3)), "s": r4(ms * 1e-3),
          "e2e_poses_per_s": r4(len(ts) / e2e_s), "frac": r4(achieved / fp32_peak), "tflops": r4(achieved),
          "density_s": r4(dens_s), "in": "gear_pair 256^3 GPU assets, cmd_bench poses"}
    if cpu_ok:
        C1h, C2h = np.asarray(W1), np.asarray(W2)
        idx = np.array([0, 1, 4097, (hi - lo) - 1])
        got = res[idx].cpu().numpy().view(np.complex128)
        parity["C3"] = parity_of_poses(C1h, C2h, False, dom, dcell, c, Rs[lo:hi][idx], t_eff[idx], got)
        rate, n, dt = cpu_reference_rate(C1h, C2h, Rs, ts - c + np.einsum("nij,j->ni", Rs, c), 1,
                                         args.stage_cpu_seconds, consts=(None, c, dom, dcell))
        st["cpu"] = {"value": r4(rate), "unit": "poses/s", "cores": 1, "kind": "reference",
                     "days_1e6": r4(1e6 / rate / 86400)}
    del poses, res, W1, W2, a1, a2
    return st


def stage_field(args, rank, world, parity, cpu_ok):
    """C4: the full translational field at 512^3 (full spectra, w = N, wrap)
    of the gear pair, one cmd_bench rotation (seed 1) and R = I; slab-decomposed across
    ranks when world > 1.  Roofline 24 B/voxel; cuFFT C2C
    of the same size timed beside it as the speed bar; parity on the m' =
    128^3 windowed variant's voxels against the C restatement of the cascade."""
    import torch

    from paper_1711_05017_b200 import parallel
    from paper_1711_05017_b200.energy import score_field_device

    n4 = args.field_n
    hbm = float(_peaks()["hbm_gbs"])
    W1, W2, g, dens_s = _gpu_windows("gear_pair", n4, n4, world, rank)
    a1, a2 = _Asset(g, W1, True), _Asset(g, W2, True)
    R4 = cmd_bench_poses(1, 1.0, seed=1)[0][0]
    if world > 1:
        fn = lambda: parallel.score_field_slab(a1, a2, R4, None, precision=32)  # noqa: E731
    else:
        fn = lambda: score_field_device(a1, a2, R4, None, precision=32)  # noqa: E731
    fn()
    torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(_time_ms(fn), world)
    alg = 24.0 * n4 ** 3
    st = {"n": n4, "n_gpus": world, "ms": r4(ms), "gvox_per_s": r4(n4 ** 3 / (ms * 1e-3) / 1e9),
          "roofline": {"bound": "hbm", "achieved": r4(alg / (ms * 1e-3) / 1e9), "peak": hbm, "unit": "GB/s",
                       "frac": r4(alg / (ms * 1e-3) / 1e9 / hbm), "work": "24 B/voxel"},
          "density_s": r4(dens_s), "in": "gear_pair 512^3 GPU spectra"}
    # the survey's second rotation, R = I (lattice-aligned: every index comes from the tie tables)
    if world > 1:
        fi = lambda: parallel.score_field_slab(a1, a2, np.eye(3), None, precision=32)  # noqa: E731
    else:
        fi = lambda: score_field_device(a1, a2, np.eye(3), None, precision=32)  # noqa: E731
    fi()
    torch.cuda.synchronize()
    barrier(world)
    ms_i = max_over_ranks(_time_ms(fi), world)
    st["identity_R"] = {"ms": r4(ms_i), "gvox_per_s": r4(n4 ** 3 / (ms_i * 1e-3) / 1e9),
                        "frac": r4(alg / (ms_i * 1e-3) / 1e9 / hbm)}
    if world == 1:  # cuFFT C2C inverse of the same size (torch.fft -> cuFFT), the speed bar
        x = torch.empty((n4,) * 3, dtype=torch.complex64, device="cuda")
        x.normal_()
        st["cufft_c2c_ms"] = r4(_time_ms(lambda: torch.fft.ifftn(x)))
        del x
    del a1, a2, W1, W2
    torch.cuda.empty_cache()
    if cpu_ok:  # windowed variant m' = 128^3 in the 512^3 grid: voxels vs the C restatement of the cascade
        import oracle

        rng = np.random.default_rng(4)
        wv = 128
        k2 = (np.arange(wv) - wv // 2).astype(np.float64) ** 2
        amp = 1.0 / (1.0 + k2[:, None, None] + k2[None, :, None] + k2[None, None, :])
        C1 = (rng.standard_normal((wv,) * 3) + 1j * rng.standard_normal((wv,) * 3)) * amp
        C2 = (rng.standard_normal((wv,) * 3) + 1j * rng.standard_normal((wv,) * 3)) * amp
        from paper_1711_05017_b200 import backend

        V1, V2 = backend.DeviceWindow(C1), backend.DeviceWindow(C2)
        land = score_field_device(_Asset(g, V1, False), _Asset(g, V2, False), R4, None, precision=32)
        st["windowed_ms"] = r4(_time_ms(lambda: score_field_device(_Asset(g, V1, False), _Asset(g, V2, False), R4,
                                                                   None, precision=32)))
        picks = [(0, 0, 0), (n4 // 2, n4 // 2, n4 // 2), (17, 300, n4 - 1), (n4 - 1, 5, 260), (100, 200, 300),
                 (400, 33, 77)]
        vals = land.reshape((n4,) * 3)
        got = np.array([complex(vals[p].item()) for p in picks])
        c, dom, dcell = g.center(), g.delta_omega(), 1.0 / (g.node_count * g.cell_volume)
        from concurrent.futures import ThreadPoolExecutor

        pts = [np.asarray(g.origin) + g.spacing * np.asarray(p, dtype=np.float64) for p in picks]
        with ThreadPoolExecutor(max_workers=len(picks)) as pool:
            want = np.array(list(pool.map(lambda p: oracle.cascade(C1, C2, False, dom, dcell, R4, p - c + R4 @ c,
                                                                   c)[0], pts)))
        l1 = oracle.score_field_scale(C1, C2, False, g.dims, g.spacing, R4)
        parity["C4"] = parity_entry(got, want, np.full(len(picks), l1), "oracle C cascade at t = p_j (windowed 128^3)")
        del land, vals, V1, V2
        torch.cuda.empty_cache()
        nc = 128
        rngc = np.random.default_rng(SEED)
        Cc1 = rngc.normal(size=(nc,) * 3) + 1j * rngc.normal(size=(nc,) * 3)
        Cc2 = rngc.normal(size=(nc,) * 3) + 1j * rngc.normal(size=(nc,) * 3)
        t0 = time.perf_counter()
        oracle.score_field(Cc1, Cc2, True, (nc,) * 3, (-1.0,) * 3, 2.0 / nc, R4)
        dt = time.perf_counter() - t0
        st["cpu"] = {"value": r4(nc ** 3 / dt), "unit": "voxels/s", "cores": 1, "kind": "port",
                     "sample": f"numpy restatement of energy.score_field at {nc}^3"}
    return st


def stage_haptic(args, parity, cpu_ok, fp32_peak):
    """C5: bolt-nut 256^3, K=64 (w = 128) from GPU-built densities of the
    ~10^5-face meshes; a screw trajectory (2 turns, pitch 0.1) paced at
    1 kHz, one evaluate per frame from a resident query grid; then the same
    session held to part of the GPU while a 256^3 landscape runs in a worker
    thread."""
    import torch

    from paper_1711_05017_b200.energy import score_field_device
    from paper_1711_05017_b200.haptic import HapticSession

    n5, w5 = 256, 128
    W1, W2, g, dens_s = _gpu_windows("bolt_nut", n5, w5, 1, 0)
    f5 = _Asset(g, W1, False), _Asset(g, W2, False)
    frames = args.haptic_frames
    th = np.linspace(0.0, 4.0 * np.pi, frames)
    pitch = 0.1
    R5 = np.stack([axis_rot(2, a) for a in th])
    t5 = np.stack([np.array([0.0, 0.0, 0.3 - pitch * a / (2 * np.pi)]) for a in th])
    sess = HapticSession(f5[0], f5[1], None)
    sess.run(R5[:200], t5[:200], rate_hz=1000.0)  # warm
    run = sess.run(R5, t5, rate_hz=1000.0)
    live = live_fraction(R5[:: max(1, frames // 8)], w5)
    gpu_us = run["gpu_us_p50"]
    achieved = 240.0 * live * w5 ** 3 / (gpu_us * 1e-6) / 1e12
    missed = [{k: r4(v) for k, v in m.items() if k in ("frame", "us", "gpu_us", "gpu_poll_gap_us", "gpu_clock_gap_us")}
              for m in run["missed"][:4]]
    st = {"frames": run["frames"], "p50_us": r4(run["p50_us"]), "p99_us": r4(run["p99_us"]),
          "max_us": r4(run["max_us"]), "misses": run["deadline_misses"], "missed": missed,
          "miss_cause": "GPU-wide stall (gpu_clock_gap_us)" if run["deadline_misses"] else None,
          "realtime": run["realtime"], "gpu_us_p50": r4(gpu_us),
          "roofline": {"bound": "fp32", "achieved": r4(achieved), "peak": r4(fp32_peak), "unit": "TFLOP/s",
                       "frac": r4(achieved / fp32_peak), "work": f"240 flop x live modes ({live:.3f} x {w5 ** 3})"},
          "density_s": r4(dens_s), "in": "bolt_nut 256^3 GPU assets (75852 + 98816 faces)"}
    # concurrency: a landscape export in a worker thread while the session serves frames
    # on a subset of the SMs (the reference service's field worker, service.py:305-318)
    gl = scenes_mod().get_scene("bolt_nut").grid(256)
    L1, L2 = _Asset(gl, W1, False), _Asset(gl, W2, False)
    done = {}

    def export():
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            t0 = time.perf_counter()
            k = 0
            while time.perf_counter() - t0 < 1.5:
                score_field_device(L1, L2, R5[k % frames], None, precision=32)
                k += 1
            stream.synchronize()
            done["fields"] = k
            done["s"] = time.perf_counter() - t0

    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    worker = threading.Thread(target=export)
    worker.start()
    crun = sess.run(R5[:2000], t5[:2000], rate_hz=1000.0, max_sms=nsm * 3 // 4)
    worker.join()
    st["concurrent"] = {"frames": crun["frames"], "p99_us": r4(crun["p99_us"]), "max_us": r4(crun["max_us"]),
                        "misses": crun["deadline_misses"], "fields_done": done.get("fields"),
                        "fields_per_s": r4(done.get("fields", 0) / max(done.get("s", 1e-9), 1e-9)),
                        "server_sms": nsm * 3 // 4}
    # the platform's own GPU-wide stalls in the same run: every SM spins on the
    # clock for 5 s with no host interaction (gf_measure_stalls)
    from paper_1711_05017_b200 import _lib

    hb = np.zeros(4)
    _lib.check(_lib.LIB.gf_measure_stalls(5.0, 500.0, _lib.dptr(hb)))
    st["platform_stalls"] = {"seconds": 5.0, "max_gap_us": r4(hb[0]), "gaps_over_500us_per_sm": [int(hb[1]), int(hb[2])],
                             "probe": "clock-only warp per SM, no host interaction"}
    if cpu_ok:
        C1h, C2h = np.asarray(W1), np.asarray(W2)
        c, dom, dcell = g.center(), g.delta_omega(), 1.0 / (g.node_count * g.cell_volume)
        from paper_1711_05017_b200.energy import Configuration, evaluate

        idx = [0, frames // 3, frames // 2, frames - 1]
        with_s = []
        for i in idx:
            ev = evaluate(f5[0], f5[1], Configuration(R5[i], t5[i]))
            with_s.append(np.concatenate([[ev.score.real], ev.force, ev.torque]))
        tp = np.array([t5[i] - c + R5[i] @ c for i in idx])
        from concurrent.futures import ThreadPoolExecutor

        import oracle

        with ThreadPoolExecutor(max_workers=4) as pool:
            want = list(pool.map(lambda k: ref_cascade(C1h, C2h, False, dom, dcell, R5[idx[k]], tp[k], c),
                                 range(len(idx))))
            l1 = list(pool.map(lambda k: oracle.cascade_term_scales(C1h, C2h, False, dom, dcell, R5[idx[k]], tp[k], c),
                               range(len(idx))))
        want = np.array([np.concatenate([[w_[0].real], w_[1:4].real, w_[4:7].real]) for w_ in want])
        parity["C5"] = parity_entry(np.array(with_s), want, np.asarray(l1).real, "oracle/_ref _core.cascade_3d")
        t0 = time.perf_counter()
        for k in range(2):
            ref_cascade(C1h, C2h, False, dom, dcell, R5[idx[k]], tp[k], c)
        st["cpu"] = {"value": r4(2 / (time.perf_counter() - t0)), "unit": "queries/s", "cores": 1,
                     "kind": "reference", "per_query_ms": r4((time.perf_counter() - t0) / 2 * 1e3)}
    del f5, sess, W1, W2, L1, L2
    torch.cuda.empty_cache()
    return st


def stage_window(args, parity, cpu_ok):
    """Stage 2: forward DFT + truncation + centring of a 256^3 complex128
    field to the w = 96 window (spectral.forward_dft / truncate /
    center_window); parity at 128^3 against the numpy restatement."""
    import torch

    from paper_1711_05017_b200.descriptor import ComplexField, SampleGrid
    from paper_1711_05017_b200.spectral import forward_window

    hbm = float(_peaks()["hbm_gbs"])
    dev = torch.device("cuda", torch.cuda.current_device())
    gen = torch.Generator(device=dev)
    gen.manual_seed(SEED)
    gw = SampleGrid(3, (256,) * 3, (-1.0,) * 3, 2.0 / 256)
    fw = ComplexField(gw, torch.randn(256 ** 3, dtype=torch.complex128, device=dev, generator=gen))
    ms = _time_ms(lambda: forward_window(fw, 96))
    alg = 16.0 * 256 ** 3 + 16.0 * 96 ** 3
    st = {"ms": r4(ms), "roofline": {"bound": "hbm", "achieved": r4(alg / (ms * 1e-3) / 1e9), "peak": hbm,
                                     "unit": "GB/s", "frac": r4(alg / (ms * 1e-3) / 1e9 / hbm)}}
    if cpu_ok:
        import oracle

        fh = fw.values.reshape((256,) * 3)
        t0 = time.perf_counter()
        A = oracle.forward_dft(fh, (256,) * 3, (-1.0,) * 3, 2.0 / 256)
        want = oracle.center_window(A, (256,) * 3, (-1.0,) * 3, 2.0 / 256, 96)
        st["cpu"] = {"value": r4((time.perf_counter() - t0) * 1e3), "unit": "ms", "cores": 1, "kind": "port"}
        got = forward_window(fw, 96).cpu().numpy()
        parity["W"] = {"rel": r4(np.max(np.abs(got - want)) / np.max(np.abs(want))), "n": int(want.size),
                       "vs": "numpy restatement of forward_dft + center_window"}
    del fw
    torch.cuda.empty_cache()
    return st


def stage_density(args, fp64_peak, parity, cpu_ok):
    """Stage 1: affinity_field of the C1 bored block at 64^3 and of the gear
    at 128^3, with the FP64 work counted (~200 FP64 flops per node-element
    pair) against the FP64 pipe measured in this run; flags
    and stats at 32^3 against the oracle's C restatement."""
    import torch

    from paper_1711_05017_b200.descriptor import affinity_field

    st = {}
    for key, scene, n in (("peg64", "peg_in_hole", 64), ("gear128", "gear_pair", 128)):
        sc = scenes_mod().get_scene(scene)
        gd = sc.grid(n)
        affinity_field(sc.fixed, gd, sc.kernel)
        dt = None
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fd = affinity_field(sc.fixed, gd, sc.kernel)
            d1 = time.perf_counter() - t0
            dt = d1 if dt is None else min(dt, d1)
        nf = len(sc.fixed.mesh.faces)
        pairs = gd.node_count * nf
        dev_s = fd.stats["seconds_distance"] + fd.stats["seconds_sweep"]
        st[key] = {"ms": r4(dt * 1e3), "pairs_per_s": r4(pairs / dt), "faces": nf,
                   "frac_fp64": r4(200.0 * pairs / dev_s / 1e12 / fp64_peak)}
    if cpu_ok:
        import oracle

        sc = scenes_mod().get_scene("gear_pair")
        g = sc.grid(32)
        f = affinity_field(sc.fixed, g, sc.kernel)
        want, flags, stats, _, _ = oracle.affinity_values(*sc.fixed.element_arrays(), g.dims, g.origin, g.spacing)
        vals = np.asarray(f.values)
        parity["D"] = {"flags_equal": f.flags == flags,
                       "stats_equal": all(f.stats[k] == stats[k] for k in ("excluded", "eta_clamped", "worst_residual",
                                                                           "unresolved_nodes", "inside_nodes")),
                       "rel": r4(np.max(np.abs(vals - want)) / np.max(np.abs(want))), "n": int(g.node_count),
                       "vs": "oracle C restatement (gear 32^3)"}
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
        st["cpu"] = {"value": r4(gc.node_count * len(m.faces) / dt), "unit": "node-face pairs/s", "cores": 1,
                     "kind": "reference"}
    return st


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
    ap.add_argument("--sweep-poses", type=int, default=1000000)
    ap.add_argument("--stage-cpu-seconds", type=float, default=3.0)
    ap.add_argument("--haptic-frames", type=int, default=10000)
    ap.add_argument("--field-n", type=int, default=512)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.warmup < 3 and args.impl == "b200":
        print("note: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_engine(args)


if __name__ == "__main__":
    sys.exit(main())
