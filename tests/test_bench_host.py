"""bench.py's reference arm runs on the host alone (no GPU): one short run
through the reference's compiled kernel (oracle/_ref) must print one JSON
line with the contract's keys."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_contract_line():
    sys.path.insert(0, ROOT)
    import oracle

    if oracle.ref_core() is None:
        pytest.skip("oracle/_ref not built")
    env = dict(os.environ, RANK="0", WORLD_SIZE="1")
    proc = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                           "--warmup", "1", "--ref-seconds", "0.3"], capture_output=True, text=True, env=env,
                          timeout=300, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr[-2000:]
    line = json.loads(proc.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"


def test_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with two ranks
    (torch.distributed.run, loopback rendezvous): the reference arm's line
    reports n_gpus 2 and only rank 0 prints it."""
    sys.path.insert(0, ROOT)
    import oracle

    if oracle.ref_core() is None:
        pytest.skip("oracle/_ref not built")
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    proc = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                           "--steps", "1", "--warmup", "0", "--ref-seconds", "0.2"], capture_output=True, text=True,
                          env=env, timeout=300, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr[-2000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["impl"] == "reference"
