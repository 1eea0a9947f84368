"""Asset directories on the GPU (assets.py): the reference-written golden
manifest loads straight to the device and evaluates to the reference's
recorded EnergyEvals; a directory precomputed here is deterministic, has the
reference's manifest layout, and matches the reference's files (flags bit
for bit, complex64 payloads to float tolerance)."""

import json
import os

import numpy as np
import pytest

from paper_1711_05017_b200 import assets, backend
from paper_1711_05017_b200.descriptor import read_field
from paper_1711_05017_b200.energy import Configuration, evaluate
from paper_1711_05017_b200.spectral import read_spectrum

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(__file__), "golden")
GOLD = os.path.join(HERE, "manifest_peg3d16")
EVALS = np.load(os.path.join(HERE, "manifest_peg3d16_evals.npz"))


def _check_evals(fixed, moving, rtol):
    for pose, want in zip(EVALS["poses"], EVALS["evals"]):
        R, t, mp = pose[:9].reshape(3, 3), pose[9:12], int(pose[12]) or None
        ev = evaluate(fixed, moving, Configuration(R, t), m_prime=mp)
        got = np.concatenate([[ev.energy], ev.force, ev.torque])
        np.testing.assert_allclose(got, want, rtol=rtol, atol=rtol * np.max(np.abs(want)))


@pytest.mark.parametrize("prec,rtol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_golden_directory_on_device_matches_reference_evals(prec, rtol):
    prev = backend.precision()
    backend.set_precision(prec)
    try:
        _, fixed, moving = assets.load_assets(GOLD, device=True)
        assert fixed.spectrum._dev is not None and fixed.spectrum._host is None
        _check_evals(fixed, moving, rtol)
    finally:
        backend.set_precision(prev)


def test_precompute_matches_reference_directory(tmp_path):
    out1, out2 = tmp_path / "a", tmp_path / "b"
    man1 = assets.precompute(str(out1), 16, scene="peg3d", modes=512)
    man2 = assets.precompute(str(out2), 16, scene="peg3d", modes=512)
    assert man1["parts"] == man2["parts"]  # deterministic: identical artifact hashes
    gold = json.loads(open(os.path.join(GOLD, "manifest.json")).read())
    assert man1.keys() == gold.keys() and man1["grid"] == gold["grid"] and man1["kernel"] == gold["kernel"]
    for name, part in gold["parts"].items():
        mine = man1["parts"][name]
        assert {k: v for k, v in mine.items() if k != "sha256"} == {k: v for k, v in part.items() if k != "sha256"}
        for rel in part["sha256"]:
            a, b = os.path.join(GOLD, rel), str(out1 / rel)
            if rel.endswith(".gfld"):
                fa, fb = read_field(a), read_field(b)
                assert fa.flags == fb.flags
                np.testing.assert_allclose(fb.values, fa.values, atol=1e-6 * np.max(np.abs(fa.values)))
            else:
                sa, sb = read_spectrum(a), read_spectrum(b)
                np.testing.assert_allclose(sb.amplitudes, sa.amplitudes, atol=1e-6 * np.max(np.abs(sa.amplitudes)))
    backend.set_precision("fp64")
    try:
        _, fixed, moving = assets.load_assets(str(out1))
        _check_evals(fixed, moving, 1e-5)
    finally:
        backend.set_precision("fp32")


def test_solid_manifests_merge_and_mismatch(tmp_path):
    """Per-solid precompute merges fixed and moving parts into one manifest
    when grid and kernel agree (cli.py:208-216), and refuses otherwise."""
    out = tmp_path / "m3"
    assets.precompute(str(out), 8, solid="box", role="fixed", domain=6.0)
    man = assets.precompute(str(out), 8, solid="icosphere", role="moving", domain=6.0)
    assert set(man["parts"]) == {"fixed", "moving"}
    assert man["parts"]["fixed"]["solid_kind"] == "file"  # named by role, as the reference does
    _, fixed, moving = assets.load_assets(str(out))
    ev = evaluate(fixed, moving, Configuration(np.eye(3), [0.0, 0.0, 0.75]))
    assert ev.force.shape == (3,) and ev.torque.shape == (3,) and np.isfinite(ev.energy)
    out2 = tmp_path / "m3b"
    assets.precompute(str(out2), 8, solid="box", role="fixed", domain=6.0)
    with pytest.raises(ValueError, match="different grid or kernel"):
        assets.precompute(str(out2), 8, solid="icosphere", role="moving", domain=8.0)
