"""Asset directories (assets.py) on the host: the reference-written golden
manifest (tests/golden/manifest_peg3d16, made by make_manifest_golden.py)
verifies, loads, and round-trips byte for byte; tampering is detected."""

import json
import os
import shutil

import numpy as np
import pytest

from paper_1711_05017_b200 import assets
from paper_1711_05017_b200.spectral import Spectrum, TruncatedSpectrum, read_spectrum, write_spectrum
from paper_1711_05017_b200.descriptor import read_field, write_field

GOLD = os.path.join(os.path.dirname(__file__), "golden", "manifest_peg3d16")


def test_golden_manifest_verifies_and_loads():
    man, base = assets.load_manifest(GOLD)
    assert man["grid"]["dims"] == [16, 16, 16] and man["modes"] == 512
    man2, fixed, moving = assets.load_assets(GOLD, device=False)
    assert man2 == man
    assert not fixed.movable and moving.movable
    assert isinstance(fixed.spectrum, Spectrum) and isinstance(fixed.truncated, TruncatedSpectrum)
    assert fixed.truncated.m_prime == 512 and fixed.vector is None
    assert len(moving.vector.components) == 3
    np.testing.assert_array_equal(fixed.solid_box[0], man["parts"]["fixed"]["bbox"][0])


def test_files_round_trip_byte_for_byte(tmp_path):
    man, base = assets.load_manifest(GOLD)
    for part in man["parts"].values():
        for rel in part["sha256"]:
            src = os.path.join(base, rel)
            dst = tmp_path / rel
            if rel.endswith(".gspc"):
                write_spectrum(read_spectrum(src), dst)
            else:
                write_field(read_field(src), dst)
            assert assets.sha256_file(dst) == part["sha256"][rel], rel


def test_hash_mismatch_is_detected(tmp_path):
    d = tmp_path / "m"
    shutil.copytree(GOLD, d)
    p = d / "moving.trunc.gspc"
    raw = bytearray(p.read_bytes())
    raw[-1] ^= 1
    p.write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="hash mismatch"):
        assets.load_assets(str(d), device=False)


def test_manifest_needs_both_roles(tmp_path):
    d = tmp_path / "m"
    shutil.copytree(GOLD, d)
    man = json.loads((d / "manifest.json").read_text())
    del man["parts"]["moving"]
    (d / "manifest.json").write_text(json.dumps(man))
    with pytest.raises(ValueError, match="one fixed and one movable"):
        assets.load_assets(str(d), device=False)
