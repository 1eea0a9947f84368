"""The reference's own hot-path test modules, unmodified, against this engine.

`make -C oracle ref` copies /root/reference/pkg/tests/{conftest, test_energy,
test_spectral, test_descriptor, test_backend, test_scenes, test_solids}.py
(test_acceptance imports the out-of-scope CLI at module level; its hot-path
criteria are restated in test_acceptance_gpu.py) and the reference's
slow-path checker (geofield/oracle.py) into oracle/_ref/suite/ (git-ignored;
it travels to the GPU box with the built libraries).  They run here in a
child pytest with `geofield` resolving to this package
(tests/reference_suite/geofield) and the float64 engine selected
(GEOFIELD_PRECISION=fp64: the reference's own tolerances, 1e-9 .. 1e-12).

Named expected failures: the reference tests of its CPU core / numpy
fallback switch (test_backend.py).  This engine has one backend and refuses
`use("fallback")` by design, so tests that compare the two CPU paths cannot
run; everything else must pass.
"""

import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "oracle", "_ref", "suite")
SHIM = os.path.join(ROOT, "tests", "reference_suite")

# test ids (module::name, parametrisation stripped) allowed to fail, and why
EXPECTED = {
    "test_backend.py::test_use_validates": "core/fallback switch: the engine has no CPU fallback backend",
    "test_backend.py::test_distance_parity_2d": "compares the CPU core with the numpy fallback",
    "test_backend.py::test_distance_parity_3d": "compares the CPU core with the numpy fallback",
    "test_backend.py::test_winding_parity": "compares the CPU core with the numpy fallback",
    "test_backend.py::test_affinity_field_parity": "compares the CPU core with the numpy fallback",
    "test_backend.py::test_cascade_parity": "compares the CPU core with the numpy fallback",
    "test_backend.py::test_cascade_parity_3d": "compares the CPU core with the numpy fallback",
    "test_scenes.py::test_registry": "the registry also holds the BASELINE.json scenes (peg_in_hole, gear_pair, ...)",
}


def test_reference_suites_unmodified(tmp_path):
    if not os.path.isdir(SUITE):
        pytest.skip("oracle/_ref/suite not built (make -C oracle ref in the build container)")
    report = tmp_path / "suite.xml"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([SHIM, ROOT, os.environ.get("PYTHONPATH", "")]),
               GEOFIELD_REFERENCE_SUITE=SUITE, GEOFIELD_PRECISION="fp64")
    proc = subprocess.run([sys.executable, "-m", "pytest", SUITE, "-q", "-p", "no:cacheprovider",
                           f"--junitxml={report}", "--rootdir", SUITE], capture_output=True, text=True, env=env,
                          cwd=SUITE, timeout=1800)
    assert report.exists(), proc.stdout[-3000:] + proc.stderr[-3000:]
    failed, passed = [], 0
    for case in ET.parse(report).getroot().iter("testcase"):
        name = f"{os.path.basename(case.get('file') or case.get('classname', '').replace('.', '/') + '.py')}::" \
               f"{case.get('name').split('[')[0]}"
        bad = case.find("failure") is not None or case.find("error") is not None
        if bad and name not in EXPECTED:
            failed.append(name)
        elif not bad and case.find("skipped") is None:
            passed += 1
    assert not failed, f"reference tests failing on the engine: {sorted(set(failed))}\n{proc.stdout[-4000:]}"
    assert passed >= 100, proc.stdout[-3000:]  # energy + spectral + descriptor + scenes + solids
