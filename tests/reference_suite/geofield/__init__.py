"""`geofield` -> paper_1711_05017_b200, for running the reference's own test
modules unmodified (TEST INFRASTRUCTURE; never imported by the product).

The reference suites import `geofield`, its submodules (`backend`,
`descriptor`, `energy`, `scenes`, `solids`, `spectral`) and its slow-path
checker `geofield.oracle` (/root/reference/pkg/src/geofield/__init__.py:3,
/root/reference/pkg/tests/test_energy.py:7).  Each engine module is
registered under the reference's name; `geofield.oracle` is the reference's
own oracle module, copied unmodified into oracle/_ref/suite by
`make -C oracle ref` (its test infrastructure, like the suites themselves).
"""

import importlib
import importlib.util
import os
import sys

import paper_1711_05017_b200 as _engine
from paper_1711_05017_b200 import *  # noqa: F401,F403  (the reference's public names)

_SUBMODULES = ("backend", "descriptor", "energy", "scenes", "solids", "spectral")
for _name in _SUBMODULES:
    _mod = importlib.import_module(f"paper_1711_05017_b200.{_name}")
    sys.modules[f"geofield.{_name}"] = _mod
    globals()[_name] = _mod

_SUITE = os.environ.get("GEOFIELD_REFERENCE_SUITE", "")
_ORACLE = os.path.join(_SUITE, "_reference_oracle.py")
if os.path.exists(_ORACLE):
    _spec = importlib.util.spec_from_file_location("geofield.oracle", _ORACLE)
    oracle = importlib.util.module_from_spec(_spec)
    sys.modules["geofield.oracle"] = oracle
    _spec.loader.exec_module(oracle)

__version__ = _engine.__version__
