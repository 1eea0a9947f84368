"""Golden asset directory written by the UNMODIFIED reference CLI.

Run in the build container (needs /root/reference):
    python tests/golden/make_manifest_golden.py

Builds the reference like make_golden.py, runs its own
`geofield.cli.main(["precompute", "--scene", "peg3d", "--grid", "16",
"--modes", "512", ...])` into tests/golden/manifest_peg3d16/, then loads
that directory through the reference's `load_assets` and records
`evaluate` at a few poses (and the reference's precompute kernel and grid)
in manifest_peg3d16_evals.npz.  Fixtures are committed; /root/reference is
never read at test time.
"""

import importlib.util
import os
import shutil

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "manifest_peg3d16")


def main():
    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(HERE, "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    mg.build_reference()
    from geofield import backend
    from geofield.cli import load_assets, main as cli_main
    from geofield.energy import Configuration, evaluate

    assert backend.current() == "core"
    if os.path.exists(OUT):
        shutil.rmtree(OUT)
    assert cli_main(["precompute", "--scene", "peg3d", "--grid", "16", "--modes", "512", "--out", OUT]) == 0
    man, fixed, moving = load_assets(OUT)
    rng = np.random.default_rng(20260814)
    poses, rows = [], []
    for k in range(4):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        w, x, y, z = q
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                      [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                      [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
        if k == 0:
            R = np.eye(3)
        t = rng.uniform(-0.2, 0.2, size=3)
        for mp in (None, 512):
            ev = evaluate(fixed, moving, Configuration(R, t), m_prime=mp)
            poses.append(np.concatenate([R.ravel(), t, [mp or 0]]))
            rows.append(np.concatenate([[ev.energy], ev.force, ev.torque]))
    np.savez(os.path.join(HERE, "manifest_peg3d16_evals.npz"), poses=np.array(poses), evals=np.array(rows))
    print("wrote", OUT, sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
