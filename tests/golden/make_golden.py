"""Generate golden fixtures from the UNMODIFIED reference package.

Run in the build container (needs /root/reference):
    python tests/golden/make_golden.py

It copies /root/reference/pkg to /tmp/gf_refpkg, builds the reference's
Cython core in place (python setup.py build_ext --inplace), imports
`geofield` from there and writes small .npz fixtures next to this script.
Fixtures are committed; /root/reference is never read at test time.
"""

import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "/root/reference/pkg"
DST = "/tmp/gf_refpkg"
SEED = 20260814


def build_reference():
    if not os.path.exists(os.path.join(DST, "src", "geofield")):
        shutil.copytree(SRC, DST)
    so = [f for f in os.listdir(os.path.join(DST, "src", "geofield")) if f.startswith("_core") and f.endswith(".so")]
    if not so:
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=DST, check=True,
                       stdout=subprocess.DEVNULL)
        # setuptools puts the extension under src/ with package_dir; make sure it is importable
        for root, _, files in os.walk(DST):
            for f in files:
                if f.startswith("_core") and f.endswith(".so") and "geofield" not in root:
                    shutil.copy(os.path.join(root, f), os.path.join(DST, "src", "geofield", f))
    sys.path.insert(0, os.path.join(DST, "src"))


def main():
    build_reference()
    import geofield
    from geofield import backend, oracle, scenes
    from geofield.descriptor import IntegrationPolicy, KernelSpec, affinity_field, indicator_field
    from geofield.energy import Configuration, PartAsset, _wrap_mask, evaluate, score_field
    from geofield.spectral import center_window, forward_dft, truncate

    assert backend.current() == "core", "reference core did not build"
    print("reference geofield from", geofield.__file__)
    kernel = KernelSpec(sigma=0.5, lambda_in=1.0, lambda_out=3.0)
    out = {}

    # --- 3D affinity fields (stage 1) on small grids
    peg = scenes.get_scene("peg3d")
    g16 = peg.grid(16)
    for name, solid in (("socket", peg.fixed), ("peg", peg.moving)):
        f = affinity_field(solid, g16, kernel)
        out[f"aff3d_{name}_values"] = f.values
        out[f"aff3d_{name}_flags"] = np.asarray(f.flags, dtype=np.int64)
        out[f"aff3d_{name}_stats"] = np.asarray([f.stats[k] for k in
                                                 ("excluded", "eta_clamped", "worst_residual",
                                                  "unresolved_nodes", "inside_nodes")], dtype=np.float64)
    out["aff3d_grid"] = np.asarray([g16.dims[0], g16.origin[0], g16.spacing])
    ico = scenes.icosphere(0.5, 2)
    box = scenes.box_mesh((0.8, 1.0, 0.6))
    gico = scenes.grid_for_pair(box, ico, 16)
    fi = affinity_field(ico, gico, kernel)
    out["aff3d_ico_values"] = fi.values
    out["aff3d_ico_flags"] = np.asarray(fi.flags, dtype=np.int64)
    out["aff3d_ico_grid"] = np.asarray([gico.dims[0], gico.origin[0], gico.spacing])
    ind = indicator_field(box, gico)
    out["ind3d_box_values"] = ind.values

    # --- 2D affinity field (random polygon, the reference suite's seed)
    rng = np.random.default_rng(SEED)
    fixed2 = scenes.random_polygon(rng, n_vertices=9, r_min=0.45, r_max=0.8)
    moving2 = scenes.random_polygon(rng, n_vertices=7, r_min=0.3, r_max=0.55)
    g2 = scenes.grid_for_pair(fixed2, moving2, 32)
    f2a = affinity_field(fixed2, g2, kernel)
    f2b = affinity_field(moving2, g2, kernel)
    out["aff2d_fixed_values"] = f2a.values
    out["aff2d_fixed_flags"] = np.asarray(f2a.flags, dtype=np.int64)
    out["aff2d_moving_values"] = f2b.values
    out["aff2d_grid"] = np.asarray([g2.dims[0], g2.origin[0], g2.spacing])

    # --- spectra and windows (stage 2) of the peg3d 16^3 fields
    f1 = affinity_field(peg.fixed, g16, kernel)
    f2 = affinity_field(peg.moving, g16, kernel)
    s1 = forward_dft(f1)
    out["spec3d_fixed_full"] = s1.amplitudes
    out["win3d_fixed_m512"] = center_window(truncate(s1, 512))
    out["win3d_fixed_full"] = center_window(s1)

    # --- queries (stage 3): evaluate at generic and lattice poses, full and truncated
    a1 = PartAsset.from_field("fixed", f1, solid_box=peg.fixed.bbox)
    a2 = PartAsset.from_field("moving", f2, movable=True, solid_box=peg.moving.bbox)
    prng = np.random.default_rng(7)
    poses, results = [], []
    for k in range(12):
        q = prng.normal(size=4)
        R = oracle._axis_rotation(3, k % 3, 0.0) if k < 2 else None
        if R is None:
            from geofield.cli import _parse_rotation
            R = _parse_rotation(",".join(str(v) for v in q), 3)
        t = prng.uniform(-0.6, 0.6, 3)
        for mp in (None, 512, 4096):
            res = evaluate(a1, a2, Configuration(R, t), mp)
            poses.append(np.concatenate([R.ravel(), t, [0 if mp is None else mp]]))
            results.append(np.concatenate([[res.score.real, res.score.imag], res.force, res.torque]))
    out["eval3d_poses"] = np.asarray(poses)
    out["eval3d_results"] = np.asarray(results)

    # --- landscape (stage 4) at a generic rotation, truncated and full
    from geofield.cli import _parse_rotation
    Rg = _parse_rotation("0.9,0.2,-0.3,0.25", 3)
    out["field3d_R"] = Rg
    out["field3d_m512"] = score_field(a1, a2, Rg, 512).values
    land_full = score_field(a1, a2, Rg)
    out["field3d_full"] = land_full.values
    out["field3d_wrap_mask"] = land_full.wrap_mask.ravel()

    # --- geometry as the reference builds it (pins the host mirror's scenes)
    out["geom_socket_tri"] = peg.fixed.mesh.triangles
    out["geom_peg_tri"] = peg.moving.mesh.triangles
    out["geom_ico_tri"] = ico.mesh.triangles
    out["geom_box_tri"] = box.mesh.triangles
    out["geom_poly2_a"] = fixed2.polygon.seg_a
    out["geom_poly2_b"] = fixed2.polygon.seg_b
    out["geom_lbracket_tri"] = scenes.lbracket(0.4).mesh.triangles

    path = os.path.join(HERE, "reference_small.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
