"""Asset I/O straight to the device.

Mirrors the reference's precompute / manifest / load path
(/root/reference/pkg/src/geofield/cli.py:84-227): one manifest.json per
asset directory, GFLD field and GSPC spectrum files, sha256 of every tracked
file checked on load.  Files and manifest are byte-compatible with the
reference (same header layout, complex64 payload, same manifest keys and
JSON formatting), so a directory written here loads in the reference and
vice versa.

What changes is where the work runs:

* `precompute` builds the affinity field on the GPU (`affinity_field` ->
  `gf_affinity_grid`), its spectra with the GPU transform (`forward_dft`),
  and writes the files from those device results;
* `load_assets(..., device=True)` reads each GSPC payload (complex64 at a
  fixed header offset) into pinned host memory and copies it to the device
  in one DMA, upcast to complex128 there; the window centre phase is then
  applied on the device in float64 by `center_window_device` when a window
  is first requested.  No complex128 host array is ever built.
"""

from __future__ import annotations

import hashlib
import json
import os
import time

import numpy as np

from . import _lib, containers
from .descriptor import KernelSpec, SampleGrid, affinity_field, write_field
from .energy import PartAsset
from .spectral import Spectrum, TruncatedSpectrum, VectorSpectrum, read_spectrum, truncate, write_spectrum

__all__ = ["precompute", "precompute_part", "load_manifest", "load_assets", "read_spectrum_device", "sha256_file",
           "BUILTIN_SOLIDS"]

def _builtin_solids():
    from .scenes import box_mesh, icosphere, lbracket

    # the reference CLI's named solids (cli.py:26-30)
    return {
        "box": lambda: box_mesh((0.8, 1.0, 0.6)),
        "icosphere": lambda: icosphere(0.5),
        "lbracket": lambda: lbracket(0.4),
    }


BUILTIN_SOLIDS = ("box", "icosphere", "lbracket")


def sha256_file(path):
    """Streaming sha256 of a file (cli.py:43-48)."""
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for chunk in iter(lambda: fh.read(1 << 22), b""):
            h.update(chunk)
    return h.hexdigest()


def _manifest_path(path):
    return os.path.join(path, "manifest.json") if os.path.isdir(path) else path


def load_manifest(path):
    """Parse a manifest and verify every tracked file's hash (cli.py:88-99)."""
    path = _manifest_path(path)
    with open(path, "r", encoding="utf-8") as fh:
        man = json.load(fh)
    base = os.path.dirname(os.path.abspath(path))
    for part in man["parts"].values():
        for rel, want in part["sha256"].items():
            if sha256_file(os.path.join(base, rel)) != want:
                raise ValueError(f"hash mismatch for {rel}")
    return man, base


def _read_header(fh):
    d, dims, origin, spacing, count = containers.unpack_header(fh, b"GSPC")
    return SampleGrid(d, dims, origin, spacing), int(count)


def read_spectrum_device(path):
    """GSPC file -> Spectrum / TruncatedSpectrum whose amplitudes live on the
    device.  The complex64 payload is read into pinned memory and moved in
    one host->device copy; the complex128 upcast happens on the GPU."""
    import torch

    dev = _lib.ensure_device()
    with open(path, "rb") as fh:
        grid, m_prime = _read_header(fh)
        pinned = torch.empty(m_prime, dtype=torch.complex64, pin_memory=True)
        view = pinned.numpy().view(np.uint8)
        got = fh.readinto(memoryview(view))
        if got != 8 * m_prime:
            raise ValueError(f"truncated GSPC payload in {path}")
    amps = pinned.to(f"cuda:{dev}", non_blocking=True).to(torch.complex128)
    if m_prime == grid.node_count:
        return Spectrum(grid, amps)
    return TruncatedSpectrum(grid, m_prime, amps)


def load_assets(manifest_path, device=True):
    """Rebuild the (fixed, moving) PartAsset pair from a manifest directory
    (cli.py:102-130).  device=True keeps every spectrum on the GPU."""
    man, base = load_manifest(manifest_path)
    read = read_spectrum_device if device else read_spectrum
    assets = {}
    for name, part in man["parts"].items():
        spec = read(os.path.join(base, part["spectrum"]))
        trunc = read(os.path.join(base, part["truncated"])) if part.get("truncated") else None
        vec = None
        if part.get("vector"):
            vec = VectorSpectrum([read(os.path.join(base, p)) for p in part["vector"]])
        assets[name] = PartAsset(name, spec, truncated=trunc, vector=vec, movable=part["movable"],
                                 solid_box=(np.asarray(part["bbox"][0]), np.asarray(part["bbox"][1])))
    fixed = next((a for a in assets.values() if not a.movable), None)
    moving = next((a for a in assets.values() if a.movable), None)
    if fixed is None or moving is None:
        raise ValueError("manifest needs one fixed and one movable part")
    return man, fixed, moving


def precompute_part(name, solid, grid, kernel, movable, out_dir, m_prime=None, log=None):
    """Field -> spectra -> files for one part; returns its manifest entry
    (cli.py:133-175).  Field and transforms run on the GPU."""
    t0 = time.perf_counter()
    fld = affinity_field(solid, grid, kernel)
    t1 = time.perf_counter()
    asset = PartAsset.from_field(name, fld, movable=movable, solid_box=solid.bbox)
    t2 = time.perf_counter()
    files = {"field": f"{name}.field.gfld", "spectrum": f"{name}.scalar.gspc"}
    write_field(fld, os.path.join(out_dir, files["field"]))
    write_spectrum(asset.spectrum, os.path.join(out_dir, files["spectrum"]))
    trunc_rel = None
    if m_prime:
        trunc_rel = f"{name}.trunc.gspc"
        write_spectrum(truncate(asset.spectrum, m_prime), os.path.join(out_dir, trunc_rel))
    vec_rels = []
    if movable:
        for k, comp in enumerate(asset.vector.components):
            rel = f"{name}.moment{k}.gspc"
            write_spectrum(comp, os.path.join(out_dir, rel))
            vec_rels.append(rel)
    t3 = time.perf_counter()
    tracked = [files["field"], files["spectrum"]] + vec_rels + ([trunc_rel] if trunc_rel else [])
    if log is not None:
        log(f"[{name}] field {t1 - t0:.2f}s  transforms {t2 - t1:.2f}s  write {t3 - t2:.2f}s")
    return {
        "solid_kind": "builtin" if name in BUILTIN_SOLIDS else "file",
        "movable": movable,
        "bbox": [np.asarray(solid.bbox[0]).tolist(), np.asarray(solid.bbox[1]).tolist()],
        "field": files["field"],
        "spectrum": files["spectrum"],
        "truncated": trunc_rel,
        "vector": vec_rels,
        "sha256": {rel: sha256_file(os.path.join(out_dir, rel)) for rel in tracked},
    }


def precompute(out_dir, grid_n, scene=None, solid=None, role="fixed", modes=None, kernel=None, domain=None,
               log=None):
    """Write a reference-compatible asset directory (cli.py:178-227).

    Either `scene` (a registered scene name: both parts) or `solid` (a
    built-in solid name or a Solid object) with `role` ("fixed"/"moving"),
    merged into an existing manifest with the same grid and kernel."""
    from .scenes import get_scene, grid_for_pair

    if scene is not None:
        sc = get_scene(scene)
        kernel = kernel or sc.kernel
        grid = grid_for_pair(sc.fixed, sc.moving, grid_n, domain=domain or sc.domain, center=sc.grid_center)
        parts = {"fixed": (sc.fixed, False), "moving": (sc.moving, True)}
    else:
        if solid is None:
            raise ValueError("need a scene or a solid")
        kernel = kernel or KernelSpec()
        if isinstance(solid, str):
            solid = _builtin_solids()[solid]()
        grid = grid_for_pair(solid, solid, grid_n, domain=domain)
        parts = {role: (solid, role == "moving")}
    os.makedirs(out_dir, exist_ok=True)
    man = {"version": 1, "scene": scene,
           "grid": {"dimension": grid.dimension, "dims": list(grid.dims), "origin": list(grid.origin),
                    "spacing": grid.spacing},
           "kernel": {"sigma": kernel.sigma, "lambda_in": kernel.lambda_in, "lambda_out": kernel.lambda_out},
           "modes": modes,
           "parts": {}}
    mpath = _manifest_path(out_dir)
    if os.path.exists(mpath) and scene is None:
        with open(mpath, "r", encoding="utf-8") as fh:
            old = json.load(fh)
        if old["grid"] != man["grid"] or old["kernel"] != man["kernel"]:
            raise ValueError("existing manifest has different grid or kernel")
        man = old
    for name, (s, movable) in parts.items():
        man["parts"][name] = precompute_part(name, s, grid, kernel, movable, out_dir, modes, log=log)
    with open(mpath, "w", encoding="utf-8") as fh:
        json.dump(man, fh, indent=1, sort_keys=True)
    return man
