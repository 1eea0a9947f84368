"""Build libgeofield_b200.so in-tree with nvcc for sm_100a (no JIT, no cache).

Usage: python paper_1711_05017_b200/_build.py [-v] [-f]   (or __graft_entry__.build())
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "libgeofield_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-I", os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def _ext_path():
    import sysconfig

    return os.path.join(HERE, "_gf_fast" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_pyfast(force=False):
    """The CPython binding of the per-frame session query (csrc/pyfast.c),
    built with the host C compiler against this interpreter and numpy."""
    import sysconfig

    import numpy

    src, out = os.path.join(HERE, "csrc", "pyfast.c"), _ext_path()
    if not force and os.path.exists(out) and os.path.getmtime(out) > os.path.getmtime(src):
        return out
    cc = os.environ.get("CC", "gcc")
    subprocess.run([cc, "-O2", "-shared", "-fPIC", "-Wall", "-I", sysconfig.get_paths()["include"],
                    "-I", numpy.get_include(), "-o", out, src], check=True)
    return out


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return any(os.path.getmtime(p) > t for p in deps)


# files whose float64 decision path must round every operation separately
# (bit-exact distances / exclusion / subdivision vs the reference's no-FMA
# x86-64 build)
NO_FMA = {"density.cu"}


def build(verbose=False, force=False):
    build_pyfast(force)
    if not force and not needs_build():
        return OUT
    from concurrent.futures import ThreadPoolExecutor

    objdir = os.path.join(HERE, "csrc", "_obj")
    os.makedirs(objdir, exist_ok=True)
    for stale in glob.glob(os.path.join(objdir, "*.o")):
        os.remove(stale)
    cmds, objs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        flags = [f for f in FLAGS if f != "-shared"]
        if os.path.basename(src) in NO_FMA:
            flags.append("-fmad=false")
        cmd = [NVCC, *flags, "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        cmds.append(cmd)
        objs.append(obj)
    # one nvcc per translation unit, concurrently (fft.cu / field.cu dominate)
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as pool:
        for r in pool.map(lambda c: subprocess.run(c, check=True), cmds):
            pass
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT, *objs], check=True)
    return OUT


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(OUT)
