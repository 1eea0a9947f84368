"""Probe: affinity_field wall time for the BASELINE meshes at growing grids
(sizes the bench's C3/C4/C5 asset builds need).  Optional argv: name:n ..."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1711_05017_b200 import scenes  # noqa: E402
from paper_1711_05017_b200.descriptor import affinity_field  # noqa: E402

cases = [("gear_pair", 128), ("gear_pair", 256), ("peg_in_hole", 256), ("bolt_nut", 64), ("bolt_nut", 128)]
if len(sys.argv) > 1:
    cases = [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[1:]]
for name, n in cases:
    sc = scenes.get_scene(name)
    g = sc.grid(n)
    for which in ("fixed", "moving"):
        solid = getattr(sc, which)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f = affinity_field(solid, g, sc.kernel)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        nf = len(solid.mesh.faces)
        st = {k: (round(v, 3) if isinstance(v, float) else v) for k, v in f.stats.items()}
        print(f"{name} {which} n={n} faces={nf} {dt:.2f}s pairs/s={g.node_count * nf / dt:.3e} {st}", flush=True)
