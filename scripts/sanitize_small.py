"""Tiny invocation of every kernel family, for compute-sanitizer runs."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from paper_1711_05017_b200 import backend as be, scenes, parallel
from paper_1711_05017_b200.descriptor import affinity_field, KernelSpec
from paper_1711_05017_b200.energy import PartAsset, evaluate, Configuration, score_field
from conftest import synthetic_window, random_rotation
rng = np.random.default_rng(0)
for w, wrap in ((8, False), (16, True)):
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    for prec in ("fp32", "fp64"):
        be.cascade(C1, C2, wrap, (0.1,) * 3, 1.0, random_rotation(rng), rng.normal(size=3), [0, 0, 0], precision=prec)
        W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
        poses = torch.from_numpy(be.pack_poses(np.stack([random_rotation(rng) for _ in range(5)]), rng.normal(size=(5, 3)))).cuda()
        be.cascade_batch(W1, W2, wrap, (0.1,) * 3, 1.0, [0, 0, 0], poses, precision=prec)
        be.cascade_batch(W1, W2, wrap, (0.1,) * 3, 1.0, [0, 0, 0], poses, precision=prec, serial=True)
peg = scenes.get_scene("peg3d")
g = peg.grid(16)
f1 = affinity_field(peg.fixed, g, KernelSpec())
f2 = affinity_field(peg.moving, g, KernelSpec())
a1 = PartAsset.from_field("a", f1, solid_box=peg.fixed.bbox)
a2 = PartAsset.from_field("b", f2, movable=True, solid_box=peg.moving.bbox)
for mp in (512, None):
    evaluate(a1, a2, Configuration(random_rotation(rng), [0.1, 0.2, 0.0]), mp)
    score_field(a1, a2, random_rotation(rng), mp)
parallel.score_field_slab(a1, a2, random_rotation(rng), None)
rng2 = np.random.default_rng(1)
poly = scenes.random_polygon(rng2, 8)
affinity_field(poly, scenes.grid_for_pair(poly, poly, 16), KernelSpec())
torch.cuda.synchronize()
print("sanitize workload done")
