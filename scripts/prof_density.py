import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_05017_b200 import scenes
from paper_1711_05017_b200.descriptor import affinity_field
sc = scenes.get_scene(sys.argv[1] if len(sys.argv) > 1 else "peg_in_hole")
g = sc.grid(int(sys.argv[2]) if len(sys.argv) > 2 else 64)
for _ in range(2):
    f = affinity_field(sc.fixed, g, sc.kernel)
print(f.stats)
