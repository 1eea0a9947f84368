import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_05017_b200 import _lib
_lib.ensure_device(0)
for blocks in (1, 148, 444, 1024):
    h, d = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.LIB.gf_measure_launch(2000, blocks, ctypes.byref(h), ctypes.byref(d)))
    print(f"blocks={blocks:5d} host {h.value:6.2f} us/launch  device {d.value:6.2f} us/launch")
