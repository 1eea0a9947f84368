import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1711_05017_b200 import _lib
_lib.ensure_device(0)
out = np.zeros(4)
_lib.check(_lib.LIB.gf_measure_roundtrip(2000, _lib.dptr(out)))
print(f"launch+mapped completion p50 {out[0]:.2f} us | pre-armed WaitValue release p50 {out[1]:.2f} us | "
      f"GPU mapped read {out[2]:.0f} ns | mapped write+fence.sys {out[3]:.0f} ns")
