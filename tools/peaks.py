"""Print the live FFMA / DFMA microbenchmark rates of this GPU."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_14616_b200 import lib
L = lib()
for name in ("mpirg_ffma_peak", "mpirg_dfma_peak"):
    tf, ms = C.c_double(), C.c_double()
    rc = getattr(L, name)(C.byref(tf), C.byref(ms))
    print(name, rc, f"{tf.value:.2f} TFLOP/s", f"{ms.value:.3f} ms")
