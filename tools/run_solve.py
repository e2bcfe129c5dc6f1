"""Factor once (cfg2a shape) and run one IR solve, for TRSV/residual profiling."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2311_14616_b200 import lib, mpir
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
L = lib()
a = np.empty(n * n)
L.mpirg_gen_greens_operator(n, 800.0, a.ctypes.data)
b = np.empty(n)
L.mpirg_gen_normal_matrix(n, 1, 0, b.ctypes.data)
f = mpir.Factorization(a.reshape(n, n).T, working="double", factor="single", resid_term=False)
rep = f.solve(b, ce=10.0, litmax=int(sys.argv[2]) if len(sys.argv) > 2 else 20)
print("reason", rep["reason"], "iters", len(rep["rhist"]) - 1, "device_ms", rep["device_ms"])
