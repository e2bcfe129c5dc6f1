"""Debug: GPU LU vs oracle on one case; print differing elements."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import oracle
from helpers import greens, normal_matrix, demote_host, to_dev, from_dev
from paper_2311_14616_b200 import kernels

kind, n, prec = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
nb = int(sys.argv[4]) if len(sys.argv) > 4 else 0
a64 = greens(n, 1.0) if kind == "greens" else normal_matrix(n, 3)
a = demote_host(a64, prec) if prec else a64
st, want, ipw, _, _ = oracle.restatement().lu(a, prec)
d = to_dev(a)
ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
kernels.lu_factor(d, ipiv, n, nb=nb)
got = from_dev(d)
print("ipiv equal", np.array_equal(ipiv.cpu().numpy(), ipw))
gb = got.view(np.uint32 if prec == 1 else np.uint64)
wb = want.view(np.uint32 if prec == 1 else np.uint64)
bad = np.argwhere(gb != wb)
print("ndiff", len(bad))
print("rows", sorted(set(bad[:,0].tolist()))[:20], "cols", sorted(set(bad[:,1].tolist()))[:20])
for i, j in bad[:6]:
    print(i, j, repr(got[i, j]), repr(want[i, j]))
