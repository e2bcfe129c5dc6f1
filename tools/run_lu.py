"""Run one (or a few) device LU factorizations for profiling (ncu target)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--prec", type=int, default=1)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--solve", action="store_true", help="also run the IR solve (cfg2a)")
    ap.add_argument("--randn", type=int, default=-1, help="N(0,1) matrix with this seed")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2311_14616_b200 import kernels, lib
    L = lib()
    n = a.n
    buf = np.empty(n * n)
    if a.randn >= 0:
        L.mpirg_gen_normal_matrix(n, n, a.randn, buf.ctypes.data)
    else:
        L.mpirg_gen_greens_operator(n, 800.0, buf.ctypes.data)
    src = torch.from_numpy(buf).cuda()
    if a.prec == 1:
        src = src.float()
    elif a.prec == 2:
        src = src.half().view(torch.int16)
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    for _ in range(a.reps):
        d = src.clone()
        kernels.lu_factor(d, ipiv, n)
    torch.cuda.synchronize()
    if a.solve:
        import bench  # noqa: F401
        from paper_2311_14616_b200 import mpir
        b = np.empty(n)
        L.mpirg_gen_normal_matrix(n, 1, 0, b.ctypes.data)
        f = mpir.Factorization(buf.reshape(n, n).T, working="double", factor="single",
                               resid_term=False)
        f.solve(b, ce=10.0, litmax=20)
    print("ok")


if __name__ == "__main__":
    main()
