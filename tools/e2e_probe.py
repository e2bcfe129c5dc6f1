"""cfg2a: refactor + solve from device vs from pinned host memory (wall and factor
ms), to split the e2e overhead; run with MPIRG_LU_TIMELINE=1 for the chain timeline
of the streamed (host) refactor."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_2311_14616_b200 import _lib as L, configs, mpir
    n = 4096
    cfg = configs.config("cfg2a")
    a = cfg["a"].reshape(n, n).T
    f = mpir.Factorization(a, working="double", factor="single", resid_term=False)
    lib = L.lib()
    host = torch.from_numpy(cfg["a"]).pin_memory()
    dev = host.cuda()
    bh = torch.from_numpy(cfg["b"]).pin_memory()
    bd = bh.cuda()
    err = L.mpirg_error()
    tp = L.mpirg_term_params(1.0, 10.0, 0.5, 20)
    rh, dh = (C.c_double * 21)(), (C.c_double * 21)()
    xs = torch.empty(n, dtype=torch.float64).pin_memory()
    xd = torch.empty(n, dtype=torch.float64, device="cuda")
    reps = 2 if os.environ.get("MPIRG_LU_TIMELINE") else 8
    for name, ap, bp, xp, on_dev in (("device", dev, bd, xd, 1), ("host", host, bh, xs, 0)):
        tf, ts, fms = [], [], []
        for i in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            L.check(lib.mpirg_factorization_refactor(f._h, C.c_void_p(ap.data_ptr()), on_dev,
                                                     C.byref(err)), err)
            t1 = time.perf_counter()
            rep = L.mpirg_report(xp.data_ptr(), on_dev, rh, dh, 21, 0, 0, 0, 0.0)
            L.check(lib.mpirg_ir_solve(f._h, C.c_void_p(bp.data_ptr()), on_dev, C.byref(tp),
                                       C.byref(rep), C.byref(err)), err)
            t2 = time.perf_counter()
            if i >= reps // 2:
                tf.append((t1 - t0) * 1e3)
                ts.append((t2 - t1) * 1e3)
                fms.append(lib.mpirg_factorization_last_factor_ms(f._h))
        print(f"{name}: refactor wall {np.mean(tf):.3f} ms (factor_ms {np.mean(fms):.3f}), "
              f"solve wall {np.mean(ts):.3f} ms (device {rep.solve_ms:.3f})", flush=True)


if __name__ == "__main__":
    main()
