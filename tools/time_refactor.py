"""Wall/device time of refactor from a device pointer vs from pinned host memory (cfg2a)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_2311_14616_b200 import _lib as L, mpir
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    a = mpir.build_operator(n, 800.0)
    f = mpir.Factorization(a, working="double", factor="single", resid_term=False)
    lib = L.lib()
    host = torch.from_numpy(np.asfortranarray(a).ravel(order="F")).pin_memory()
    dev = host.cuda()
    err = L.mpirg_error()
    for name, ptr, on_dev in (("device", dev.data_ptr(), 1), ("host", host.data_ptr(), 0)):
        ts = []
        for i in range(6):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            L.check(lib.mpirg_factorization_refactor(f._h, C.c_void_p(ptr), on_dev, C.byref(err)),
                    err)
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"{name}: wall ms {['%.2f' % t for t in ts]} last factor_ms "
              f"{lib.mpirg_factorization_last_factor_ms(f._h):.2f}", flush=True)


if __name__ == "__main__":
    main()
