"""Time config 5b batches (count systems of N=1024) for several worker counts."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--count", type=int, default=128)
    ap.add_argument("--workers", default="1,4,8,16,32")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2311_14616_b200 import configs, mpir
    n, count = a.n, a.count
    base = [configs.batch_system(n, i) for i in range(count)]
    adev = torch.from_numpy(np.concatenate(base)).cuda()
    bdev = torch.ones((count, n), dtype=torch.float64, device="cuda")
    for w in a.workers.split(","):
        os.environ["MPIRG_BATCH_WORKERS"] = w
        mpir.batch_solve(adev[: 4 * n * n], bdev[:4], factor="single", resid_term=False,
                         ce=10.0, litmax=10)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = mpir.batch_solve(adev, bdev, factor="single", resid_term=False, ce=10.0,
                                litmax=10)
        dt = time.perf_counter() - t0
        ok = sum(r["status"] == 0 for r in reps)
        print(f"workers={w:>3} count={count} n={n} wall={dt * 1e3:8.1f} ms "
              f"device={mpir.batch_solve.last_device_ms:8.1f} ms "
              f"per-system={dt / count * 1e3:6.2f} ms ok={ok}", flush=True)


if __name__ == "__main__":
    main()
