"""bench.py --gpus N (N > 1) / --config cfg5a --dist: BASELINE.json configs[4](a).

Workload: A = I - G, N = 65536 (fp64, 34.4 GB, resident on rank 0 like the
single-GPU handle's a_high), b = ones(N), <TW,TF,TR> = <fp64, fp32, fp64>,
ce = 10, litmax = 10. One "step" = the whole time-to-solution through
``dist.DistributedFactorization``:
    rank 0: ||A||_1 + demotion to fp32            (mpirg_factorization_cast)
    scatter of the owned fp32 column blocks        (1-D block-cyclic, block 512)
    LU on all ranks, panels + pivots broadcast     (mpirg_dlu_factor: C++ loop,
                                                    NCCL over NVLink, TMA-fed
                                                    paired update per rank)
    gather of the factors to rank 0
    rank 0: ir_solve_report                        (mpirg_ir_solve)
``value`` = seconds per step, CUDA events on each rank's stream between
barriers, max over ranks; ``scaling`` is "strong" (the one N = 65536 system is
fixed as N grows). ``e2e`` = the same call chain from pinned HOST memory on
rank 0 (H2D of the 34.4 GB matrix and of b, D2H of x inside the timed region).
The line also carries rank 0's single-GPU time for the same workload
(``single_gpu_same_workload``) so the scaling efficiency can be read off one run.

The reference has no distributed code; the CPU baseline is the
compiled reference at N = 4096 extrapolated (bench.reference_solve).
"""
from __future__ import annotations

import ctypes as C
import statistics
import time

import bench as B


def run_ours(args, world, rank, local):
    import numpy as np
    import torch
    import torch.distributed as tdist
    from paper_2311_14616_b200 import _lib as L
    from paper_2311_14616_b200 import configs, dist as D, mpir
    lib = L.lib()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n = args.n or configs.FULL_N["cfg5a"]
    ce, litmax = 10.0, 10
    if world > 1 and not tdist.is_initialized():
        raise RuntimeError("bench_dist needs the process group (torchrun)")
    comm = D.Comm() if world > 1 else _SoloComm()
    df = D.DistributedFactorization(n, comm, resid_term=False, block_cols=args.block_cols,
                                    device=local)
    tp = mpir.update_parms(None, ce, None, litmax)
    a_pin = b_dev = b_pin = x_pin = None
    if rank == 0:
        # A straight into pinned host memory (one 34 GB copy, used by e2e), then
        # into the handle's a_high through the first refactor
        a_pin = torch.empty(n * n, dtype=torch.float64).pin_memory()
        configs.greens(n, 1.0, a_pin.numpy())
        b_pin = torch.ones(n, dtype=torch.float64).pin_memory()
        x_pin = torch.empty(n, dtype=torch.float64).pin_memory()
        b_dev = b_pin.to(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step(host=False):
        """One time-to-solution; device ms on this rank between the two events."""
        B.barrier(world)
        torch.cuda.synchronize()
        ev0.record()
        if rank == 0:
            df.refactor(a_pin if host else None, a_on_device=not host)
            rep = df.solve(b_pin.to(dev, non_blocking=True) if host else b_dev, tp=tp)
            if host:
                x_pin.copy_(torch.from_numpy(rep["x"]))
        else:
            df.refactor(None)
            rep = None
        ev1.record()
        ev1.synchronize()
        return ev0.elapsed_time(ev1), rep

    # first call: A from the pinned host copy into a_high (also a warm-up)
    t0 = time.perf_counter()
    _, rep = step(host=True)
    first_s = time.perf_counter() - t0
    for _ in range(max(0, args.warmup - 1)):
        step()
    clocks = B.ClockSampler(local).__enter__()
    ms, fac_s = [], []
    B.barrier(world)
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    for _ in range(args.steps):
        m, rep = step()
        ms.append(m)
        fac_s.append(df.factor_s)
    torch.cuda.synchronize()
    B.barrier(world)
    t_wall = time.perf_counter() - t_wall0
    mean_ms = B.max_over_ranks(statistics.mean(ms), world)
    fac_mean_s = B.max_over_ranks(statistics.mean(fac_s), world)
    e2e = None
    if not args.no_e2e:
        e2e_t = []
        for i in range(1 + args.steps):
            B.barrier(world)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            step(host=True)
            if i >= 1:
                e2e_t.append(time.perf_counter() - t0)
        e2e = {"value": B.max_over_ranks(statistics.mean(e2e_t), world), "unit": "s",
               "h2d_bytes_per_step": (n * n + n) * 8, "d2h_bytes_per_step": n * 8,
               "note": "rank 0 holds the host matrix; H2D at the host link rate dominates"}
    clocks.__exit__(None, None, None)

    # the same workload on rank 0's GPU alone (single-GPU LU in the same handle)
    solo = None
    if rank == 0 and world > 1 and not args.no_cpu_baseline:
        err = L.mpirg_error()
        cap = litmax + 1
        rh, dh = (C.c_double * cap)(), (C.c_double * cap)()
        sol = torch.empty(n, dtype=torch.float64, device=dev)
        tt = []
        for i in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            L.check(lib.mpirg_factorization_refactor(df.f._h, None, 1, C.byref(err)), err)
            r1 = L.mpirg_report(sol.data_ptr(), 1, rh, dh, cap, 0, 0, 0, 0.0)
            L.check(lib.mpirg_ir_solve(df.f._h, b_dev.data_ptr(), 1, C.byref(tp), C.byref(r1),
                                       C.byref(err)), err)
            torch.cuda.synchronize()
            tt.append(time.perf_counter() - t0)
        solo = {"value": tt[1], "unit": "s", "steps": 1, "warmup": 1,
                "x_equal_to_distributed": bool(np.array_equal(
                    sol.cpu().numpy().view(np.uint64), rep["x"].view(np.uint64)))}
    B.barrier(world)
    if rank != 0:
        return None
    # size-independent checks of the N = 65536 solution (the oracle LU would need
    # hours): no interchanges, mirror symmetry, distance to the continuum
    # solution, and the oracle's own compensated residual on the host matrix
    x = rep["x"]
    ipiv = df.f.ipiv()
    t = np.arange(n) / (n - 1.0)
    u = np.cos(t) + (1.0 - np.cos(1.0)) / np.sin(1.0) * np.sin(t)
    checks = {"interchanges": int((ipiv != np.arange(n)).sum()),
              "max_abs_x_minus_continuum": float(np.abs(x - u).max()),
              "h2": (1.0 / (n - 1)) ** 2,
              "max_abs_x_minus_reversed": float(np.abs(x - x[::-1]).max())}
    checks.update(B.host_residual_check(a_pin.numpy(), x, np.ones(n), df.f.a_norm1))
    peaks, peak_src = B.measured_peaks()
    ffma, ffma_ms = C.c_double(0.0), C.c_double(0.0)
    lib.mpirg_ffma_peak(C.byref(ffma), C.byref(ffma_ms))
    flops = 2.0 * n ** 3 / 3.0
    lu_tf = flops / fac_mean_s / 1e12
    line = {
        "metric": B.METRIC, "value": mean_ms / 1e3, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64/f32 (TW=f64, TF=f32, TR=f64)",
        "data": "synthetic (A = I - G by the reference's trapezoid rule, greens.cpp:28-59)",
        "config": {"workload": f"cfg5a: N={n}, <f64,f32,f64>, ce={ce}, litmax={litmax}",
                   "n": n, "nb": 64,
                   "parallelism": (f"1-D block-cyclic, block {df.be.block_cols}, "
                                   f"{world} rank(s), panel+pivot broadcast over "
                                   + ("NCCL (mpirg_comm_bcast)" if world > 1 else "nothing (1 rank)")),
                   "l2": "inputs (51 GB) far larger than L2",
                   "a_resident_in_hbm": "rank 0 (fp64); the fp32 blocks are scattered per step"},
        "factor_s": fac_mean_s,
        "iters": len(rep["rhist"]) - 1, "reason": rep["reason"],
        "roofline": {"kernel": "lu (distributed: cast + scatter + panels + broadcasts + "
                               "updates + gather)",
                     "bound": "fp32-ffma", "achieved": lu_tf,
                     "peak": ffma.value * world, "unit": "TFLOP/s",
                     "frac": lu_tf / (ffma.value * world) if ffma.value else None,
                     "traffic": None,
                     "peak_source": f"{world} x fp32 FFMA microbenchmark (mpirg_ffma_peak); "
                                    "TF32/tensor cores excluded by contract",
                     "peak_kind": peak_src},
        "e2e": e2e, "first_call_from_host_s": first_s,
        "gpu_launches": None,
        "clocks": {**clocks.summary(), "window": "timed and e2e steps (nvidia-smi -lms 50)"},
        "wall_s_timed_region": t_wall, "checks": checks,
        "nccl_version": lib.mpirg_comm_version(),
    }
    if solo:
        line["single_gpu_same_workload"] = solo
    if not args.no_cpu_baseline:
        wl = {"n": n, "tw": 0, "tf": 1, "tr": 0, "on_the_fly": -1, "resid_term": False,
              "ce": ce, "litmax": litmax}
        sub = type(args)(**{**vars(args), "config": "cfg5a"})
        line["cpu_baseline"] = B.cpu_baseline(sub, wl, None, None)
    return line


class _SoloComm:
    """World size 1 without a process group (python bench.py --config cfg5a --dist)."""
    rank, size, backend, group = 0, 1, "none", None

    def broadcast(self, t, src):
        pass

    def send(self, *a):
        raise RuntimeError("one rank")

    recv = send
