"""bench.py --config cfg5b: BASELINE.json configs[4](b), the batch of independent systems.

Workload: ``--count`` (default 4096) independent systems of N = 1024,
A_ij ~ U[-1, 1] + N*delta_ij (fp64, seed = system index),
b = ones(N) (BASELINE leaves b unspecified), <TW,TF,TR> = <fp64, fp32, fp64>,
LPS corrections, ce = 10, litmax = 10. Each system is exactly one
MPFactorization + ir_solve_report (the reference's API: one
object per concurrent solve), driven through the C-ABI ``mpirg_batch_ir_solve``.

Sharding (BASELINE: "one batch slice per GPU"): rank r of W solves systems
[r*count/W, (r+1)*count/W) with no collective; ``value`` = seconds for the whole
batch = max over ranks of the device time of one rank's slice (``scaling``
"strong": the total batch is fixed as W grows).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import statistics
import time
from concurrent.futures import ThreadPoolExecutor

import bench as B

N_SYS = 1024
CE, LITMAX = 10.0, 10


def _slice(count, world, rank):
    return rank * count // world, (rank + 1) * count // world


def _generate(lo, hi, n, out_ptr):
    """Seeded systems lo..hi-1 (column-major, fp64) into host memory at out_ptr."""
    from paper_2311_14616_b200 import configs
    g = configs._gen()
    step = n * n * 8

    def one(i):
        g.mpirg_gen_diag_dominant(n, i, float(n), C.c_void_p(out_ptr + (i - lo) * step))

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        list(ex.map(one, range(lo, hi)))


def _workload(args, count):
    return (f"cfg5b: {args.count} independent systems, N={N_SYS}, <f64,f32,f64>, "
            f"ce={CE}, litmax={LITMAX}, b=ones")


def run_ours(args, world, rank, local):
    import numpy as np
    import torch
    from paper_2311_14616_b200 import _lib as L
    lib = L.lib()
    torch.cuda.set_device(local)
    n = N_SYS
    lo, hi = _slice(args.count, world, rank)
    count = hi - lo
    a_pin = torch.empty(count * n * n, dtype=torch.float64).pin_memory()
    _generate(lo, hi, n, a_pin.data_ptr())
    b_pin = torch.ones(count * n, dtype=torch.float64).pin_memory()
    a_dev = a_pin.cuda()
    b_dev = b_pin.cuda()
    sol_dev = torch.empty(count * n, dtype=torch.float64, device="cuda")
    sol_pin = torch.empty(count * n, dtype=torch.float64).pin_memory()
    cfg = L.mpirg_config(0, 1, 0, -1, 0, L.LU_EXACT, 0, local)
    tp = L.mpirg_term_params(1.0, CE, 0.5, LITMAX)
    cap = LITMAX + 1
    rh = np.zeros((count, cap))
    dh = np.zeros((count, cap))
    rlen = np.zeros(count, dtype=np.int32)
    reason = np.zeros(count, dtype=np.int32)
    status = np.zeros(count, dtype=np.int32)
    err = L.mpirg_error()

    def batch(a, b, sol, on_device):
        ms = C.c_double(0.0)
        L.check(lib.mpirg_batch_ir_solve(count, n, C.byref(cfg), a.data_ptr(), b.data_ptr(),
                                         on_device, C.byref(tp), sol.data_ptr(),
                                         rh.ctypes.data, dh.ctypes.data, cap,
                                         rlen.ctypes.data, reason.ctypes.data,
                                         status.ctypes.data, C.byref(ms), C.byref(err)), err)
        return ms.value

    for _ in range(args.warmup):
        batch(a_dev, b_dev, sol_dev, 1)
    torch.cuda.synchronize()
    nclass = len(L.KERNEL_CLASSES)
    ms_k = (C.c_double * nclass)()
    cnt_k = (C.c_int * nclass)()
    lib.mpirg_profile_collect(ms_k, cnt_k, nclass)
    B.barrier(world)
    torch.cuda.synchronize()
    step_ms = []
    t0 = time.perf_counter()
    with B.ClockSampler(local) as clocks:
        for _ in range(args.steps):
            step_ms.append(batch(a_dev, b_dev, sol_dev, 1))
        torch.cuda.synchronize()
    B.barrier(world)
    t_wall = time.perf_counter() - t0
    mean_ms = B.max_over_ranks(statistics.mean(step_ms), world)
    ok = bool((status == 0).all())
    reasons = sorted({L.REASONS[int(r)] for r in reason})
    iters = [int(k) - 1 for k in rlen]

    # per-kernel split from one further, profiled pass (event pairs per launch)
    lib.mpirg_profile_enable(1)
    prof_ms = batch(a_dev, b_dev, sol_dev, 1)
    lib.mpirg_profile_enable(0)
    lib.mpirg_profile_collect(ms_k, cnt_k, nclass)

    # e2e: the same C-ABI call on pinned HOST buffers (H2D of A, b and D2H of x
    # inside the timed region)
    e2e = None
    if not args.no_e2e:
        e2e_t = []
        for i in range(1 + args.steps):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            batch(a_pin, b_pin, sol_pin, 0)
            dt = time.perf_counter() - t1
            if i >= 1:
                e2e_t.append(dt)
        host_same = torch.equal(sol_pin, sol_dev.cpu())
        e2e = {"value": B.max_over_ranks(statistics.mean(e2e_t), world), "unit": "s",
               "h2d_bytes_per_step": count * (n * n + n) * 8,
               "d2h_bytes_per_step": count * (n * 8 + 2 * 8 * cap + 12),
               "x_equal_to_device_path": bool(host_same)}

    peaks, peak_src = B.measured_peaks()
    hbm = float(peaks.get("hbm_gbs", B.HBM_FALLBACK))
    ffma, ffma_ms = C.c_double(0.0), C.c_double(0.0)
    lib.mpirg_ffma_peak(C.byref(ffma), C.byref(ffma_ms))
    work = B.lu_work(n, 64)
    passes = sum(iters)
    kernels = {}
    for i, name in enumerate(L.KERNEL_CLASSES):
        kms = ms_k[i]
        if kms <= 0:
            continue
        d = {"ms_summed_over_streams": kms, "launches": cnt_k[i],
             "ms_per_launch": kms / max(cnt_k[i], 1)}
        if name == "gemm":
            d.update(bound="fp32-ffma", unit="TFLOP/s", peak=ffma.value,
                     achieved=count * work["gemm"] / (kms * 1e-3) / 1e12)
        elif name == "panel":
            d.update(bound="latency (one pivot search per column)", unit="TFLOP/s",
                     peak=ffma.value, achieved=count * work["panel"] / (kms * 1e-3) / 1e12)
        elif name == "cast":
            d.update(bound="hbm", unit="GB/s", peak=hbm,
                     achieved=count * n * n * 12 / (kms * 1e-3) / 1e9)
        elif name in ("trsv_lower", "trsv_upper"):
            d.update(bound="hbm", unit="GB/s", peak=hbm,
                     achieved=cnt_k[i] * n * n / 2.0 * 4 / (kms * 1e-3) / 1e9)
        elif name == "residual":
            d.update(bound="hbm", unit="GB/s", peak=hbm,
                     achieved=cnt_k[i] * n * n * 8 / (kms * 1e-3) / 1e9)
        if d.get("peak"):
            d["frac"] = d["achieved"] / d["peak"]
        kernels[name] = d
    dom = max((k for k in kernels if "achieved" in kernels[k]),
              key=lambda k: kernels[k]["ms_summed_over_streams"])
    dk = kernels[dom]
    roofline = {"kernel": dom, "bound": "hbm" if dk.get("bound") == "hbm" else "tensor",
                "bound_detail": dk.get("bound"), "achieved": dk.get("achieved"),
                "peak": dk.get("peak"), "unit": dk.get("unit"), "frac": dk.get("frac"),
                "traffic": None, "peak_kind": peak_src,
                "note": "systems run concurrently on several streams, so a launch's duration "
                        "includes SM sharing with the other systems' kernels"}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_sample(args, n, seconds=15.0,
                         gpu_x=sol_dev.cpu().numpy().reshape(count, n), gpu_rlen=rlen)
    if rank == 0:
        launches = int(sum(cnt_k[i] for i in range(nclass)))
        line = {
            "metric": B.METRIC, "value": mean_ms / 1e3, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64/f32 (TW=f64, TF=f32, TR=f64)",
            "data": "synthetic (seeded: libstdc++ mt19937_64 per system index, SURVEY 8(d))",
            "config": {"workload": _workload(args, count), "n": n, "systems": args.count,
                       "systems_per_rank": count,
                       "parallelism": f"batch slice per GPU x{world}, no collective",
                       "l2": f"inputs larger than L2 ({count * n * n * 8 / 1e9:.1f} GB of A)",
                       "a_resident_in_hbm": True,
                       "workers_per_gpu": int(os.environ.get("MPIRG_BATCH_WORKERS", "16")),
                       "mode": os.environ.get("MPIRG_BATCH_MODE", "batched kernels (groups of "
                                              + os.environ.get("MPIRG_BATCH_GROUP", "128") + ")")},
            "systems_per_s": args.count / (mean_ms / 1e3),
            "all_ok": ok, "reasons": reasons,
            "iters_min": min(iters), "iters_max": max(iters),
            "profiled_step_ms": prof_ms,
            "roofline": roofline, "kernels": kernels, "ffma_peak_tflops": ffma.value,
            "e2e": e2e, "gpu_launches": launches, "clocks": clocks.summary(),
            "wall_s_timed_region": t_wall,
        }
        if cpu:
            line["cpu_baseline"] = cpu
            if "parity_checked_systems" in cpu:
                line["parity_checked_systems"] = cpu["parity_checked_systems"]
                line["parity_all_systems"] = bool(cpu["parity_all_checked_equal"] and
                                                  cpu["parity_checked_systems"] == args.count)
                line["parity_all_checked_equal"] = cpu["parity_all_checked_equal"]
        print(json.dumps(line), flush=True)


def _ref_solves(impl, n, count, threads):
    """Reference solves of systems 0..count-1 on `threads` host threads, each
    thread a contiguous run of systems; a system's matrix is generated just
    before its solve and only the solves are timed. Returns (max over threads
    of the summed solve seconds, reports)."""
    import numpy as np
    from paper_2311_14616_b200 import configs

    b = np.ones(n)
    chunks = [range(t * count // threads, (t + 1) * count // threads) for t in range(threads)]

    def run(chunk):
        busy, reps = 0.0, []
        for i in chunk:
            a = configs.batch_system(n, i).reshape(n, n).T
            t0 = time.perf_counter()
            reps.append(impl.ir(0, 1, 0, a, b, resid_term=False, ce=CE, litmax=LITMAX))
            busy += time.perf_counter() - t0
        return busy, reps

    with ThreadPoolExecutor(max_workers=threads) as ex:
        out = list(ex.map(run, chunks))
    return max(o[0] for o in out), [r for o in out for r in o[1]]


def cpu_sample(args, n, seconds=15.0, gpu_x=None, gpu_rlen=None):
    """The compiled reference on a bounded sample of the batch, all host cores,
    extrapolated to the whole batch (systems are independent)."""
    import oracle
    impl, kind = oracle.reference(), "reference"
    if impl is None:
        impl, kind = oracle.restatement(), "port"
    threads = os.cpu_count() or 1
    dt1, _ = _ref_solves(impl, n, 1, 1)  # one system: size the sample
    m = int(seconds / max(dt1, 1e-3)) * threads
    m = min(max(m, threads), args.count)
    dt, reps = _ref_solves(impl, n, m, threads)
    full = dt * args.count / m
    out = {"value": full, "unit": "s", "cores": threads, "kind": kind,
           "sample": f"systems 0..{m - 1} of {args.count} (N={n}) solved by the compiled "
                     f"reference on {threads} host threads in {dt:.2f} s (solve time only), "
                     f"scaled x{args.count / m:.1f} to the whole batch",
           "reasons": sorted({r["reason"] for r in reps if r["reason"]})}
    if gpu_x is not None:
        # the free parity check: every system the CPU leg solved against the GPU
        # batch's solution and history length, bit for bit
        import numpy as np
        k = min(m, gpu_x.shape[0])
        same = [bool(np.array_equal(reps[i]["x"].view(np.uint64), gpu_x[i].view(np.uint64))
                     and len(reps[i]["rhist"]) == int(gpu_rlen[i])) for i in range(k)]
        out["parity_checked_systems"] = k
        out["parity_all_checked_equal"] = all(same)
        out["parity_first_mismatch"] = None if all(same) else same.index(False)
    return out


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path on this host's cores."""
    if rank != 0:
        return
    n = N_SYS
    vals = []
    cpu = None
    for i in range(args.warmup + args.steps):
        cpu = cpu_sample(args, n, seconds=6.0)
        if i >= args.warmup:
            vals.append(cpu["value"])
    v = statistics.mean(vals)
    cpu["value"] = v
    line = {
        "impl": "reference", "metric": B.METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64/f32",
        "data": "synthetic (seeded: libstdc++ mt19937_64 per system index, SURVEY 8(d))",
        "config": {"workload": _workload(args, args.count), "n": n, "systems": args.count},
        "cpu_baseline": cpu,
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
